cd /root/repo; mkdir -p gpurun_out
bash tools/gpu_plans.sh "--config C1" "32,4 16,9 4,37 32,2 16,8 8,16 4,32 2,64 8,9 16,4"
SP_LIB_AB=build/ab/trace.so timeout 300 python tools/trace_fused.py --config C1 > gpurun_out/trace.log 2>&1
