cd /root/repo; mkdir -p gpurun_out
bash tools/gpu_ab.sh "base cur" "--config C3" "--config C1"
timeout 600 python -m pytest tests/test_gpu_f3.py -x -q 2>&1 | tail -2 | tee -a gpurun_out/ab.log
