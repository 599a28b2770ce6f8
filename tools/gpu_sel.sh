cd /root/repo; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f3.py tests/test_gpu_edge.py -x -q -k "select or ragged or c1_full or c3_full or c2_sampled or keep or wave" 2>&1 | tail -2 | tee gpurun_out/ab.log
bash tools/gpu_ab.sh "base cur" "--config C1 --no-tune" "--config C3 --no-tune" "--config C2 --no-tune" > /dev/null 2>&1
