cd /root/repo; mkdir -p gpurun_out
for v in base cur; do echo "== $v" >> gpurun_out/ab.log; SP_LIB_AB=build/ab/$v.so timeout 300 python tools/time_score.py 4096 8192 16384 65536 2>&1 | cut -c1-120 >> gpurun_out/ab.log; done
bash tools/gpu_ab.sh "base cur" "--config C1" "--config C1 --kv e4m3" > /dev/null 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "forced or c1 or peer or split or head" 2>&1 | tail -2 >> gpurun_out/ab.log
