cd /root/repo; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_f3.py -x -q 2>&1 | tail -2 | tee gpurun_out/bs.txt
for a in "--paged 8" "--paged 16" "--paged 32" "--paged 64" "--paged 128" "--paged 256" ""; do echo -n "$a: "; timeout 300 python bench.py $a --steps 10 --warmup 4 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('score %.4f ms frac %.3f' % (d['roofline']['kernel_ms'], d['roofline']['frac']))"; done 2>&1 | tee -a gpurun_out/bs.txt
rm -f gpurun_out/ab.log; bash tools/gpu_ab.sh "base cur" "--config C3" "--config C1" "--config C2" > /dev/null 2>&1; cat gpurun_out/ab.log >> gpurun_out/bs.txt
