cd /root/repo; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_f3.py -x -q 2>&1 | tail -3 | tee gpurun_out/f34.txt
for a in "--kv e4m3 --paged 16" "--kv e4m3 --paged 128" "--kv e4m3"; do echo -n "$a: "; timeout 300 python bench.py $a --steps 10 --warmup 4 --no-cpu-baseline 2>/tmp/e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('score %.4f ms frac %.3f' % (d['roofline']['kernel_ms'], d['roofline']['frac']))" || tail -3 /tmp/e; done 2>&1 | tee -a gpurun_out/f34.txt
