cd /root/repo; exec > >(tee gpurun_out/run.log) 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "not c4" 2>&1 | tail -2
q() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])"; }
for c in C3 C2 C1; do
echo "$c coupled"; timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | q
echo "$c local"; SP_FUSED_DEBUG_LOCAL=1 timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | q
done
