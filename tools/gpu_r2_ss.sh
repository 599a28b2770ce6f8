#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_ss.log) 2>&1
timeout 1500 python -m pytest tests/test_gpu_score_select.py tests/test_gpu_host.py -q -m gpu -x -rf --tb=short 2>&1 | grep -v "^score_select\|^run_host" | tail -15
for c in C3 C1 C4 C2; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --no-read-peak 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$c step %.4f ms kernel %.4f ms (score only %.4f) frac %.3f launches %d' % (d['ms_per_step'], r['kernel_ms'], r['score_only_ms'], r['frac'], d['gpu_launches']))"; done
