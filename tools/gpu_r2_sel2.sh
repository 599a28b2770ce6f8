#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_sel2.log) 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seq.py tests/test_gpu_f3.py -q -m gpu -x -rf --tb=short -k "select or seq or ragged or secondary or token_level or gather" 2>&1 | tail -3
timeout 300 python tools/time_select.py 2>&1 | tail -9
timeout 300 python bench.py --config C4 --chunk 1 --pool 1 --keep 0.9 --no-cpu-baseline --no-e2e --no-read-peak 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('C4 token-level keep .9: step %.4f ms kernel %.4f ms' % (d['ms_per_step'], r['kernel_ms']))"
