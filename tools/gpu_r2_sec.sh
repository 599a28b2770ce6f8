#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_sec.log) 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -rf --tb=short -k "secondary or token_level" 2>&1 | grep -v "^full/" | tail -14
for a in "--config C1 --R 1" "--config C3 --R 1" "--config C1 --R 9" "--config C1 --chunk 1 --pool 1" "--config C4 --chunk 1 --pool 1 --keep 0.9"; do timeout 300 python bench.py $a --no-cpu-baseline --no-e2e --no-read-peak > gpurun_out/r2_bench_sec_$(echo $a | tr -d ' -').json 2>/dev/null; python -c "
import json,sys; d=json.loads(open('gpurun_out/r2_bench_sec_$(echo $a | tr -d ' -').json').read().strip().splitlines()[-1]); r=d['roofline']
print('$a: %s step %.4f ms kernel %.4f ms frac %.3f value %.3g' % (d['config']['workload'], d['ms_per_step'], r['kernel_ms'], r['frac'], d['value']))"; done
