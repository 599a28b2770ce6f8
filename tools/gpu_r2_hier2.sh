#!/bin/bash
# Round-2: designated-merger hierarchical exchange + one-launch PDL select: correctness, sweeps, per-rank replay, bench.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_hier2.log) 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seq.py tests/test_gpu_f3.py tests/test_gpu_host.py -q -m gpu -x \
  -k "forced or peer or c1_full or c0 or geometries or seq or tune or split or head or deterministic or lse or select or ragged or gather or host" 2>&1 | tail -4
timeout 900 python tools/plan_sweep.py C1 8,16,0 8,18,0 8,16,1 8,18,1 4,37,1 4,37,0 \
  C3 37,4,0 37,4,1 64,2,1 74,2,1 32,4,1 148,1,1 128,1,1 \
  C4 69,2,0 74,2,0 74,2,1 147,1,1 148,1,1 128,1,1 \
  C2 1,2,0 1,2,1 2>&1
timeout 600 python tools/peer_replay.py C3 2 C3 4 C3 8 C4 2 C4 4 C4 8 2>&1
for c in C1 C3; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_pdl_$c.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_pdl_$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$c', 'step %.4f ms kernel %.4f ms select+gaps %.1f us frac %.3f plan %s tuned %s' % (d['ms_per_step'], r['kernel_ms'], 1000*(d['ms_per_step']-r['kernel_ms']), r['frac'], d['config']['plan'], d['config']['plan_tuned']))"; done
