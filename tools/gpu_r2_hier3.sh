#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_hier3.log) 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seq.py tests/test_gpu_f3.py tests/test_gpu_host.py -q -m gpu -x -rf \
  -k "forced or peer or c1_full or c0 or geometries or seq or tune or split or head or deterministic or lse or select or ragged or gather or host" 2>&1 | tail -25
timeout 600 python tools/peer_replay.py C3 2 C3 4 C3 8 C4 2 C4 4 C4 8 2>&1
q() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('step %.4f ms kernel %.4f ms select+gaps %.1f us' % (d['ms_per_step'], r['kernel_ms'], 1000*(d['ms_per_step']-r['kernel_ms'])))"; }
for rep in 1 2; do for c in C1 C3; do
  echo -n "$c pdl: "; timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --no-read-peak 2>/dev/null | q
  echo -n "$c nopdl: "; SP_SELECT_NO_PDL=1 timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --no-read-peak 2>/dev/null | q
done; done
timeout 300 python tools/time_select.py 2>&1 | tail -8; SP_SELECT_NO_PDL=1 timeout 300 python tools/time_select.py 2>&1 | tail -8
timeout 900 python tools/plan_sweep.py C1 8,16,0 8,16,1 4,37,1 8,18,1 16,9,1 \
  C3 37,4,0 37,4,1 64,2,1 74,2,1 32,4,1 148,1,1 \
  C4 69,2,0 74,2,1 147,1,1 128,1,1 C2 1,2,0 1,2,1 2>&1
