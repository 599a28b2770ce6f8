#!/bin/bash
# A/B: deferred-finalize staging size (partial-map loads per selection thread), same box.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/loads.log) 2>&1
for rep in 1 2; do
for L in 16 8 4; do
  for c in C1 C3 C2; do
    SP_DEFER_LOADS=$L timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --no-read-peak 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('loads $L $c step %.4f kernel %.4f gap %.1f us value %.2fM' % (d['ms_per_step'], r['kernel_ms'], 1000*(d['ms_per_step']-r['kernel_ms']), d['value']/1e6))"
  done
done
done
