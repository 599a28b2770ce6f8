#!/bin/bash
# C1/C3 bench lines vs the number of timed steps (graph length) and repeated.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/steps.log) 2>&1
for st in 20 100 20 100; do for c in C1 C3; do
  timeout 600 python bench.py --config $c --steps $st --no-cpu-baseline --no-e2e --no-read-peak 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$c steps $st step %.4f kernel %.4f frac %.3f value %.2fM tuned %.4f' % (d['ms_per_step'], r['kernel_ms'], r['frac'], d['value']/1e6, d['config']['plan_tuned']['ms_per_launch']))"
done; done
