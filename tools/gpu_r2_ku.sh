#!/bin/bash
# A/B: epilogue loads in flight per thread (24 vs 32) and C1 plans, same box.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/ku.log) 2>&1
for lib in ku24 ku32 ku24 ku32; do
  for c in C1 C3; do
    SP_LIB_AB=build/ab/$lib.so timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --no-read-peak 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$lib $c step %.4f kernel %.4f frac %.3f value %.2fM plan %s' % (d['ms_per_step'], r['kernel_ms'], r['frac'], d['value']/1e6, d['config']['plan_tuned']))"
  done
done
for pl in 8,16 8,18; do SP_LIB_AB=build/ab/ku24.so timeout 600 python bench.py --config C1 --plan $pl --no-cpu-baseline --no-e2e --no-read-peak 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('plan $pl C1 step %.4f kernel %.4f frac %.3f' % (d['ms_per_step'], r['kernel_ms'], r['frac']))"; done
