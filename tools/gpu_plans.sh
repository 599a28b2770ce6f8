#!/bin/bash
# Plan sweep of the fused kernel: tools/gpu_plans.sh "<bench args>" "plan1 plan2 ..." [more pairs]
cd /root/repo; mkdir -p gpurun_out; exec > >(tee -a gpurun_out/plans.log) 2>&1
q() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('step %.4f ms  score %.4f ms  frac %.3f  plan %s' % (d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['config']['plan']))"; }
while [ $# -ge 2 ]; do
  args=$1; plans=$2; shift 2
  for pl in auto $plans; do
    echo -n "$args | $pl: "
    if [ "$pl" = auto ]; then timeout 300 python bench.py $args --steps 10 --warmup 4 --no-e2e --no-cpu-baseline 2>/tmp/e | q || tail -2 /tmp/e
    else timeout 300 python bench.py $args --plan $pl --steps 10 --warmup 4 --no-e2e --no-cpu-baseline 2>/tmp/e | q || tail -2 /tmp/e; fi
  done
done
