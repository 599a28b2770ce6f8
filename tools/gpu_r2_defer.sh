#!/bin/bash
# Deferred finalize (the selection computes the importance from the partial maps): correctness, timelines, benches.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/defer.log) 2>&1
timeout 1500 python -m pytest tests/test_gpu_score_select.py tests/test_gpu_host.py -q -x -m gpu 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "run_host or select" 2>&1 | tail -2
SP_LIB_AB=build/ab/seltrace.so SEL_GTIME=0 timeout 300 python tools/sel_trace.py 2>&1 | grep -v "^  alone\|score CTAs\|after score"
for c in C3 C1 C2 C4; do
  for mode in "" "--two-launch"; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e $mode 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$c $mode step %.4f kernel %.4f gap %.1f us frac %.3f value %.2fM plan %s' % (d['ms_per_step'], r['kernel_ms'], 1000*(d['ms_per_step']-r['kernel_ms']), r['frac'], d['value']/1e6, d['config']['plan_tuned']), d['clocks']['sm_mhz'])"
  done
done
