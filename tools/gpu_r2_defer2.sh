#!/bin/bash
# Deferred finalize with one batch of partial-map loads per thread: correctness, timelines, A/B vs two launches and min n_ug.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/defer4.log) 2>&1
timeout 1500 python -m pytest tests/test_gpu_score_select.py tests/test_gpu_host.py -q -x -m gpu 2>&1 | tail -2
SP_DEFER_MIN_UG=2 timeout 900 python -m pytest tests/test_gpu_score_select.py tests/test_gpu_parity.py -k "forced or c1_full or c3_full or head or split or geometries or c0" -q -x -m gpu 2>&1 | tail -2
SP_LIB_AB=build/ab/seltrace.so SEL_GTIME=0 timeout 300 python tools/sel_trace.py 2>&1 | grep "score_select\|per CTA"
for c in C3 C1 C2 C4; do
  for mode in "" "--two-launch" "DEF2"; do
  if [ "$mode" = "DEF2" ]; then export SP_DEFER_MIN_UG=2; mode=""; tag=def2; else unset SP_DEFER_MIN_UG; tag="$mode"; fi
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e $mode 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$c $tag step %.4f kernel %.4f gap %.1f us frac %.3f value %.2fM plan %s' % (d['ms_per_step'], r['kernel_ms'], 1000*(d['ms_per_step']-r['kernel_ms']), r['frac'], d['value']/1e6, d['config']['plan_tuned']), d['clocks']['sm_mhz'])"
  done
done
unset SP_DEFER_MIN_UG
