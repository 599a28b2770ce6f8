#!/bin/bash
# Boundary-counter chunk phase, batched epilogue loads: correctness, timelines, graph timings, benches.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/sel8.log) 2>&1
timeout 1200 python -m pytest tests/test_gpu_score_select.py -q -x -m gpu 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "forced or c1_full or c3_full or head_sharded or c0 or geometries or split or deterministic or lse or run_host" 2>&1 | tail -2
SP_LIB_AB=build/ab/seltrace.so SEL_GTIME=0 timeout 300 python tools/sel_trace.py
DIAG_NS=512,4096,16384,32768 DIAG_PLANS="8,16;8,18" timeout 900 python tools/c1_diag.py
for c in C3 C1; do
  for mode in "" "--two-launch"; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e $mode 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$c $mode step %.4f kernel %.4f gap %.1f us frac %.3f value %.2fM plan %s' % (d['ms_per_step'], r['kernel_ms'], 1000*(d['ms_per_step']-r['kernel_ms']), r['frac'], d['value']/1e6, d['config']['plan_tuned']), d['clocks']['sm_mhz'])"
  done
done
