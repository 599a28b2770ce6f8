#!/bin/bash
# Atomic-max cross-unit-group epilogue: full GPU suite, timelines, diag, benches.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/epi2.log) 2>&1
SP_LIB_AB=build/ab/seltrace.so SEL_GTIME=0 timeout 300 python tools/sel_trace.py 2>&1 | grep -v "^  alone"
DIAG_NS=512,4096,16384,32768 DIAG_PLANS="8,16;8,18;4,37;16,8" timeout 900 python tools/c1_diag.py
for c in C3 C1; do
  for mode in "" "--two-launch"; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e $mode 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$c $mode step %.4f kernel %.4f gap %.1f us frac %.3f value %.2fM plan %s' % (d['ms_per_step'], r['kernel_ms'], 1000*(d['ms_per_step']-r['kernel_ms']), r['frac'], d['value']/1e6, d['config']['plan_tuned']), d['clocks']['sm_mhz'])"
  done
done
timeout 2400 python -m pytest tests -q -m gpu -x -rf --tb=short 2>&1 | grep -v "^randn\|^regimes\|^c3_planted\|^c4_\|^seq_select\|^run_host\|^full/\|^randn_c0\|^score_select\|^secondary" | tail -6
