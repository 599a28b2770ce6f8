#!/bin/bash
# Explicit shared-memory accesses (LDS/STS/ATOMS) in the fused kernel: correctness, timelines, diag, benches.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/epi5.log) 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_score_select.py tests/test_gpu_edge.py tests/test_gpu_seq.py tests/test_gpu_f3.py tests/test_gpu_f4.py -q -x -m gpu -k "not c4_keep_sweep and not token_level" 2>&1 | tail -2
SP_LIB_AB=build/ab/seltrace.so SEL_GTIME=0 SEL_CFGS=C1 timeout 300 python tools/sel_trace.py 2>&1 | grep -v "^  alone\|score CTAs"
DIAG_NS=512,4096,16384,32768 DIAG_PLANS="8,16;8,18;4,37" timeout 900 python tools/c1_diag.py
for c in C3 C1 C2 C4; do
  for mode in "" "--two-launch"; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e $mode 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$c $mode step %.4f kernel %.4f gap %.1f us frac %.3f value %.2fM plan %s' % (d['ms_per_step'], r['kernel_ms'], 1000*(d['ms_per_step']-r['kernel_ms']), r['frac'], d['value']/1e6, d['config']['plan_tuned']), d['clocks']['sm_mhz'])"
  done
done
timeout 600 python tools/peer_replay.py C3 8 C4 8 C4 4 2>&1 | tail -6
