#!/bin/bash
# Per-rank peer-kernel replays and the C1 kernel after the branch-free epilogue loads.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/peer2.log) 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "forced or peer or head or split or c1_full" 2>&1 | tail -2
timeout 600 python tools/peer_replay.py C4 8 C3 8 C4 4 C4 2 2>&1 | tail -6
DIAG_NS=4096,16384 DIAG_PLANS="8,16;8,18" timeout 900 python tools/c1_diag.py
for i in 1 2; do timeout 600 python bench.py --config C1 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('C1 step %.4f kernel %.4f frac %.3f value %.2fM plan %s' % (d['ms_per_step'], r['kernel_ms'], r['frac'], d['value']/1e6, d['config']['plan_tuned']))"; done
