#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_cap.log) 2>&1
timeout 600 python tools/time_score.py 4096 16384 32768 131072 2>&1 | cut -c1-60
timeout 900 python tools/peer_replay.py C4 8 C3 8 2>&1 | cut -c1-120
for c in C3 C1 C2; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --no-read-peak 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$c step %.4f ms kernel %.4f ms frac %.3f tuned %s' % (d['ms_per_step'], r['kernel_ms'], r['frac'], d['config']['plan_tuned']))"; done
