#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_stages.log) 2>&1
for st in 3 4 5 6 8; do echo -n "C3 e4m3 stages<=$st: "; SP_FUSED_MAXSTAGES=$st timeout 300 python tools/plan_sweep.py --kv e4m3 C3 37,4,0 2>&1 | tail -1; done
for st in 3 4 5 6 8; do echo -n "C1 e4m3 stages<=$st: "; SP_FUSED_MAXSTAGES=$st timeout 300 python tools/plan_sweep.py --kv e4m3 C1 8,16,0 2>&1 | tail -1; done
for st in 3 4; do echo -n "C4 stages<=$st: "; SP_FUSED_MAXSTAGES=$st timeout 300 python tools/plan_sweep.py C4 69,2,0 2>&1 | tail -1; done
for st in 3 4 5; do echo -n "N16K stages<=$st: "; SP_FUSED_MAXSTAGES=$st timeout 300 python tools/time_score.py 16384 2>&1 | cut -c1-40; done
