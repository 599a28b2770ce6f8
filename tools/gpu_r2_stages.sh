#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_stages.log) 2>&1
for st in 3 4 5; do for nq in 2 4; do echo -n "C1 stages<=$st nq=$nq: "; SP_FUSED_NQ=$nq SP_FUSED_MAXSTAGES=$st timeout 300 python tools/plan_sweep.py C1 8,16 2>&1 | tail -1; done; done
for st in 3 4 5; do echo -n "C3 stages<=$st: "; SP_FUSED_MAXSTAGES=$st timeout 300 python tools/plan_sweep.py C3 37,4 2>&1 | tail -1; done
for st in 2 3 4; do echo -n "C2 stages<=$st: "; SP_FUSED_MAXSTAGES=$st timeout 300 python tools/plan_sweep.py C2 1,2 2>&1 | tail -1; done
