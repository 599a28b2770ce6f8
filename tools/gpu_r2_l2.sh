#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_l2.log) 2>&1
for rep in 1 2; do for h in 0 1; do echo "== hint $h"; SP_FUSED_L2HINT=$h timeout 300 python tools/time_score.py 4096 16384 32768 2>&1 | cut -c1-40; SP_FUSED_L2HINT=$h timeout 300 python tools/plan_sweep.py C2 1,2,0 2>&1 | tail -1; done; done
