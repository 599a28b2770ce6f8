#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_pst.log) 2>&1
for st in 2 3 4; do echo "stages<=$st"; SP_FUSED_MAXSTAGES=$st timeout 600 python tools/peer_replay.py C4 8 C3 8 2>&1 | cut -c1-110; done
for st in 2 3 4; do echo -n "single 16K/4K stages<=$st: "; SP_FUSED_MAXSTAGES=$st timeout 300 python tools/time_score.py 4096 16384 2>&1 | cut -c1-30 | tr '\n' ' '; echo; done
