#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_sel.log) 2>&1
for tpc in 256 512 1024 2048 4096; do echo "== tpc $tpc"; SP_SELECT_TPC=$tpc timeout 300 python tools/time_select.py 2>&1 | tail -7 | head -4; done
