#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_noacc.log) 2>&1
for rep in 1 2; do for v in cur3 noacc; do echo "== $v"; SP_LIB_AB=build/ab/$v.so timeout 300 python tools/time_score.py 4096 32768 2>&1 | cut -c1-40; done; done
