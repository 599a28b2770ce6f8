#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_c1trace.log) 2>&1
SP_LIB_AB=build/ab/trace.so timeout 300 python tools/trace_fused.py --config C1 --plan 8,16 2>&1 | head -80
