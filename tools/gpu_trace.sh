#!/bin/bash
# Timelines of the fused kernel from a -DSP_FUSED_TRACE build (build/ab/trace.so).
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/trace.log) 2>&1
for args in "--config C2 --kv e4m3" "--config C2" "--config C3 --kv e4m3" "--config C3" "--config C1 --kv e4m3"; do
  echo "=== $args"; SP_LIB_AB=build/ab/trace.so timeout 300 python tools/trace_fused.py $args 2>&1 | grep -v "^   \|^CTA [0-9]*: first\|tile  " 
done
