#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_sanitize.log) 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  echo "=== $tool"
  timeout 1200 compute-sanitizer --tool $tool --kernel-regex kns=sp --print-limit 20 python tools/sanitize.py 2>&1 | grep -v "^$" | tail -12
done
