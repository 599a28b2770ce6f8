#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2s3_sanitize.log) 2>&1
which compute-sanitizer || export PATH=/usr/local/cuda/bin:$PATH
timeout 300 python tools/sanitize.py 2>&1 | tail -3
for tool in memcheck synccheck racecheck; do
  echo "=== $tool"
  timeout 1500 compute-sanitizer --tool $tool --kernel-name kns=sp --print-limit 6 python tools/sanitize.py > gpurun_out/san_$tool.txt 2>&1
  grep -E "^========= (Invalid|Uninit|Race|Error|[A-Za-z]+ access|    at|ERROR SUMMARY|RACECHECK SUMMARY|Program hit)" gpurun_out/san_$tool.txt | head -30
  grep "sanitize workload done" gpurun_out/san_$tool.txt
  tail -3 gpurun_out/san_$tool.txt
done
