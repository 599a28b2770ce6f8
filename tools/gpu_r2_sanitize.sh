#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_sanitize.log) 2>&1
for tool in memcheck synccheck racecheck initcheck; do
  echo "=== $tool"
  timeout 1500 compute-sanitizer --tool $tool --kernel-name kns=sp --print-limit 6 python tools/sanitize.py > /tmp/san_$tool.txt 2>&1
  grep -E "^========= (Invalid|Uninit|Race|Error|[A-Za-z]+ access|    at|ERROR SUMMARY|RACECHECK SUMMARY|Program hit)" /tmp/san_$tool.txt | head -30
  grep "sanitize workload done" /tmp/san_$tool.txt
done
