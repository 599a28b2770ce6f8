#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_c1prof.log) 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fused -s 4 -c 1 -o gpurun_out/prof_c1_fused -f \
  python bench.py --config C1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-read-peak --plan 8,16 2>&1 | tail -15
ls -la gpurun_out/*.ncu-rep
