#!/bin/bash
# Round-2 baseline pass: GPU tests, smoke, default bench line, C1 line.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_base.log) 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/r2_bench_C3.json 2> gpurun_out/r2_bench_C3.err; tail -1 gpurun_out/r2_bench_C3.json
timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/r2_bench_C1.json 2>/dev/null; tail -1 gpurun_out/r2_bench_C1.json
