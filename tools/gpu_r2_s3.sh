#!/bin/bash
# Round-2 session-3 check of HEAD: GPU tests, smoke, bench lines C3 (default), C1, C4.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2s3.log) 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -q -m gpu -x -rf --tb=short 2>&1 | grep -v "^randn\|^regimes\|^c3_planted\|^c4_\|^seq_select\|^run_host\|^full/\|^randn_c0\|^score_select" | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in C3 C1 C4; do
  timeout 600 python bench.py --config $c > gpurun_out/s3_bench_$c.json 2> gpurun_out/s3_bench_$c.err; tail -c 400 gpurun_out/s3_bench_$c.json; echo
done
