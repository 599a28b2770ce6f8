#!/bin/bash
# One GPU-box pass: full GPU tests, smoke, default bench line, ncu launch list
# and --set full captures of the fused score and select kernels.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/full.log) 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fused -s 6 -c 1 -o gpurun_out/prof_fused -f \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_select -s 6 -c 1 -o gpurun_out/prof_select -f \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
ls -la gpurun_out/launches.csv gpurun_out/*.ncu-rep
