#!/bin/bash
# Round-2 final pass: GPU tests, smoke, default bench line, ncu launch list + --set full of the C3 score and select kernels.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_final.log) 2>&1
timeout 2400 python -m pytest tests -q -m gpu -x -rf --tb=short 2>&1 | grep -v "^randn\|^regimes\|^c3_planted\|^c4_\|^seq_select\|^run_host\|^full/\|^randn_c0\|^score_select" | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/r2_bench_C3.json 2> gpurun_out/r2_bench_C3.err; tail -c 600 gpurun_out/r2_bench_C3.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-tune --no-read-peak > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fused -s 4 -c 1 -o gpurun_out/r2_prof_fused -f \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-tune --no-read-peak > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_select -s 4 -c 1 -o gpurun_out/r2_prof_select -f \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-tune --no-read-peak > /dev/null 2>&1
ls -la gpurun_out/r2_launches.csv gpurun_out/r2_prof_*.ncu-rep
