#!/bin/bash
# Session-3 pass: GPU tests, smoke, bench lines (C3 default with e2e + cpu baseline; C0-C4), launch list, ncu captures.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/s3final.log) 2>&1
timeout 2400 python -m pytest tests -q -m gpu -x -rf --tb=short 2>&1 | grep -v "^randn\|^regimes\|^c3_planted\|^c4_\|^seq_select\|^run_host\|^full/\|^randn_c0\|^score_select\|^secondary\|^C\|^   " | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/s3f_bench_C3.json 2> gpurun_out/s3f_bench_C3.err; tail -c 300 gpurun_out/s3f_bench_C3.json; echo
for c in C1 C2 C4 C0; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/s3f_bench_$c.json 2> gpurun_out/s3f_bench_$c.err; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s3f_bench_ref.json 2> gpurun_out/s3f_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/s3f_launches.csv \
  python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-tune --no-read-peak > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fused -s 4 -c 1 -o gpurun_out/s3f_prof_fused -f \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-tune --no-read-peak > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_select -s 3 -c 1 -o gpurun_out/s3f_prof_select -f \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-tune --no-read-peak > /dev/null 2>&1
ls -la gpurun_out/s3f_launches.csv gpurun_out/s3f_prof_*.ncu-rep
