#!/bin/bash
# One GPU-box pass: full GPU tests, smoke, default bench line, ncu launch list
# and --set full captures of the fused score and select kernels.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/full.log) 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-tune > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fused -s 6 -c 1 -o gpurun_out/prof_fused -f \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-tune > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_select -s 6 -c 1 -o gpurun_out/prof_select -f \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-tune > /dev/null 2>&1
ls -la gpurun_out/launches.csv gpurun_out/*.ncu-rep
# secondary lines (rows f3 / f4) and the e4m3 kernel's DRAM traffic
for a in "--kv e4m3" "--kv e4m3 --config C2" "--paged 16" "--paged 256" "--paged 16 --config C2 --ragged"; do
  n=$(echo "$a" | tr -d ' -'); timeout 300 python bench.py $a --no-cpu-baseline > gpurun_out/bench_$n.json 2>/dev/null; tail -c 400 gpurun_out/bench_$n.json
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fused -c 2 --csv \
  --log-file gpurun_out/f4_traffic.csv python bench.py --kv e4m3 --steps 1 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fused -c 2 --csv \
  --log-file gpurun_out/f3_traffic.csv python bench.py --paged 16 --steps 1 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
