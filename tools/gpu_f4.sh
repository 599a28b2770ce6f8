#!/bin/bash
# Row f4 pass: e4m3 parity tests, e4m3 bench lines (C3, C2, C1), DRAM traffic of the e4m3 fused kernel.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/f4.log) 2>&1
timeout 900 python -m pytest tests/test_gpu_f4.py -x -q 2>&1 | tail -15
for c in C3 C2 C1; do
  timeout 300 python bench.py --kv e4m3 --config $c --no-cpu-baseline > gpurun_out/bench_f4_$c.json 2> gpurun_out/bench_f4_$c.err; tail -c 1500 gpurun_out/bench_f4_$c.json; echo
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fused -c 3 --csv \
  --log-file gpurun_out/f4_traffic.csv python bench.py --kv e4m3 --steps 1 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
tail -4 gpurun_out/f4_traffic.csv
