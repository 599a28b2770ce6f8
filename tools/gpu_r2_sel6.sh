#!/bin/bash
# Selection phase A in the score kernel's epilogue + one-barrier radix passes + flat compaction.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/sel6.log) 2>&1
timeout 1200 python -m pytest tests/test_gpu_score_select.py tests/test_gpu_seq.py tests/test_gpu_f3.py tests/test_gpu_edge.py -q -x -m gpu 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "select or gather or c1_full or c3_full or planted or run_host or secondary or token_level" 2>&1 | tail -3
SP_LIB_AB=build/ab/seltrace.so timeout 300 python tools/sel_trace.py
for c in C3 C1; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/s6_bench_$c.json 2> gpurun_out/s6_bench_$c.err; tail -c 1500 gpurun_out/s6_bench_$c.json | head -c 700; echo
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --two-launch > gpurun_out/s6_bench2_$c.json 2> gpurun_out/s6_bench2_$c.err; tail -c 1500 gpurun_out/s6_bench2_$c.json | head -c 700; echo
done
