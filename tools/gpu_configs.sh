#!/bin/bash
# One bench line per BASELINE.json config (single GPU) + the reference arm, into gpurun_out/.
cd /root/repo; mkdir -p gpurun_out
for c in C1 C2 C4 C0; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_cfg_$c.json 2> gpurun_out/bench_cfg_$c.err; tail -c 300 gpurun_out/bench_cfg_$c.json; echo; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2>&1; tail -c 300 gpurun_out/bench_reference.json
