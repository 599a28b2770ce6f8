#!/bin/bash
# Round-2: sequence-sharded select (row e), run_host parity, full GPU suite, bench lines.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_row_e.log) 2>&1
timeout 900 python -m pytest tests/test_gpu_seq.py tests/test_gpu_host.py -q -m gpu -x 2>&1 | tail -30
timeout 2400 python -m pytest tests -q -m gpu -x --deselect tests/test_gpu_seq.py --deselect tests/test_gpu_host.py 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/r2_bench_C3.json 2> gpurun_out/r2_bench_C3.err; tail -1 gpurun_out/r2_bench_C3.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_ref.json 2>&1; tail -1 gpurun_out/r2_bench_ref.json
