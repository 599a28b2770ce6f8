#!/bin/bash
# Round-2 full pass: GPU tests, smoke, bench lines, per-rank peer replay incl. plan sweep.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_full.log) 2>&1
timeout 2400 python -m pytest tests -q -m gpu -x -rf --tb=short 2>&1 | grep -v "^randn\|^regimes\|^c3_planted\|^c4_\|^seq_select\|^run_host\|^full/\|^randn_c0" | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/r2_bench_C3.json 2> gpurun_out/r2_bench_C3.err; tail -c 1500 gpurun_out/r2_bench_C3.json
for c in C1 C2 C4; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2_bench_$c.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$c step %.4f ms kernel %.4f ms frac %.3f value %.3g' % (d['ms_per_step'], r['kernel_ms'], r['frac'], d['value']))"; done
timeout 900 python tools/peer_replay.py C4 8 C4 8:32,4 C4 8:8,18 C4 8:37,4 C4 8:16,8 C3 8 C3 8:4,37 C3 8:16,9 2>&1
