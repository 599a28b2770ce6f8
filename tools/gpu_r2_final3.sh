#!/bin/bash
# Session-3 final pass: bench lines (C3 default with e2e + cpu baseline; C0-C4; secondary lines), launch list, ncu captures.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/final4.log) 2>&1
timeout 600 python bench.py > gpurun_out/f4_bench_C3.json 2> gpurun_out/f4_bench_C3.err; tail -c 300 gpurun_out/f4_bench_C3.json; echo
for c in C1 C2 C4 C0; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/f4_bench_$c.json 2> gpurun_out/f4_bench_$c.err; done
timeout 600 python bench.py --kv e4m3 --no-cpu-baseline --no-e2e > gpurun_out/f4_bench_f4_C3.json 2> /dev/null
timeout 600 python bench.py --paged 16 --no-cpu-baseline --no-e2e > gpurun_out/f4_bench_f4_paged16.json 2> /dev/null
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f4_bench_ref.json 2> gpurun_out/f4_bench_ref.err
for c in C3 C1 C2 C4 C0 f4_C3 f4_paged16; do python -c "
import json,sys; d=json.loads(open('gpurun_out/f4_bench_$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$c step %.4f kernel %.4f frac %.3f value %.2fM e2e %s launch %s' % (d['ms_per_step'], r['kernel_ms'], r['frac'], d['value']/1e6, (d.get('e2e') or {}).get('value'), d['config'].get('launch')), d['clocks'])"; done
timeout 2400 python -m pytest tests -q -m gpu -x -rf --tb=short 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/f4_launches.csv \
  python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-tune --no-read-peak > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fused -s 4 -c 1 -o gpurun_out/f4_prof_fused -f \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-tune --no-read-peak > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fused -s 1 -c 1 -o gpurun_out/f4_prof_fused_c1 -f \
  python bench.py --config C1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-tune --no-read-peak --two-launch > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_select -s 3 -c 1 -o gpurun_out/f4_prof_select -f \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-tune --no-read-peak > /dev/null 2>&1
ls -la gpurun_out/f4_launches.csv gpurun_out/f4_prof_*.ncu-rep
