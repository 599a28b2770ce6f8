#!/bin/bash
# Graph-timed plan tuner: benches, then the full GPU suite and smoke.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/tune2.log) 2>&1
for c in C1 C3 C2 C4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$c step %.4f kernel %.4f frac %.3f read_frac %.3f value %.2fM plan %s' % (d['ms_per_step'], r['kernel_ms'], r['frac'], r['read_peak']['frac'], d['value']/1e6, d['config']['plan_tuned']), d['clocks']['sm_mhz'])"
done
timeout 2400 python -m pytest tests -q -m gpu -x -rf --tb=short 2>&1 | grep -v "^randn\|^regimes\|^c3_planted\|^c4_\|^seq_select\|^run_host\|^full/\|^randn_c0\|^score_select\|^secondary\|^C\|^   " | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
