#!/bin/bash
# Last check of HEAD: selection/score_select/host tests, smoke, default bench line, reference arm (defaults).
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/last.log) 2>&1
timeout 1500 python -m pytest tests/test_gpu_score_select.py tests/test_gpu_host.py tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x -m gpu -k "not c4_keep_sweep and not token_level" 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
/usr/bin/time -f "wall %e s" timeout 900 python bench.py > gpurun_out/last_bench.json 2> gpurun_out/last_bench.err; tail -1 gpurun_out/last_bench.err
/usr/bin/time -f "wall %e s" timeout 900 python bench.py --impl reference > gpurun_out/last_ref.json 2> gpurun_out/last_ref.err; tail -1 gpurun_out/last_ref.err
python -c "
import json
for f in ('gpurun_out/last_bench.json','gpurun_out/last_ref.json'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d.get('value'), d.get('ms_per_step'), d.get('steps'), (d.get('roofline') or {}).get('frac'), d.get('clocks'))"
