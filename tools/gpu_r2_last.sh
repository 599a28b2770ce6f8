#!/bin/bash
# Default bench line and reference arm (defaults), wall clock of each.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/last.log) 2>&1
s=$(date +%s.%N); timeout 900 python bench.py > gpurun_out/last_bench.json 2> gpurun_out/last_bench.err; e=$(date +%s.%N); echo "bench wall $(echo "$e - $s" | bc) s"
s=$(date +%s.%N); timeout 900 python bench.py --impl reference > gpurun_out/last_ref.json 2> gpurun_out/last_ref.err; e=$(date +%s.%N); echo "reference wall $(echo "$e - $s" | bc) s"
python -c "
import json
for f in ('gpurun_out/last_bench.json','gpurun_out/last_ref.json'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d.get('value'), d.get('ms_per_step'), d.get('steps'), (d.get('roofline') or {}).get('frac'), d.get('clocks'), (d.get('e2e') or {}).get('value'))"
