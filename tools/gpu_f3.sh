#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/f3.log) 2>&1
timeout 600 python -m pytest tests/test_gpu_f3.py -x -q 2>&1 | tail -2
for a in "--config C3" "--config C3 --paged 16" "--config C3 --paged 16 --paged-layout nhd" "--config C3 --paged 256" "--config C2 --paged 16" "--config C2 --paged 16 --ragged" "--config C3 --paged 64" "--config C1 --paged 16"; do
  timeout 300 python bench.py $a --no-cpu-baseline > /tmp/o.json 2>/tmp/e || tail -3 /tmp/e
  python -c "import json; d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); print('$a', '| step %.4f ms score %.4f ms frac %.3f value %.3g' % (d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['value']))"
  n=$(echo "$a" | tr -d ' -'); tail -1 /tmp/o.json > gpurun_out/bench_f3_$n.json
done
