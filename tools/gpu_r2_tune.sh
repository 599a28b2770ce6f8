#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_tune.log) 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f4.py -q -m gpu -x -k "tune or forced or peer or c1_full or c3_full" 2>&1 | tail -2
for a in "--config C3" "--config C1" "--config C2" "--config C4" "--config C3 --kv e4m3" "--config C2 --kv e4m3"; do timeout 300 python bench.py $a --no-cpu-baseline --no-e2e --no-read-peak 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$a: step %.4f ms kernel %.4f ms frac %.3f stages %s tuned %s' % (d['ms_per_step'], r['kernel_ms'], r['frac'], d['config']['plan']['stages'] if d['config']['plan'] else None, d['config']['plan_tuned']))"; done
timeout 600 python tools/peer_replay.py C4 8 C3 8 2>&1 | cut -c1-110
