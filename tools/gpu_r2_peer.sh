#!/bin/bash
# Round-2: pipelined peer exchange + select workspace fix: correctness, per-rank replay, benches.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_peer.log) 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seq.py tests/test_gpu_f3.py tests/test_gpu_host.py -q -m gpu -x -rf --tb=short \
  -k "split_api or forced or peer or c1_full or c0 or geometries or seq or tune or split or head or deterministic or lse or select or ragged or gather or host" 2>&1 | tail -25
timeout 600 python tools/peer_replay.py C3 2 C3 4 C3 8 C4 2 C4 4 C4 8 2>&1
timeout 600 python tools/time_score.py 4096 8192 16384 32768 65536 2>&1
for c in C1 C3; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --no-read-peak 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$c step %.4f ms kernel %.4f ms select+gaps %.1f us' % (d['ms_per_step'], r['kernel_ms'], 1000*(d['ms_per_step']-r['kernel_ms'])))"; done
