#!/bin/bash
# Round-2: hierarchical exchange -- correctness (parity, forced plans, peer virtual ranks) and plan sweeps.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_hier.log) 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seq.py tests/test_gpu_f4.py -q -m gpu -x \
  -k "forced or peer or c1_full or c3_full or c0 or geometries or seq or tune or split or head or deterministic or lse" 2>&1 | tail -4
timeout 900 python tools/plan_sweep.py C1 8,16,0 8,18,0 8,16,1 8,18,1 4,37,1 16,9,1 32,4,1 16,8,1 2,74,1 \
  C3 37,4,0 37,4,1 64,2,1 74,2,1 32,4,1 148,1,1 128,1,1 \
  C4 74,2,0 74,2,1 147,1,1 148,1,1 128,1,1 \
  C2 1,2,0 1,2,1 2,1,0 2,1,1 2>&1
timeout 600 python tools/peer_time.py C3 2 C3 4 C3 8 C4 2 C4 4 C4 8 2>&1
