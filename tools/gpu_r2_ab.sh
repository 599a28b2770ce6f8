#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_ab.log) 2>&1
for rep in 1 2; do for v in r1 cur2; do echo "== $v"; SP_LIB_AB=build/ab/$v.so timeout 300 python tools/time_score.py 4096 32768 2>&1 | cut -c1-40; done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seq.py -q -m gpu -x -k "peer or dist" 2>&1 | tail -2
timeout 900 python tools/peer_replay.py C4 8 C3 8 C4 4 C4 2 2>&1
