#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_diag.log) 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seq.py -q -m gpu -x -k "peer or dist" 2>&1 | tail -2
timeout 900 python tools/peer_replay.py C3 8 C4 8 C4 4 C4 2 C3 2 2>&1
timeout 600 python tools/time_score.py 4096 16384 2>&1
SP_LIB_AB=build/ab/trace.so timeout 600 python tools/peer_diag.py 4096 8 2>&1 | tail -3
SP_LIB_AB=build/ab/trace.so timeout 600 python tools/peer_diag.py 16384 8 2>&1 | tail -3
