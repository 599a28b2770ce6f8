#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_selq.log) 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seq.py tests/test_gpu_f3.py -q -m gpu -x -k "select or gather or seq or ragged or c1_full or c0 or both_regimes" 2>&1 | tail -2
timeout 300 python tools/time_select.py 2>&1 | tail -7
