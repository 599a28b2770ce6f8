#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_sel5.log) 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seq.py -q -m gpu -x -k "select or seq or secondary" 2>&1 | tail -1
for i in 1 2; do timeout 300 python tools/time_select.py 2>&1 | tail -9; done
