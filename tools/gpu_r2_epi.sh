#!/bin/bash
# Cross-unit-group epilogue rework: parity subset, small-prompt diagnosis, selection timeline.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/epi.log) 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "forced or c1_full or c3_full or head_sharded or c0 or geometries or split or deterministic or lse" 2>&1 | tail -3
DIAG_NS=512,1024,2048,4096,8192,16384,32768 DIAG_PLANS="8,16;4,37;8,18;4,32;16,9;2,74" timeout 900 python tools/c1_diag.py
SP_LIB_AB=build/ab/seltrace.so timeout 300 python tools/sel_trace.py
