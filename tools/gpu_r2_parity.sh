#!/bin/bash
# Round-2 parity additions: device generator modes, full-mantissa inputs, planted exact-regime fixtures.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/r2_parity.log) 2>&1
timeout 2400 python -m pytest tests/test_gpu_parity.py -q -m gpu -x \
  -k "generator or randn or planted or regimes or c3_full or c4_keep" 2>&1 | tail -80
