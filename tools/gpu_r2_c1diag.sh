#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/c1diag.log) 2>&1
DIAG_PLANS="8,16;4,37;16,8;8,18;4,32;2,74;16,9" timeout 900 python tools/c1_diag.py
