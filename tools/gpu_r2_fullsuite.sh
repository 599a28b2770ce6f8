#!/bin/bash
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/fullsuite.log) 2>&1
timeout 2400 python -m pytest tests -q -m gpu -rf --tb=short 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
