#!/bin/bash
# A/B: the peer gather's partials per batch (16 vs 10), per-rank replays; peer parity tests.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/pb.log) 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seq.py -q -x -m gpu -k "peer or seq or dist" 2>&1 | tail -2
for lib in pb10 pb16 pb10 pb16; do echo "== $lib"; SP_LIB_AB=build/ab/$lib.so timeout 600 python tools/peer_replay.py C4 8 C3 8 2>&1 | tail -2; done
