#!/bin/bash
# A/B: scope of the local partial-statistics loads (gpu vs sys), same box.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/ld.log) 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "forced or peer or c1_full or c3_full" 2>&1 | tail -1
for lib in ldsys ldgpu ldsys ldgpu; do
  for c in C3 C1; do
    SP_LIB_AB=build/ab/$lib.so timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --no-read-peak 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$lib $c step %.4f kernel %.4f frac %.3f value %.2fM' % (d['ms_per_step'], r['kernel_ms'], r['frac'], d['value']/1e6))"
  done
  SP_LIB_AB=build/ab/$lib.so timeout 600 python tools/peer_replay.py C4 8 2>&1 | tail -1
done
