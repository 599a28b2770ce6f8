#!/bin/bash
# A/B timing of build/ab/<name>.so variants: tools/gpu_ab.sh "name1 name2" "bench args 1" "bench args 2" ...
cd /root/repo; mkdir -p gpurun_out; exec > >(tee -a gpurun_out/ab.log) 2>&1
names=$1; shift
q() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('step %.4f ms  score %.4f ms  frac %.3f' % (d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac']))"; }
for rep in 1 2; do for a in "$@"; do for v in $names; do echo -n "$a | $v: "; SP_LIB_AB=build/ab/$v.so timeout 300 python bench.py $a --steps 10 --warmup 4 --no-e2e --no-cpu-baseline 2>/tmp/ab_err | q || tail -3 /tmp/ab_err; done; done; done
