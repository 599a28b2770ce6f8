cd /root/repo; exec > >(tee gpurun_out/run.log) 2>&1
q() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])"; }
for rep in 1 2; do for c in C3 C2 C1; do for v in base cur; do echo "$c $v"; SP_LIB_AB=build/ab/$v.so timeout 300 python bench.py --config $c --steps 10 --warmup 4 --no-e2e --no-cpu-baseline 2>&1 | q; done; done; done
