cd /root/repo; mkdir -p gpurun_out
for c in C3 C2; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fused -s 3 -c 1 -o gpurun_out/prof_f4_$c -f \
  python bench.py --kv e4m3 --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fused -s 3 -c 1 -o gpurun_out/prof_bf16_C2 -f \
  python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
