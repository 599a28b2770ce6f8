cd /root/repo; mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fused -s 6 -c 1 -o gpurun_out/prof_f4 -f \
  python bench.py --kv e4m3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-tune > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fused -s 6 -c 1 -o gpurun_out/prof_f3 -f \
  python bench.py --paged 16 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
ls -la gpurun_out/prof_f3.ncu-rep gpurun_out/prof_f4.ncu-rep
