#!/bin/bash
# Epilogue/teardown timeline (trace build) + ncu source-level stalls of the selection kernel alone.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/sel9.log) 2>&1
SP_LIB_AB=build/ab/seltrace.so SEL_GTIME=0 timeout 300 python tools/sel_trace.py
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_select -s 3 -c 1 -o gpurun_out/sel_alone -f python tools/sel_once.py > /dev/null 2>&1
python tools/ncu_stalls.py gpurun_out/sel_alone.ncu-rep select_body.cuh 45
ncu -i gpurun_out/sel_alone.ncu-rep --page details --csv 2>/dev/null | grep -i "Duration\|Registers Per\|Achieved Occupancy" | head
