#!/bin/bash
# C4 kernel: phase stamps (problem 0 in a full-occupancy batch) and one ncu --set full capture (with source) of a 8,880-problem launch
mkdir -p gpurun_out
MLSB_DEBUG_STAMPS=1 timeout 300 python scripts/prof_c4.py 1184 > gpurun_out/c4_stamps.log 2>&1; grep -E "STAMPS|batch" gpurun_out/c4_stamps.log | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lse_reg_kernel -s 3 -c 1 -o gpurun_out/c4_full \
   python scripts/prof_c4.py 8880 > gpurun_out/c4_ncu.log 2>&1; echo ncu_rc=$?
