#!/bin/bash
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck synccheck memcheck; do
  timeout 900 $CS --tool $tool --kernel-name regex:lse_reg_kernel --print-limit 50 python scripts/dbg/san_c4.py 2 > gpurun_out/san_c4_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/san_c4_$tool.log
done
