#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fac_apply|k_trsv_chain" -s 6 -c 4 \
  -o gpurun_out/cz_prof python scripts/run_big.py --config C3 --reps 1 > gpurun_out/cz_prof.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/cz_prof.log
