mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv \
  -k regex:"gemm|panel|tmerge|splitk|k_" python scripts/run_big.py --config C3 --reps 1 > gpurun_out/c3_ncu.log 2>&1; echo c3l_rc=$?
python scripts/launch_summary.py gpurun_out/c3_launches.csv 30
