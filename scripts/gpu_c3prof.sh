python scripts/run_big.py --config C3 --reps 1 > gpurun_out/c3p_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python scripts/run_big.py --config C3 --reps 1 > gpurun_out/c3p_ncu.log 2>&1
echo rc=$?
tail -2 gpurun_out/c3p_ncu.log
