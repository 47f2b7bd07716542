timeout 900 python -m pytest tests/test_gpu_large.py -q -m gpu -x -rf > gpurun_out/large.log 2>&1; echo tests_rc=$?
grep -E "FAILED|passed|failed|Error" gpurun_out/large.log | head -5
python scripts/run_big.py --config C3 --reps 3 2>&1 | tail -1
python scripts/run_big.py --config C5 --reps 3 2>&1 | tail -1
python scripts/run_big.py --config C3 --reps 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python scripts/run_big.py --config C3 --reps 1 > /dev/null 2>&1; echo ncu_rc=$?
