mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_large.py -q -m gpu -x > gpurun_out/tests_large.log 2>&1; tail -2 gpurun_out/tests_large.log
MLSB_FACT_PROF=1 timeout 600 python scripts/run_big.py --config C3 --reps 3 > gpurun_out/c3.json 2> gpurun_out/c3.err; echo c3_rc=$?
tail -c 900 gpurun_out/c3.json; grep -E "stage|total|panels|inner|merge|trail" gpurun_out/c3.err | tail -12
