mkdir -p gpurun_out
MLSB_FACT_PROF=1 timeout 300 python scripts/run_big.py --config C3 --reps 2 2>&1 | grep "\[fact\]" | tail -1
timeout 1200 python -m pytest tests/test_gpu_large.py tests/test_gpu_gmres.py tests/test_gpu_direct.py -q -m gpu -rf > gpurun_out/tests_large.log 2>&1; echo tests_rc=$?
tail -8 gpurun_out/tests_large.log
timeout 600 python scripts/run_big.py --config C3 --reps 3 > gpurun_out/c3.json 2>&1; echo c3_rc=$?
tail -c 600 gpurun_out/c3.json
timeout 600 python scripts/run_big.py --config C5 --reps 2 > gpurun_out/c5.json 2>&1; echo c5_rc=$?
tail -c 500 gpurun_out/c5.json
timeout 300 python scripts/wy_bench.py 71.9 8192 > gpurun_out/wy_new.log 2>&1; cat gpurun_out/wy_new.log
