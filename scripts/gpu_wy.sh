mkdir -p gpurun_out
timeout 300 python scripts/wy_bench.py > gpurun_out/wy_new.log 2>&1; echo new_rc=$?
cat gpurun_out/wy_new.log | tail -8
MLSB_GEMM_OLD=1 timeout 300 python scripts/wy_bench.py > gpurun_out/wy_old.log 2>&1; echo old_rc=$?
cat gpurun_out/wy_old.log | tail -8
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_gmres.py tests/test_gpu_direct.py -q -m gpu -x -rf > gpurun_out/tests_large.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/tests_large.log
timeout 600 python scripts/run_big.py --config C3 --reps 3 > gpurun_out/c3.json 2>&1; echo c3_rc=$?
tail -c 700 gpurun_out/c3.json
