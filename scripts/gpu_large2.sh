mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_gmres.py tests/test_gpu_direct.py -q -m gpu -x -rf > gpurun_out/tests_large.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/tests_large.log
timeout 600 python scripts/run_big.py --config C3 --reps 3 > gpurun_out/c3.json 2>&1; echo c3_rc=$?
tail -c 700 gpurun_out/c3.json
timeout 600 python scripts/run_big.py --config C5 --reps 2 > gpurun_out/c5.json 2>&1; echo c5_rc=$?
tail -c 600 gpurun_out/c5.json
