timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -rf > gpurun_out/tests.log 2>&1; echo rc=$?
grep -E "Error|assert|FAILED|passed|failed" gpurun_out/tests.log | head -20
