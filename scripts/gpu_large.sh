timeout 1200 python -m pytest tests/test_gpu_large.py -q -m gpu -x -rf > gpurun_out/large.log 2>&1; echo rc=$?
grep -E "Error|error|assert|FAILED|passed|failed" gpurun_out/large.log | head -20
