timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -rf > gpurun_out/tests.log 2>&1; echo tests_rc=$?
grep -E "Error|assert|FAILED|passed|failed" gpurun_out/tests.log | head -10
MLSB_DEBUG_STAMPS=1 python scripts/prof_c4.py 1184 2>&1 | grep -E "STAMPS|phases|batch" | tail -3
