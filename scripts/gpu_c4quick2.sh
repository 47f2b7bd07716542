bash scripts/gpu_c4quick.sh
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_atsize.py -q -m gpu -x 2>&1 | tail -3
