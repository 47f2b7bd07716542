bash scripts/gpu_c4quick.sh
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "batched or unaligned or device" 2>&1 | tail -3
