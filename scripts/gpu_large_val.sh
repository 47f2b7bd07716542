mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_large.py tests/test_gpu_gmres.py tests/test_gpu_direct.py tests/test_gpu_atsize.py tests/test_gpu_dropin.py -q -m gpu -x 2>&1 | tail -3
