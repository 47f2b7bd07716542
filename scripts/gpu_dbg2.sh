mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_large.py -q -m gpu -x > gpurun_out/pytest_large.log 2>&1; tail -3 gpurun_out/pytest_large.log
bash scripts/gpu_c4quick.sh > gpurun_out/c4quick.log 2>&1; tail -6 gpurun_out/c4quick.log
bash scripts/gpu_c4prof.sh > gpurun_out/c4prof.log 2>&1; tail -3 gpurun_out/c4prof.log
