set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
free -g | head -2; nproc
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -rf 2>&1 | tail -30
timeout 600 python bench.py --steps 3 --warmup 2 --cpu-seconds 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo rc=$?
cat gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
timeout 300 python bench.py --config C1 --steps 20 --warmup 3
timeout 300 python bench.py --config C2 --steps 20 --warmup 3
