timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -rf 2>&1 | tail -5
python scripts/prof_c4.py 1184
timeout 600 python bench.py --steps 3 --warmup 2 --cpu-seconds 3 --no-e2e > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo rc=$?
cat gpurun_out/bench3.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline_fp32']['achieved'], d['solves'])"; tail -3 gpurun_out/bench3.err
