# quick iteration: parity tests of the tile kernels, phase stamps, C4 bench
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py -q -m gpu -rf -x > gpurun_out/tests.log 2>&1; echo tests_rc=$?
grep -E "Error|assert|FAILED|passed|failed" gpurun_out/tests.log | head -10
MLSB_DEBUG_STAMPS=1 timeout 300 python scripts/prof_c4.py 1184 2>&1 | grep -E "STAMPS|phases|batch" | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_c4.json').read().strip().splitlines()[-1])
print('value', round(d['value']), 'ms', round(d['ms_per_step'],2), 'e2e', round(d.get('e2e',{}).get('value',0)), 'iters', d['solves'], 'clk', d['clocks'])"
