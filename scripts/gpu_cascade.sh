#!/bin/bash
# persistent cascade kernels: large-path GPU tests, then C3 / C5 timing (new vs MLSB_CASCADE_OLD)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_gmres.py tests/test_gpu_direct.py -x -q > gpurun_out/cz_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/cz_tests.log
for cfg in C3 C5; do
  MLSB_LOOP_PROF=1 timeout 300 python scripts/run_big.py --config $cfg --reps 2 > gpurun_out/cz_$cfg.json 2> gpurun_out/cz_$cfg.err; echo "$cfg rc=$?"
  MLSB_CASCADE_OLD=1 timeout 300 python scripts/run_big.py --config $cfg --reps 2 > gpurun_out/cz_${cfg}_old.json 2>/dev/null
done
