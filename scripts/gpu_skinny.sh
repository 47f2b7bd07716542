#!/bin/bash
# A/B of the skinny inner-update kernels (MLSB_SKINNY_OLD=1 = three GEMMs)
mkdir -p gpurun_out
for v in old new old new; do
  if [ $v = old ]; then export MLSB_SKINNY_OLD=1; else unset MLSB_SKINNY_OLD; fi
  echo "== $v"; MLSB_FACT_PROF=1 timeout 300 python scripts/run_big.py --config C3 --reps 2 2>&1 | grep -E "fact|ms|C3" | tail -8
done
unset MLSB_SKINNY_OLD
for c in C5 C2; do echo "== $c"; timeout 300 python scripts/run_big.py --config $c --reps 2 2>&1 | tail -3; done
timeout 1500 python -m pytest tests/test_gpu_large.py tests/test_gpu_gmres.py tests/test_gpu_direct.py -m gpu -q -x 2>&1 | tail -5
