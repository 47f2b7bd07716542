mkdir -p gpurun_out
for v in 0 1 2; do
  echo "variant $v"
  MLSB_PANEL_256=$v timeout 300 python scripts/wy_bench.py 2>&1 | grep -E "panel 8192"
  MLSB_PANEL_256=$v timeout 600 python scripts/run_big.py --config C3 --reps 3 2>&1 | grep -o '"factorization": [0-9.]*'
done
