python scripts/run_big.py --config C3 --reps 1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|panel_kernel" --launch-skip 40 -c 6 -o gpurun_out/prof_gemm python scripts/run_big.py --config C3 --reps 1 > gpurun_out/ncu_gemm.log 2>&1
echo rc=$?; tail -3 gpurun_out/ncu_gemm.log
