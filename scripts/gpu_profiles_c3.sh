mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:"sgemm128|panel_reg_kernel" -f -o gpurun_out/prof_c3_gemm python scripts/ncu_gemm_cases.py > gpurun_out/ncu_gemm.log 2>&1; echo gemm_rc=$?
timeout 900 ncu --set full --clock-control none -k regex:"k_resid_stream|k_wy_upd|k_wy_dot|k_trsv_diag128" -s 0 -c 4 -f -o gpurun_out/prof_c3_ir \
   python scripts/run_big.py --config C3 --reps 1 > gpurun_out/ncu_ir.log 2>&1; echo ir_rc=$?
