# Round profiles: C4 bench line + launch list + full capture; C3 large-path kernel captures.
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench_rc=$?
tail -1 gpurun_out/bench_c4.json | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"lse_reg_kernel|fma_burn" \
  --log-file gpurun_out/c4_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo launch_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lse_reg_kernel -s 1 -c 1 -f -o gpurun_out/prof_c4_full \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
# C3: the big trailing-update GEMMs (first launches of each orientation), residual, panel, WY apply
timeout 900 ncu --set full --clock-control none -k regex:"sgemm128|k_resid_stream|panel_reg_kernel|k_wy_upd|k_wy_dot|k_trsv_diag128" \
   -c 14 -f -o gpurun_out/prof_c3 python scripts/run_big.py --config C3 --reps 1 > gpurun_out/ncu_c3.log 2>&1; echo c3_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv \
  -k regex:"gemm|panel|tmerge|splitk|k_" python scripts/run_big.py --config C3 --reps 1 > gpurun_out/c3_ncu.log 2>&1; echo c3l_rc=$?
