# launch list of the bench workload: only this library's kernels are profiled
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lse_reg_kernel|tile_solve_kernel|fma_burn" \
    --csv --log-file gpurun_out/c4_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo launch_rc=$?
# one full capture of the tile solver at the bench config (traffic, stalls)
ncu --set full --clock-control none --import-source on -k regex:lse_reg_kernel -s 1 -c 1 -o gpurun_out/prof_c4_full \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
tail -2 gpurun_out/ncu_full.log
