# 1) the driver's bench command (C4, N=1)
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench_rc=$?
tail -1 gpurun_out/bench_c4.json
# 2) launch list of the same workload (metrics-only pass)
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo launch_rc=$?
# 3) full capture of one tile-solver launch (traffic, stall reasons)
ncu --set full --clock-control none --import-source on -k regex:lse_reg_kernel -s 1 -c 1 -o gpurun_out/prof_c4_full \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
tail -2 gpurun_out/ncu_full.log
