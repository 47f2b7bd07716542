mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,smsp__cycles_active.avg --clock-control none --csv -k regex:"trsv|wy_" -s 200 -c 40 python scripts/run_big.py --config C3 --reps 1 > gpurun_out/trsv_list.csv 2>/dev/null; echo rc=$?
grep -E "trsv|wy_" gpurun_out/trsv_list.csv | awk -F'","' '{print $5, $(NF-2), $(NF)}' | sed 's/(.*)//' | head -60
