mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"trsv_diag128|k_wy_dot" -s 20 -c 2 -o gpurun_out/prof_trsv -f python scripts/run_big.py --config C3 --reps 1 > gpurun_out/ncu_trsv.log 2>&1; echo rc=$?
for k in trsv_diag128 k_wy_dot; do
ncu -i gpurun_out/prof_trsv.ncu-rep -k regex:$k --page source --csv --print-source cuda,sass > gpurun_out/src_$k.csv 2>/dev/null
python scripts/ncu_hot.py gpurun_out/src_$k.csv 14
done
ncu -i gpurun_out/prof_trsv.ncu-rep --page details --csv 2>/dev/null | grep -E '"Duration"|"Warp Cycles Per Issued|"Registers Per|"Achieved Occupancy"|Block Size|"Grid Size"' | cut -c1-200
