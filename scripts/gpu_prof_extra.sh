# extra round-2 captures: the C3 cluster panel kernel and the C2 generic tile solver
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:"panel_reg_kernel" -s 2 -c 2 -f -o gpurun_out/r02_panel python scripts/wy_bench.py > gpurun_out/r02_panel.log 2>&1; echo panel_rc=$?
timeout 600 ncu --set full --clock-control none -k regex:"tile_solve_kernel" -s 2 -c 1 -f -o gpurun_out/r02_c2 python scripts/small_times.py > gpurun_out/r02_c2.log 2>&1; echo c2_rc=$?
for r in r02_panel r02_c2; do
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/$r.details.csv 2>/dev/null
  rm -f gpurun_out/$r.ncu-rep
done
