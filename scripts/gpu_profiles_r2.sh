#!/bin/bash
# Round-2 profiles: C4 launch list + one full capture of the bench launch;
# C3 launch list and full captures of the persistent cascade kernels, the
# residual and the trailing-update GEMMs.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-records"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"lse_reg_kernel|fma_burn" \
  --log-file gpurun_out/r02_c4_launches.csv $B > gpurun_out/r02_c4_launch.log 2>&1; echo c4_launch_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lse_reg_kernel -s 3 -c 1 -f -o gpurun_out/r02_c4_full \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-records > gpurun_out/r02_c4_full.log 2>&1; echo c4_full_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c3_launches.csv \
  python scripts/run_big.py --config C3 --reps 1 > gpurun_out/r02_c3_launch.log 2>&1; echo c3_launch_rc=$?
timeout 900 ncu --set full --clock-control none -k regex:"k_fac_apply|k_trsv_chain|k_resid_stream" -c 12 -f -o gpurun_out/r02_c3_cascade \
  python scripts/run_big.py --config C3 --reps 1 > gpurun_out/r02_c3_cascade.log 2>&1; echo c3_cascade_rc=$?
timeout 900 ncu --set full --clock-control none -k regex:"sgemm128" -c 5 -f -o gpurun_out/r02_gemm \
  python scripts/dbg/gemm_rate.py > gpurun_out/r02_gemm.log 2>&1; echo gemm_rc=$?
# summaries on the box (the reports themselves exceed gpurun's copy-back limit)
for r in r02_c4_full r02_c3_cascade r02_gemm; do
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/$r.details.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed.sum,sm__cycles_elapsed.avg > gpurun_out/$r.raw.csv 2>/dev/null
done
ncu -i gpurun_out/r02_c4_full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02_c4_source.csv 2>/dev/null
gzip -f gpurun_out/r02_c4_source.csv
rm -f gpurun_out/r02_c3_cascade.ncu-rep gpurun_out/r02_gemm.ncu-rep
du -sh gpurun_out
