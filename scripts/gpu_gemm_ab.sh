mkdir -p gpurun_out
timeout 300 python scripts/wy_bench.py > gpurun_out/wy_new.log 2>&1; echo new_rc=$?
cat gpurun_out/wy_new.log | tail -12
