mkdir -p gpurun_out
timeout 1500 python scripts/dbg/gls24.py > gpurun_out/gls24.log 2>&1
