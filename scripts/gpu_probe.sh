mkdir -p gpurun_out
MLSB_DEBUG_STAMPS=1 timeout 300 python scripts/prof_c4.py 1184 2>&1 | grep -E "PROBE|j1=" | head -40
