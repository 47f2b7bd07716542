MLSB_DEBUG_STAMPS=1 timeout 300 python scripts/prof_c4.py 1184 2>&1 | grep -E "STAMPS|phases|batch" | tail -3
MLSB_DEBUG_STAMPS=1 timeout 300 python scripts/prof_c4.py 148 2>&1 | grep -E "STAMPS|PROBE|batch" | tail -3
