MLSB_DEBUG_STAMPS=1 python scripts/prof_c4.py 148 2>&1 | grep -E "STAMPS|PROBE|batch" | tail -8
