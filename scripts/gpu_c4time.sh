#!/bin/bash
# C4 device time only (no e2e / cpu / records), per MLSB_REG_OPTS variant
for o in ${OPTS:-0 1}; do for i in 1 2; do MLSB_REG_OPTS=$o python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-records 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('opts=$o', round(d['value']), round(d['ms_per_step'],2), round(d['solves']['iterations_mean'],4))"; done; done
