# C4 kernel A/B over (MLSB_REG_OPTS, MLSB_REG_OPTS2) pairs: device-resident bench line only
mkdir -p gpurun_out
for pr in ${PAIRS:-0:148 1:148 2:148 1:296 1:74}; do
  o=${pr%%:*}; o2=${pr##*:}
  MLSB_REG_OPTS=$o MLSB_REG_OPTS2=$o2 timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-records --no-cpu > gpurun_out/c4ab2.json 2> gpurun_out/c4ab2.err
  python - <<PY
import json
d = json.loads(open("gpurun_out/c4ab2.json").read().strip().splitlines()[-1])
print("opts $o opts2 $o2 value", round(d["value"]), "ms", round(d["ms_per_step"], 3), "iters", d["solves"]["iterations_mean"])
PY
done
