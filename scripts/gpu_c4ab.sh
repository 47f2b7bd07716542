# C4 kernel A/B over MLSB_REG_OPTS bits: device-resident bench line only, then the full-batch parity run of the default
mkdir -p gpurun_out
for o in ${OPTS_LIST:-0 1 2 4 5 6 7}; do
  MLSB_REG_OPTS=$o timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-records --no-cpu > gpurun_out/c4ab_$o.json 2> gpurun_out/c4ab_$o.err
  python - <<PY
import json
d = json.loads(open("gpurun_out/c4ab_$o.json").read().strip().splitlines()[-1])
print("opts $o value", round(d["value"]), "ms", round(d["ms_per_step"], 3), "iters", d["solves"]["iterations_mean"])
PY
done
bash scripts/gpu_c4quick.sh
