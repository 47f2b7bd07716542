# C4 quick check: device-resident bench line with the full-batch parity leg (no e2e / records)
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-records > gpurun_out/c4q.json 2> gpurun_out/c4q.err; echo bench_rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/c4q.json").read().strip().splitlines()[-1])
p = d["parity"]["c4"]
print("value", round(d["value"]), "ms", round(d["ms_per_step"], 3), "iters", d["solves"]["iterations_mean"], "parity ok", p["ok"], p["iter_diff_hist"], p["max_fwd_over_bound"])
PY
MLSB_DEBUG_STAMPS=1 timeout 300 python scripts/prof_c4.py 1184 2>&1 | grep -E "STAMPS|batch" | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "batched or reg or c4 or C4" 2>&1 | tail -3
