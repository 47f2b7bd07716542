mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"trsv|wy_" -s 400 -c 60 python scripts/run_big.py --config C3 --reps 1 > gpurun_out/trsv_list.csv 2>/dev/null; echo rc=$?
python3 - <<'PY'
import csv, re, collections
rows = list(csv.reader(open('gpurun_out/trsv_list.csv')))
hdr = None; out = collections.defaultdict(list)
for r in rows:
    if len(r) > 5 and r[0] == 'ID': hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    out[re.sub(r'\(.*', '', d['Kernel Name'])].append(float(d['Metric Value'].replace(',', '')) / 1000)
for k, v in out.items():
    print(f"{k[:60]:60s} n={len(v):3d} mean={sum(v)/len(v):7.2f} us min={min(v):6.2f} max={max(v):6.2f}")
PY
