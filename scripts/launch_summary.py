"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) by kernel."""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if len(r) > 5 and r[0] == 'ID': hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    if d.get('Metric Name') != 'gpu__time_duration.sum': continue
    name = re.sub(r'\(.*', '', d['Kernel Name'])[:70]
    v = float(d['Metric Value'].replace(',', ''))
    u = d.get('Metric Unit', '')
    v *= {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0}.get(u, 1.0)
    agg[name][0] += 1; agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.2f} ms over {sum(v[0] for v in agg.values())} launches")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{v[1]:9.3f} ms {v[0]:6d}  {k}")
