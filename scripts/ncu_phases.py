"""C4 register kernel: stall samples and executed warp instructions by phase, from
`ncu --page source --csv --print-source cuda,sass`.  Each SASS row is classified by
its own (innermost inlined) source line: helper functions by line range, kernel-body
lines by region; rows of other files (device_common.cuh) take the class of the
previous row in address order.  usage: ncu_phases.py src.csv "lo-hi=name;..." """
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
ranges = []
for item in sys.argv[2].split(";"):
    rng, name = item.split("=")
    lo, hi = rng.split("-")
    ranges.append((int(lo), int(hi), name))
kfile = "tile_lse_reg.cu"
fn = None; cur = None; hdr = None; sass = []
for r in rows:
    if not r: continue
    if r[0] == "File Path": fn = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": hdr = r; continue
    if len(r) < 6: continue
    if r[2] == "-": cur = (fn, int(r[0]) if r[0].isdigit() else -1); continue
    try: addr = int(r[2], 16); s = int(r[4])
    except ValueError: continue
    st = {hdr[i]: int(r[i]) for i in range(32, 49) if r[i].isdigit() and int(r[i])}
    sass.append((addr, cur, s, st, int(r[7]) if r[7].isdigit() else 0, r[3]))
sass.sort()
samp = collections.Counter(); inst = collections.Counter(); stl = collections.defaultdict(collections.Counter)
ops = collections.defaultdict(collections.Counter)
last = "other"
for addr, (f, ln), s, st, ie, text in sass:
    if f == kfile:
        name = None
        for lo, hi, nm in ranges:
            if lo <= ln <= hi: name = nm
        if name: last = name
    samp[last] += s; inst[last] += ie; stl[last].update(st)
    op = text.split()[0] if text and not text.startswith("@") else (text.split()[1] if len(text.split()) > 1 else "?")
    ops[last][op.split(".")[0]] += ie
ts, ti = sum(samp.values()), sum(inst.values())
print(f"total samples {ts}, warp instructions {ti}")
for name, v in samp.most_common():
    top = ", ".join(f"{k.replace('stall_','')} {100*c/max(1,v):.0f}%" for k, c in stl[name].most_common(4))
    topo = ", ".join(f"{k} {100*c/max(1,inst[name]):.0f}%" for k, c in ops[name].most_common(6))
    print(f"{name:12s} {100*v/ts:5.1f}% samples {100*inst[name]/ti:5.1f}% inst | {top} | {topo}")
