"""Stall samples of the C4 kernel by phase: every SASS instruction is assigned to
the kernel-body source line at or before it in address order."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
bounds = [int(x) for x in sys.argv[2].split(",")]  # region start lines
names = sys.argv[3].split(",")
kfile = sys.argv[4] if len(sys.argv) > 4 else "tile_lse_reg.cu"
kstart = int(sys.argv[5]) if len(sys.argv) > 5 else 0
# optional helper ranges attributed to a kernel line: "lo-hi=line;..."
remap = []
if len(sys.argv) > 6:
    for item in sys.argv[6].split(";"):
        rng, ln = item.split("=")
        lo, hi = rng.split("-")
        remap.append((int(lo), int(hi), int(ln)))
fn = None; cur = None; sass = []; hdr = None
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
    sass.append((addr, cur, s, st, int(r[7]) if r[7].isdigit() else 0))
sass.sort()
reg = collections.Counter(); regst = collections.defaultdict(collections.Counter); regin = collections.Counter()
last = None
for addr, (f, ln), s, st, ie in sass:
    if f == kfile and ln >= kstart: last = ln
    elif f == kfile:
        for lo, hi, to in remap:
            if lo <= ln < hi: last = to
    if last is None: continue
    k = sum(1 for b in bounds if last >= b) - 1
    name = names[k] if k >= 0 else "pre"
    reg[name] += s; regin[name] += ie
    regst[name].update(st)
tot = sum(reg.values())
for name in names:
    if name not in reg: continue
    top = ", ".join(f"{k.replace('stall_','')} {100*v/max(1,reg[name]):.0f}%" for k, v in regst[name].most_common(4))
    print(f"{name:14s} {100*reg[name]/tot:5.1f}% samples  inst {regin[name]:>12d}   {top}")
