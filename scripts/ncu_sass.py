"""ncu --page source --print-source cuda,sass CSV -> hottest SASS instructions with context."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
fn = None; cur = None; sass = []
for r in rows:
    if not r: continue
    if r[0] == "File Path": fn = r[1].split("/")[-1]; continue
    if r[0] in ("Function Name", "Line No"): continue
    if len(r) < 6: continue
    if r[2] == "-":
        cur = f"{fn}:{r[0]}"; continue
    try: addr = int(r[2], 16); s = int(r[4])
    except ValueError: continue
    sass.append((addr, r[3].strip(), s, cur))
sass.sort()
tot = sum(x[2] for x in sass)
idx = sorted(range(len(sass)), key=lambda i: -sass[i][2])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 4
print("total", tot, "instructions", len(sass))
for i in idx[:n]:
    a, ins, s, src = sass[i]
    print(f"=== {100*s/tot:.1f}%  {hex(a)} {ins}   [{src}]")
    for j in range(max(0, i - ctx), min(len(sass), i + 2)):
        print(f"     {'>' if j==i else ' '} {sass[j][2]:7d} {sass[j][1][:70]:70s} {sass[j][3]}")
