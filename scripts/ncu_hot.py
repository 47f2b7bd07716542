"""Aggregate ncu --page source (cuda,sass) CSV into hottest source lines by stall samples."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
fn = None; hdr = None; out = []
for r in rows:
    if not r: continue
    if r[0] == "File Path": fn = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 6: continue
    if r[2] != "-": continue  # sass rows
    try: s = int(r[4])
    except ValueError: continue
    out.append((s, fn, r[0], r[1][:110]))
tot = sum(o[0] for o in out)
out.sort(reverse=True)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print("total samples", tot)
for s, f, ln, src in out[:n]:
    print(f"{100*s/tot:5.1f}% {f}:{ln}  {src}")
