"""Per-source-line totals (warp instructions executed, stall samples) from
`ncu --page source --csv --print-source cuda,sass`: SASS rows are attributed
to the source row above them."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
fn = None; hdr = None; cur = None
inst = collections.Counter(); samp = collections.Counter(); src = {}
for r in rows:
    if not r: continue
    if r[0] == "File Path": fn = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8: continue
    if r[2] == "-":
        cur = (fn, r[0]); src[cur] = r[1][:110]; continue
    try:
        s = int(r[4]); ie = int(r[7])
    except ValueError:
        continue
    inst[cur] += ie; samp[cur] += s
ti, ts = sum(inst.values()), sum(samp.values())
print(f"total warp-inst {ti}  samples {ts}")
by = sys.argv[2] if len(sys.argv) > 2 else "inst"
cnt = inst if by == "inst" else samp
for k, v in cnt.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 40):
    print(f"{100*inst[k]/ti:5.1f}% inst {100*samp[k]/max(ts,1):5.1f}% samp  {k[0]}:{k[1]}  {src.get(k,'')}")
