"""profiles/c4_ncu_summary.json from one `ncu --set full` capture of the C4 bench launch:
details CSV (--page details), raw CSV (dram bytes, duration) and the source CSV
(--page source --print-source cuda,sass, gz) for the stall mix.  usage:
prof_summary.py <prefix> <problems> <out.json> [note]"""
import csv, gzip, json, sys, collections
pre, nprob, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
note = sys.argv[4] if len(sys.argv) > 4 else ""
det = {}
rows = list(csv.reader(open(pre + ".details.csv")))
hdr = rows[0]
for r in rows[1:]:
    if len(r) < 15: continue
    d = dict(zip(hdr, r))
    if "lse_reg_kernel" not in d["Kernel Name"]: continue
    det[(d["Section Name"], d["Metric Name"])] = (d["Metric Value"], d["Metric Unit"])
def g(sec, name, cast=float):
    v = det.get((sec, name))
    if v is None: return None
    try: return cast(v[0].replace(",", ""))
    except ValueError: return v[0]
raw = list(csv.reader(open(pre + ".raw.csv")))
rh = raw[0]; units = raw[1]; rv = raw[2]
rd = {h: (v, u) for h, v, u in zip(rh, rv, units)}
def scaled(key):
    v, u = rd[key]; v = float(v.replace(",", ""))
    return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1, "us": 1e-3, "s": 1e3, "cycle": 1}.get(u, 1)
dr, dw = scaled("dram__bytes_read.sum"), scaled("dram__bytes_write.sum")
res = {
    "source": note,
    "kernel": rd["Kernel Name"][0],
    "grid": rd["Grid Size"][0], "block": rd["Block Size"][0],
    "gpu_time_ms": scaled("gpu__time_duration.sum"),
    "dram_bytes_read": dr, "dram_bytes_write": dw, "dram_bytes_per_launch": dr + dw,
    "dram_bytes_per_problem": (dr + dw) / nprob,
    "lts_hit_rate_pct": g("Memory Workload Analysis", "L2 Hit Rate"),
    "issue_slots_busy_pct": g("Compute Workload Analysis", "Issue Slots Busy"),
    "ipc_active": g("Compute Workload Analysis", "Executed Ipc Active"),
    "registers_per_thread": g("Launch Statistics", "Registers Per Thread"),
    "eligible_warps_per_scheduler": g("Scheduler Statistics", "Eligible Warps Per Scheduler"),
    "executed_warp_instructions": g("Instruction Statistics", "Executed Instructions"),
    "warp_cycles_per_issued_instruction": g("Warp State Statistics", "Warp Cycles Per Issued Instruction"),
    "dynamic_smem_per_block_kb": g("Launch Statistics", "Dynamic Shared Memory Per Block"),
    "no_eligible_pct": g("Scheduler Statistics", "No Eligible"),
}
# stall mix and instruction count from the source view
try:
    f = gzip.open(pre.replace("_full", "_source") + ".csv.gz", "rt")
    st = collections.Counter(); inst = 0; hdr2 = None; seen = set()
    for r in csv.reader(f):
        if not r: continue
        if r[0] == "Line No": hdr2 = r; continue
        if hdr2 is None or len(r) < 49 or r[2] == "-": continue
        try: addr = int(r[2], 16)
        except ValueError: continue
        if addr in seen: continue
        seen.add(addr)
        if r[7].isdigit(): inst += int(r[7])
        for i in range(32, 49):
            if r[i].isdigit(): st[hdr2[i]] += int(r[i])
    tot = sum(st.values())
    res["warp_instructions_per_problem"] = inst / nprob
    res["stall_sample_share_pct"] = {k.replace("stall_", ""): round(100 * v / tot, 1) for k, v in st.most_common(10)}
except FileNotFoundError:
    pass
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
