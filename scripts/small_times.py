"""Wall time per solve (host arrays, C ABI incl. staging) and device phase split
for the single small configs C1 (LSE, tile LSE kernel) and C2 (GLS, generic
tile solver).  Usage: python scripts/small_times.py [--reps 30]"""
import argparse, json, sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2406_16499_b200 as P
from paper_2406_16499_b200 import generate as G

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=30)
a = ap.parse_args()
out = {}
for name in ("C1", "C2"):
    c = G.CONFIGS[name]
    f, s, r = c["prec"]
    cfg = P.RefinementConfig(maxit=c["maxit"], precisions=P.PrecisionConfig(factor=f, solve=s, residual=r))
    if c["kind"] == "lse":
        A, B, b, d = G.lse_problem(c["m"], c["n"], c["p"], c["kappa_A"], c["kappa_B"], c["seed"])
        run = lambda: P.mplse(P.LseProblem(A, B, b, d), cfg)
    else:
        W, V, d = G.gls_problem(c["n"], c["m"], c["p"], c["kappa_A"], c["kappa_B"], c["seed"])
        run = lambda: P.mpgls(P.GlsProblem(W, V, d), cfg)
    for _ in range(3):
        res = run()
    ts = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        res = run()
        ts.append(time.perf_counter() - t0)
    out[name] = dict(wall_ms_median=1e3 * float(np.median(ts)), wall_ms_min=1e3 * min(ts),
                     iterations=res.trace.iterations, status=res.trace.status,
                     device_ms={k: 1e3 * v for k, v in res.trace.timing.items()})
print(json.dumps(out))
