"""Debug: small GLS/LSE shapes through the large path with a poisoned arena (MLSB_POISON),
bisecting which arena buffer is read before it is written (MLSB_POISON_ZERO=i)."""
import os, subprocess, sys
CHILD = r'''
import os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2406_16499_b200 as P
from paper_2406_16499_b200 import generate as G
from oracle.oracle import Oracle
port = Oracle("port")
which = sys.argv[1]
shapes = [(12, 3, 11), (40, 20, 30), (64, 33, 40), (24, 24, 4), (50, 10, 70)] if which == "gls" else [(20, 10, 4), (70, 40, 33), (7, 5, 3), (100, 64, 64), (45, 45, 1)]
for us in ("low", "working"):
  for shape in shapes:
    cfg = P.RefinementConfig(maxit=40, precisions=P.PrecisionConfig("low", us))
    if which == "gls":
        n, m, p = shape
        W, V, d = G.gls_problem(n, m, p, 1e3, 1e2, seed=n + m + p)
        ref = port.mpgls(W, V, d, prec=("s", "s" if us == "low" else "d", "d"))
        res = P.mpgls(P.GlsProblem(W, V, d), cfg)
    else:
        m, n, p = shape
        A, B, b, d = G.lse_problem(m, n, p, 1e3, 1e2, seed=m + n + p)
        ref = port.mplse(A, B, b, d, prec=("s", "s" if us == "low" else "d", "d"))
        res = P.mplse(P.LseProblem(A, B, b, d), cfg)
    err = float(np.linalg.norm(res.state.x - ref.x) / np.linalg.norm(ref.x))
    print(which, us, shape, "ref", ref.iterations, ref.status, "gpu", res.trace.iterations, res.trace.status, "%.2e" % err, flush=True)
'''
def run(env, which):
    e = dict(os.environ); e.update(env); e["MLSB_FORCE_LARGE"] = "1"
    r = subprocess.run([sys.executable, "-c", CHILD, which], env=e, capture_output=True, text=True)
    return r.stdout + r.stderr[-2000:]
for which in ("gls", "lse"):
    base = run({}, which)
    print("== plain", which); print(base, flush=True)
    pois = run({"MLSB_POISON": "1"}, which)
    print("== poison", which); print(pois, flush=True)
    if pois != base:
        for i in range(0, 70):
            z = run({"MLSB_POISON": "1", "MLSB_POISON_ZERO": str(i)}, which)
            if z != pois:
                print("== poison, take", i, "zeroed:", which); print(z, flush=True)
