"""Time the single large BASELINE configs on the GPU (C3 LSE 8192x4096/1024,
C5 complex GLS 4096/2048/3072) and check them: C3 against the CPU reference
(oracle/_ref, ~100 s) when --oracle is given; every run against its backward
error and the paper's err-1/er-1 metrics (inc/metrics.hpp:23-56)."""
import argparse, json, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2406_16499_b200 as P
from paper_2406_16499_b200 import generate as G
from tests.helpers import gls_backward, lse_backward, rel

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--kappa", type=float, default=None)
ap.add_argument("--oracle", action="store_true")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--scale", type=int, default=1, help="divide the dimensions (quick checks)")
a = ap.parse_args()
c = dict(G.CONFIGS[a.config])
t0 = time.time()
out = {"config": a.config}
if a.config == "C3":
    m, n, p = c["m"] // a.scale, c["n"] // a.scale, c["p"] // a.scale
    kA = a.kappa or c["kappa_A"]
    A, B, b, d = G.lse_problem(m, n, p, kA, c["kappa_B"], c["seed"])
    out["gen_s"] = time.time() - t0
    cfg = P.RefinementConfig(maxit=c["maxit"])
    res = None
    ts = []
    for _ in range(a.reps):
        torch.cuda.synchronize(); t1 = time.perf_counter()
        res = P.mplse(P.LseProblem(A, B, b, d), cfg)
        ts.append(time.perf_counter() - t1)
    out.update(shape=[m, n, p], kappa_A=kA, status=res.trace.status, iterations=res.trace.iterations,
               wall_s=ts, phases=res.trace.timing,
               backward=lse_backward(A, B, b, d, res.state.x, res.state.r, res.state.v),
               err1=float(np.linalg.norm(B @ res.state.x - d) / (np.linalg.norm(B) * np.linalg.norm(res.state.x) + np.linalg.norm(d))))
    if a.oracle:
        from oracle.oracle import Oracle, available
        orc = Oracle("ref" if available("ref") else "port")
        t1 = time.time()
        ref = orc.mplse(A, B, b, d, maxit=c["maxit"])
        out.update(oracle_kind=orc.kind, oracle_s=time.time() - t1, oracle_status=ref.status,
                   oracle_iterations=ref.iterations, fwd=rel(res.state.x, ref.x),
                   fwd_bound=40 * (m + n + p + 1) * 2.0 ** -53 * kA,
                   oracle_backward=lse_backward(A, B, b, d, ref.x, ref.r, ref.v), oracle_phases=ref.phases.tolist())
else:
    n, m, p = c["n"] // a.scale, c["m"] // a.scale, c["p"] // a.scale
    W, V, d = G.gls_problem(n, m, p, c["kappa_A"], c["kappa_B"], c["seed"], cplx=True)
    out["gen_s"] = time.time() - t0
    cfg = P.RefinementConfig(maxit=c["maxit"])
    ts = []
    for _ in range(a.reps):
        torch.cuda.synchronize(); t1 = time.perf_counter()
        res = P.mpgls(P.GlsProblem(W, V, d), cfg)
        ts.append(time.perf_counter() - t1)
    er1 = np.linalg.norm(W @ res.state.x + V @ res.state.y - d) / (
        np.linalg.norm(W) * np.linalg.norm(res.state.x) + np.linalg.norm(V) * np.linalg.norm(res.state.y) + np.linalg.norm(d))
    out.update(shape=[n, m, p], status=res.trace.status, iterations=res.trace.iterations, wall_s=ts,
               phases=res.trace.timing, backward=gls_backward(W, V, d, res.state.x, res.state.y, res.state.z),
               er1=float(er1))
    if a.oracle:
        from oracle.oracle import Oracle
        orc = Oracle("port")
        t1 = time.time()
        ref = orc.mpgls(W, V, d, maxit=c["maxit"], cplx=True)
        out.update(oracle_kind="port(complex)", oracle_s=time.time() - t1, oracle_status=ref.status,
                   oracle_iterations=ref.iterations,
                   fwd=max(rel(res.state.x, ref.x), rel(res.state.y, ref.r)),
                   fwd_bound=40 * (m + n + p + 1) * 2.0 ** -53 * c["kappa_A"])
print(json.dumps(out))
