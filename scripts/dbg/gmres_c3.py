"""GMRES-IR at C3 shapes on the GPU (timing + iterations), optional reference at small scale."""
import sys, time, json
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2406_16499_b200 as P
from paper_2406_16499_b200 import generate as G
from tests.helpers import lse_backward

for kap in (1e4, 1e6):
    A, B, b, d = G.lse_problem(8192, 4096, 1024, kap, 1e2, 3)
    for pc in ("bd_split", "left"):
        cfg = P.RefinementConfig(maxit=40)
        r = P.gmres_refine_lse(P.LseProblem(A, B, b, d), cfg, precond=pc)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = P.gmres_refine_lse(P.LseProblem(A, B, b, d), cfg, precond=pc)
        dt = time.perf_counter() - t0
        print(json.dumps({"kappa": kap, "precond": pc, "status": r.trace.status, "outer": r.trace.iterations,
                          "inner": r.trace.inner_iterations, "wall_ms": dt * 1e3,
                          "phases_ms": {k: round(v * 1e3, 2) for k, v in r.trace.timing.items()},
                          "backward": lse_backward(A, B, b, d, r.state.x, r.state.r, r.state.v)}), flush=True)
