import sys, time, os; sys.path.insert(0, ".")
import torch, paper_2406_16499_b200 as P
from paper_2406_16499_b200 import generate as G
W, V, d = G.gls_problem(200, 100, 150, 1e4, 1e2, 2)
cfg = P.RefinementConfig(maxit=10)
for _ in range(3): r = P.mpgls(P.GlsProblem(W, V, d), cfg)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(10): r = P.mpgls(P.GlsProblem(W, V, d), cfg)
torch.cuda.synchronize(); print(os.environ.get("MLSB_FORCE_LARGE"), (time.perf_counter() - t0) / 10 * 1e3, "ms", r.trace.iterations, {k: round(v*1e3, 3) for k, v in r.trace.timing.items()})
