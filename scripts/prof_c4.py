"""Phase breakdown of the tile solver at the C4 shape + a small batched launch for ncu."""
import sys, time, json
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2406_16499_b200 as P
from paper_2406_16499_b200 import generate as G

A, B, b, d = G.lse_problem(256, 128, 32, 1e3, 1e1, 5)
for _ in range(3):
    r = P.mplse(P.LseProblem(A, B, b, d))
print("single C4-shape solve phases (s):", json.dumps(r.trace.timing), "iters", r.trace.iterations)
batch = int(sys.argv[1]) if len(sys.argv) > 1 else 1184
At, Bt, bt, dt, kA = G.lse_batch_torch(batch, 256, 128, 32, seed=1000)
torch.cuda.synchronize()
out = P.mplse_batched(At, Bt, bt, dt); torch.cuda.synchronize()
t0 = time.perf_counter()
out = P.mplse_batched(At, Bt, bt, dt); torch.cuda.synchronize()
print(f"batch {batch}: {1e3*(time.perf_counter()-t0):.2f} ms, iters mean {out.iterations.float().mean().item():.2f}")
