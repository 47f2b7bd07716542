"""Bitwise run-to-run reproducibility of the batched tile solvers (Appendix A.11)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2406_16499_b200 as P
from paper_2406_16499_b200 import generate as G


def check(name, run):
    o1, o2 = run(), run()
    bad = {f: int((getattr(o1, f).cpu().numpy() != getattr(o2, f).cpu().numpy()).reshape(len(o1.x), -1).any(1).sum())
           for f in ("x", "r", "v", "iterations", "status")}
    print(f"{name}: differing problems per field {bad}", flush=True)


for shape in ((256, 128, 32), (200, 100, 50), (20, 10, 4), (150, 90, 60)):
    A, B, b, d, _ = G.lse_batch_torch(2048, *shape, seed=1000, device="cuda")
    for cfg in (P.RefinementConfig(), P.RefinementConfig(precisions=P.PrecisionConfig("low", "working"))):
        check(f"LSE {shape} {cfg.precisions}", lambda: P.mplse_batched(A, B, b, d, cfg))
g = torch.Generator(device="cuda").manual_seed(5)
for (n, m, p) in ((200, 100, 150), (64, 32, 48), (40, 20, 30)):
    W = torch.randn(1024, m, n, dtype=torch.float64, device="cuda", generator=g).transpose(1, 2)
    V = torch.randn(1024, p, n, dtype=torch.float64, device="cuda", generator=g).transpose(1, 2)
    dd = torch.randn(1024, n, dtype=torch.float64, device="cuda", generator=g)
    check(f"GLS {(n, m, p)}", lambda: P.mpgls_batched(W, V, dd))
A, B, b, d, _ = G.lse_batch_torch(3000, 256, 128, 32, seed=1000, device="cuda")
full = P.mplse_batched(A, B, b, d).x.cpu().numpy()
sub = P.mplse_batched(A[1500:], B[1500:], b[1500:], d[1500:]).x.cpu().numpy()
print("C4 sub-batch equal:", np.array_equal(sub, full[1500:]))
h = P.mplse_batched(A.cpu().numpy(), B.cpu().numpy(), b.cpu().numpy(), d.cpu().numpy())
print("C4 host path equal:", np.array_equal(h.x, full))
