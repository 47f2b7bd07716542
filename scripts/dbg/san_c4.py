"""A few C4-shape problems through the register kernel (for compute-sanitizer)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2406_16499_b200 as P
from paper_2406_16499_b200 import generate as G

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
A, B, b, d, kA = G.lse_batch_torch(n, 256, 128, 32, seed=1000, device="cuda")
o = P.mplse_batched(A, B, b, d)
torch.cuda.synchronize()
print("iters", o.iterations.tolist()[:8], "err", o.errcode.tolist()[:8])
