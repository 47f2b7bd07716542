"""Debug: per-CTA timeline of the last persistent TRSV of a GMRES-IR solve (binary64 chain)."""
import ctypes as C, sys
sys.path.insert(0, ".")
import torch
import paper_2406_16499_b200 as P
from paper_2406_16499_b200 import _capi, generate as G
A, B, b, d = G.lse_problem(8192, 4096, 1024, 1e4, 1e2, 3)
buf = torch.zeros(512, dtype=torch.int64, device="cuda")
cfg = P.RefinementConfig(maxit=40)
P.gmres_refine_lse(P.LseProblem(A, B, b, d), cfg, precond="bd_split")
_capi.lib.mlsb_debug_set_czstamps(C.c_void_p(buf.data_ptr()))
P.gmres_refine_lse(P.LseProblem(A, B, b, d), cfg, precond="bd_split")
torch.cuda.synchronize()
_capi.lib.mlsb_debug_set_czstamps(None)
st = buf.cpu().numpy()
base = min(v for v in st[0:4 * 32:4] if v > 0)
for j in range(32):
    r = st[4 * j:4 * j + 4]
    lf = st[256 + 2 * j]
    if r[0] == 0:
        continue
    print(f"blk {j:2d}: ready {1e-3*(r[0]-base):8.2f} lastflag {1e-3*(lf-base) if lf else -1:8.2f} diag_start {1e-3*(r[1]-base):8.2f} loop {1e-3*(st[384+j]-r[1]):6.2f} diag {1e-3*(r[2]-r[1]):6.2f}")
