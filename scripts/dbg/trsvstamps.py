"""Debug: per-CTA timeline of the persistent TRSV (T11 solve at C3, the last trsv launch of a solve)."""
import ctypes as C, sys, os
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2406_16499_b200 as P
from paper_2406_16499_b200 import _capi, generate as G

m, n, p = 8192, 4096, 1024
A, B, b, d = G.lse_problem(m, n, p, 1e4, 1e2, 3)
buf = torch.zeros(512, dtype=torch.int64, device="cuda")
P.mplse(P.LseProblem(A, B, b, d))
_capi.lib.mlsb_debug_set_czstamps(C.c_void_p(buf.data_ptr()))
os.environ["MLSB_STOP_AFTER"] = "1"
P.mplse(P.LseProblem(A, B, b, d))
torch.cuda.synchronize()
_capi.lib.mlsb_debug_set_czstamps(None)
st = buf.cpu().numpy()
base = st[0:4 * 32:4][st[0:4 * 32:4] > 0].min()
for j in range(32):
    r = st[4 * j:4 * j + 4]
    if r[0] == 0:
        continue
    lf = st[256 + 2 * j]
    print(f"blk {j:2d}: ready {1e-3*(r[0]-base):7.2f}  lastflag {1e-3*(lf-base) if lf else -1:7.2f}  diag_start {1e-3*(r[1]-base):7.2f}  diag {1e-3*(r[2]-r[1]):5.2f}  publish {1e-3*(r[3]-base):7.2f}")
