"""Debug: per-block phase times of the persistent factor apply (last CTA) at C3."""
import ctypes as C, sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2406_16499_b200 as P
from paper_2406_16499_b200 import _capi, generate as G

m, n, p = 8192, 4096, 1024
A, B, b, d = G.lse_problem(m, n, p, 1e4, 1e2, 3)
buf = torch.zeros(512, dtype=torch.int64, device="cuda")
P.mplse(P.LseProblem(A, B, b, d))
_capi.lib.mlsb_debug_set_czstamps(C.c_void_p(buf.data_ptr()))
P.mplse(P.LseProblem(A, B, b, d))
torch.cuda.synchronize()
_capi.lib.mlsb_debug_set_czstamps(None)
st = buf.cpu().numpy().reshape(64, 8)
t0 = st[0, 0]
for s in range(64):
    if st[s, 0] == 0:
        continue
    r = st[s]
    print(f"step {s:2d}: start {1e-3*(r[0]-t0):8.2f} us  dot {1e-3*(r[6]-r[0]):6.2f} part+arrive {1e-3*(r[7]-r[6]):6.2f} pref {1e-3*(r[1]-r[7]):6.2f}  barrier {1e-3*(r[2]-r[1]):6.2f}  "
          f"ysum+T {1e-3*(r[3]-r[2]):6.2f}  z+upd {1e-3*(r[4]-r[3]):6.2f}  xs {1e-3*(r[5]-r[4]):6.2f}")
