"""One launch of each C3 trailing-update GEMM shape and one 8192-row panel, for
`ncu --set full` (scripts/gpu_profiles_c3.sh)."""
import ctypes as C, sys
sys.path.insert(0, ".")
import torch
from paper_2406_16499_b200._capi import lib
lib.mlsb_wy_gemm_f32.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, C.c_void_p, C.c_int64,
                                 C.c_void_p, C.c_int64, C.c_float, C.c_void_p, C.c_int64, C.c_void_p, C.c_size_t,
                                 C.c_void_p]
lib.mlsb_panel_f32.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_void_p,
                               C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
dev = torch.device("cuda")
work = torch.empty(128 * 9216 * 64, device=dev)
st = torch.cuda.current_stream().cuda_stream
cases = [(0, 0, 8192, 3968, 128, -1.0, 1.0), (1, 0, 128, 3968, 8192, 1.0, 0.0), (0, 0, 9088, 128, 4096, 1.0, 0.0),
         (0, 1, 9088, 4096, 128, -1.0, 1.0)]
for ta, tb, M, N, K, al, be in cases:
    ar, ac = (K, M) if ta else (M, K)
    br, bc = (N, K) if tb else (K, N)
    A = torch.randn(ac, ar, device=dev); B = torch.randn(bc, br, device=dev); Cm = torch.randn(N, M, device=dev)
    assert lib.mlsb_wy_gemm_f32(ta, tb, M, N, K, al, A.data_ptr(), ar, B.data_ptr(), br, be, Cm.data_ptr(), M,
                                work.data_ptr(), work.numel(), st) == 0
L = 8192
Mx = torch.randn(32, L, device=dev); V = torch.empty(32, L, device=dev)
tau = torch.empty(32, device=dev); T = torch.empty(32, 32, device=dev)
assert lib.mlsb_panel_f32(Mx.data_ptr(), L, 0, 0, L, 32, tau.data_ptr(), V.data_ptr(), L, T.data_ptr(), st) == 0
torch.cuda.synchronize()
print("ok")
