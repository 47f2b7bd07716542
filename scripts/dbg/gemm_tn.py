import ctypes as C, sys
sys.path.insert(0, ".")
import torch
from paper_2406_16499_b200._capi import lib
lib.mlsb_wy_gemm_f32.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, C.c_void_p, C.c_int64,
                                 C.c_void_p, C.c_int64, C.c_float, C.c_void_p, C.c_int64, C.c_void_p, C.c_size_t,
                                 C.c_void_p]
dev = torch.device("cuda")
work = torch.empty(128 * 9216 * 64, device=dev)
st = torch.cuda.current_stream().cuda_stream
ta, tb, M, N, K = 1, 0, 128, 3968, 8192
A = torch.randn(M, K, device=dev); B = torch.randn(N, K, device=dev); Cm = torch.randn(N, M, device=dev)
for _ in range(3):
    lib.mlsb_wy_gemm_f32(ta, tb, M, N, K, 1.0, A.data_ptr(), K, B.data_ptr(), K, 0.0, Cm.data_ptr(), M, work.data_ptr(), work.numel(), st)
torch.cuda.synchronize()
