"""Time the binary32 WY GEMM at the four C3 trailing-update shapes (CUDA events)."""
import ctypes as C, sys
sys.path.insert(0, ".")
import torch
from paper_2406_16499_b200._capi import lib
lib.mlsb_wy_gemm_f32.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, C.c_void_p, C.c_int64,
                                 C.c_void_p, C.c_int64, C.c_float, C.c_void_p, C.c_int64, C.c_void_p, C.c_size_t,
                                 C.c_void_p]
lib.mlsb_fp32_fma_peak_tflops.restype = C.c_double
peak = lib.mlsb_fp32_fma_peak_tflops(-1, None)
dev = torch.device("cuda")
work = torch.empty(128 * 9216 * 64, device=dev)
st = torch.cuda.current_stream().cuda_stream
cases = [("qr C-=VW2 NN", 0, 0, 8192, 3968, 128, -1.0, 1.0), ("qr W=V^T C TN", 1, 0, 128, 3968, 8192, 1.0, 0.0),
         ("rq W=Ma V NN", 0, 0, 9088, 128, 4096, 1.0, 0.0), ("rq Ma-=W2 V^T NT", 0, 1, 9088, 4096, 128, -1.0, 1.0),
         ("square 4096^3", 0, 0, 4096, 4096, 4096, 1.0, 0.0)]
for name, ta, tb, M, N, K, al, be in cases:
    ar, ac = (K, M) if ta else (M, K)
    br, bc = (N, K) if tb else (K, N)
    A = torch.randn(ac, ar, device=dev); B = torch.randn(bc, br, device=dev); Cm = torch.randn(N, M, device=dev)
    f = lambda: lib.mlsb_wy_gemm_f32(ta, tb, M, N, K, al, A.data_ptr(), ar, B.data_ptr(), br, be, Cm.data_ptr(), M,
                                     work.data_ptr(), work.numel(), st)
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); [f() for _ in range(20)]; e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    tf = 2.0 * M * N * K / ms / 1e9
    print(f"{name:18s} {ms*1e3:8.1f} us  {tf:6.2f} TFLOP/s  frac {tf/peak:.3f}")
