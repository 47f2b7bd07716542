"""Time the large path's compact-WY trailing-update GEMM (mlsb_wy_gemm_f32) and
cluster panel (mlsb_panel_f32) at the C3 shapes, with CUDA events, and check the
GEMM against a float64 torch product.  MLSB_GEMM_OLD=1 selects the previous
tiles (A/B runs)."""
import ctypes as C, json, sys
sys.path.insert(0, ".")
import torch
from paper_2406_16499_b200._capi import lib

lib.mlsb_wy_gemm_f32.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, C.c_void_p, C.c_int64,
                                 C.c_void_p, C.c_int64, C.c_float, C.c_void_p, C.c_int64, C.c_void_p, C.c_size_t,
                                 C.c_void_p]
lib.mlsb_panel_f32.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_void_p,
                               C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
dev = torch.device("cuda")
peak = float(sys.argv[1]) if len(sys.argv) > 1 else 71.9
work = torch.empty(128 * 9216 * 64, device=dev, dtype=torch.float32)
st = torch.cuda.current_stream().cuda_stream


def colmajor(r, c, ld=None):
    ld = ld or r
    return torch.randn(c, ld, device=dev, dtype=torch.float32)  # storage: column j at [j, :]


def gemm_case(name, ta, tb, M, N, K, alpha, beta, reps=20):
    ar, ac = (K, M) if ta else (M, K)
    br, bc = (N, K) if tb else (K, N)
    A = colmajor(ar, ac); B = colmajor(br, bc); Cm = colmajor(M, N)
    C0 = Cm.clone()
    args = lambda: (ta, tb, M, N, K, alpha, A.data_ptr(), ar, B.data_ptr(), br, beta, Cm.data_ptr(), M,
                    work.data_ptr(), work.numel(), st)
    assert lib.mlsb_wy_gemm_f32(*args()) == 0
    torch.cuda.synchronize()
    Ad = A.double().t(); Bd = B.double().t()  # (rows, cols) views
    opA = Ad.t() if ta else Ad
    opB = Bd.t() if tb else Bd
    ref = alpha * (opA @ opB) + beta * C0.double().t()
    err = float((Cm.double().t() - ref).abs().max() / ref.abs().max())
    ev0, ev1 = torch.cuda.Event(True), torch.cuda.Event(True)
    for _ in range(3):
        lib.mlsb_wy_gemm_f32(*args())
    ev0.record()
    for _ in range(reps):
        lib.mlsb_wy_gemm_f32(*args())
    ev1.record(); torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / reps
    tf = 2.0 * M * N * K / ms / 1e9
    return dict(case=name, M=M, N=N, K=K, ms=round(ms, 4), tflops=round(tf, 2), frac=round(tf / peak, 3),
                rel_err=err)


out = []
out.append(gemm_case("qr C-=V*W2 (NN)", 0, 0, 8192, 3968, 128, -1.0, 1.0))
out.append(gemm_case("qr W=V^T*C (TN, split-K)", 1, 0, 128, 3968, 8192, 1.0, 0.0))
out.append(gemm_case("qr W2=T^T*W (TN)", 1, 0, 128, 3968, 128, 1.0, 0.0))
out.append(gemm_case("rq W=Ma*V (NN, split-K)", 0, 0, 9088, 128, 4096, 1.0, 0.0))
out.append(gemm_case("rq Ma-=W2*V^T (NT)", 0, 1, 9088, 4096, 128, -1.0, 1.0))
out.append(gemm_case("square 4096 NN", 0, 0, 4096, 4096, 4096, 1.0, 0.0, reps=5))
# panel: 32 reflectors of a 9216-row panel
L = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
Mx = torch.randn(32, L, device=dev)
V = torch.empty(32, L, device=dev); tau = torch.empty(32, device=dev); T = torch.empty(32, 32, device=dev)
def pan():
    M2 = Mx.clone()
    return M2, (M2.data_ptr(), L, 0, 0, L, 32, tau.data_ptr(), V.data_ptr(), L, T.data_ptr(), st)
M2, a = pan()
assert lib.mlsb_panel_f32(*a) == 0
torch.cuda.synchronize()
# check: R from torch QR (up to signs)
R = torch.linalg.qr(Mx.double().t(), mode="r")[1]
Rg = torch.triu(M2.double().t()[:32, :32])
prel = float((Rg.abs() - R.abs()).abs().max() / R.abs().max())
ev0, ev1 = torch.cuda.Event(True), torch.cuda.Event(True)
ts = []
for _ in range(10):
    M2, a = pan()
    ev0.record(); lib.mlsb_panel_f32(*a); ev1.record(); torch.cuda.synchronize()
    ts.append(ev0.elapsed_time(ev1))
out.append(dict(case=f"panel {L}x32", us=round(1e3 * min(ts), 1), us_per_reflector=round(1e3 * min(ts) / 32, 2),
                rel_err_R=prel))
for o in out:
    print(json.dumps(o))

# complex64 panel (C5's QR panels have 4096 rows)
lib.mlsb_panel_c64.argtypes = lib.mlsb_panel_f32.argtypes
Lc = 4096
Mc = torch.randn(32, Lc, 2, device=dev)
Vc = torch.empty(32, Lc, 2, device=dev); tc_ = torch.empty(32, 2, device=dev); Tc = torch.empty(32, 32, 2, device=dev)
ts = []
for _ in range(10):
    M2 = Mc.clone()
    ev0.record()
    assert lib.mlsb_panel_c64(M2.data_ptr(), Lc, 0, 0, Lc, 32, tc_.data_ptr(), Vc.data_ptr(), Lc, Tc.data_ptr(), st) == 0
    ev1.record(); torch.cuda.synchronize()
    ts.append(ev0.elapsed_time(ev1))
print(json.dumps(dict(case=f"complex panel {Lc}x32", us=round(1e3 * min(ts), 1), us_per_reflector=round(1e3 * min(ts) / 32, 2))))
