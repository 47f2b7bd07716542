"""Per-phase cycle split of one register-panel reflector step (clock64 stamps
of CTA 0 / thread 0, mlsb_panel_probe_f32)."""
import ctypes as C, sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2406_16499_b200._capi import lib
lib.mlsb_panel_probe_f32.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_void_p]
dev = torch.device("cuda")
for L in [int(x) for x in sys.argv[1:]] or [8192, 4096]:
    Mx = torch.randn(32, L, device=dev)
    V = torch.empty(32, L, device=dev); tau = torch.empty(32, device=dev); T = torch.empty(32, 32, device=dev)
    pr = torch.zeros(32 * 8 + 8, dtype=torch.int64, device=dev)
    for _ in range(3):
        M2 = Mx.clone()
        assert lib.mlsb_panel_probe_f32(M2.data_ptr(), L, L, 32, tau.data_ptr(), V.data_ptr(), T.data_ptr(),
                                        pr.data_ptr(), torch.cuda.current_stream().cuda_stream) == 0
        torch.cuda.synchronize()
    allp = pr.cpu().numpy().astype(np.int64)
    kp = allp[256:261]
    print(f"L={L}: kernel stamps: load {kp[1]-kp[0]} cyc, steps {kp[2]-kp[1]} cyc, writeback {kp[3]-kp[2]} cyc, T {kp[4]-kp[3]} cyc")
    p = allp[:256].reshape(32, 8)
    names = ["partials+reduce", "sync1", "push", "wait", "coef", "sync2", "apply"]
    d = np.diff(p, axis=1)
    step = p[1:, 0] - p[:-1, 0]
    print(f"L={L}: step median {int(np.median(step))} cyc; " +
          ", ".join(f"{n} {int(np.median(d[1:, i]))}" for i, n in enumerate(names)))
