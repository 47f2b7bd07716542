"""Debug: run the C4 kernel twice on the same inputs and report which dumped
stage first differs per problem (mlsb_debug_set_dump)."""
import ctypes as C
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2406_16499_b200 as P
from paper_2406_16499_b200 import _capi, generate as G

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
A, B, b, d, kA = G.lse_batch_torch(n, 256, 128, 32, seed=1000, device="cuda")
lib = _capi.lib
stride = 160 * 1024
buf = torch.zeros(64 * stride, dtype=torch.float32, device="cuda")
lib.mlsb_debug_set_dump(C.c_void_p(buf.data_ptr()))
dumps, xs = [], []
for rep in range(3):
    buf.zero_()
    o = P.mplse_batched(A, B, b, d)
    torch.cuda.synchronize()
    dumps.append(buf.view(64, stride).cpu().numpy().copy())
    xs.append(o.x.cpu().numpy())
lib.mlsb_debug_set_dump(None)
ld, Cn = 289, 128
segs = [("M_after_RQ", 0, ld * Cn), ("tau2", 80000, 288), ("TQ_afterRQ", 80400, 1056),
        ("M_after_QR", 40000, ld * Cn), ("tau1", 84000, 128), ("TZ", 84200, 4 * 1056),
        ("TQ", 89000, 1056), ("su_init", 92000, 256), ("sw_init", 92400, 576),
        ("rout1", 93200, 576), ("cout1", 94000, 256)]
for r in (1, 2):
    print(f"--- run 0 vs run {r}: x differs in", int((xs[0] != xs[r]).any(1).sum()), "problems")
    for pi in range(64):
        first = None
        for name, off, ln in segs:
            a0, a1 = dumps[0][pi, off:off + ln], dumps[r][pi, off:off + ln]
            if not np.array_equal(a0.view(np.uint32), a1.view(np.uint32)):
                idx = np.flatnonzero(a0.view(np.uint32) != a1.view(np.uint32))
                first = (name, idx[:6].tolist(), len(idx))
                break
        if first:
            print(f"problem {pi}: first diff in {first[0]} at {first[1]} ({first[2]} words)")
            if first[0].startswith("M_"):
                i = first[1][0]
                print("   (row, col) =", (i % ld, i // ld), "vals", dumps[0][pi, segs[[s[0] for s in segs].index(first[0])][1] + i], dumps[r][pi, segs[[s[0] for s in segs].index(first[0])][1] + i])
