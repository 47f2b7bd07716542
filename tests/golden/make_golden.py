"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref, the
unmodified reference headers compiled by oracle/Makefile).  Run in the build
container where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

Each fixture stores the inputs (from the reference's own seeded generator,
inc/generate.hpp) and the reference outputs x/r/v (LSE) or x/y/z (GLS),
status, iterations and the unscaled residual history, for every precision
combination.  tests/test_oracle.py checks the restatement (oracle/port)
against these bit for bit, so the pin survives on boxes without the
reference tree.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Oracle  # noqa: E402

PRECS = [("s", "s", "d"), ("s", "d", "d"), ("d", "d", "d"), ("s", "s", "dd"), ("d", "d", "dd")]
LSE_CASES = [  # (m, n, p, cond, seed)
    (20, 10, 4, 1e2, 300), (18, 9, 3, 1e3, 505), (6, 4, 2, 1e1, 1), (40, 25, 5, 1e4, 7),
    (30, 12, 4, 1e9, 606), (200, 100, 50, 1e3, 1),
]
GLS_CASES = [  # (n, m, p, cond, seed)
    (14, 4, 12, 1e2, 300), (12, 3, 11, 1e2, 404), (8, 3, 7, 1e1, 717), (20, 10, 15, 1e4, 9),
    (200, 100, 150, 1e4, 2),
]


def main():
    ref = Oracle("ref")
    out = {}
    for (m, n, p, c, s) in LSE_CASES:
        A, B, b, d = ref.gen_lse(m, n, p, c, s)
        key = f"lse_{m}_{n}_{p}_{c:g}_{s}"
        rec = dict(A=A, B=B, b=b, d=d)
        for pr in PRECS:
            r = ref.mplse(A, B, b, d, prec=pr)
            tag = "".join(pr)
            rec.update({f"{tag}_x": r.x, f"{tag}_r": r.r, f"{tag}_v": r.v,
                        f"{tag}_status": r.status, f"{tag}_iters": r.iterations,
                        f"{tag}_hist": r.history})
        out[key] = rec
    for (n, m, p, c, s) in GLS_CASES:
        W, V, d = ref.gen_gls(n, m, p, c, s)
        key = f"gls_{n}_{m}_{p}_{c:g}_{s}"
        rec = dict(W=W, V=V, d=d)
        for pr in PRECS[:4]:
            r = ref.mpgls(W, V, d, prec=pr)
            tag = "".join(pr)
            rec.update({f"{tag}_x": r.x, f"{tag}_y": r.r, f"{tag}_z": r.v,
                        f"{tag}_status": r.status, f"{tag}_iters": r.iterations,
                        f"{tag}_hist": r.history})
        out[key] = rec
    for key, rec in out.items():
        np.savez_compressed(os.path.join(HERE, key + ".npz"), **rec)
    print(f"wrote {len(out)} fixtures to {HERE}")


if __name__ == "__main__":
    main()
