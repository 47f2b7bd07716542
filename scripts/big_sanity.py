"""Sanity solve beyond the BASELINE sizes (exercises the 512-thread register
panel for > 8192-row panels): Gaussian LSE 12000 x 6000 / 1500 and GLS
10000 / 5000 / 7000, checked by their backward errors."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2406_16499_b200 as P
from tests.helpers import lse_backward, gls_backward

rng = np.random.default_rng(7)
m, n, p = 12000, 6000, 1500
A = rng.standard_normal((m, n)); B = rng.standard_normal((p, n)); b = rng.standard_normal(m); d = rng.standard_normal(p)
t0 = time.time()
res = P.mplse(P.LseProblem(A, B, b, d), P.RefinementConfig(maxit=10))
print("LSE", m, n, p, res.trace.status, res.trace.iterations, "%.1f ms" % (1e3 * (time.time() - t0)),
      "backward %.2e" % lse_backward(A, B, b, d, res.state.x, res.state.r, res.state.v), res.trace.timing)
n2, m2, p2 = 10000, 5000, 7000
W = rng.standard_normal((n2, m2)); V = rng.standard_normal((n2, p2)); d2 = rng.standard_normal(n2)
t0 = time.time()
r2 = P.mpgls(P.GlsProblem(W, V, d2), P.RefinementConfig(maxit=10))
print("GLS", n2, m2, p2, r2.trace.status, r2.trace.iterations, "%.1f ms" % (1e3 * (time.time() - t0)),
      "backward %.2e" % gls_backward(W, V, d2, r2.state.x, r2.state.y, r2.state.z), r2.trace.timing)
