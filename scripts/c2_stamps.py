import sys; sys.path.insert(0, '.')
import paper_2406_16499_b200 as P
from paper_2406_16499_b200 import generate as G
W, V, d = G.gls_problem(200, 100, 150, 1e4, 1e2, 2)
for _ in range(3):
    r = P.mpgls(P.GlsProblem(W, V, d), P.RefinementConfig(maxit=10))
print(r.trace.timing)
