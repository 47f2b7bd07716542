import sys; sys.path.insert(0, ".")
import paper_2406_16499_b200 as P
from paper_2406_16499_b200 import generate as G
A, B, b, d = G.lse_problem(8192, 4096, 1024, 1e4, 1e2, 3)
cfg = P.RefinementConfig(maxit=40, precisions=P.PrecisionConfig("low", "working"))
for _ in range(2):
    r = P.mplse(P.LseProblem(A, B, b, d), cfg)
print(r.trace.iterations, r.trace.timing)
