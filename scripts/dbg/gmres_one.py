import sys; sys.path.insert(0, ".")
import paper_2406_16499_b200 as P
from paper_2406_16499_b200 import generate as G
A, B, b, d = G.lse_problem(8192, 4096, 1024, 1e6, 1e2, 3)
r = P.gmres_refine_lse(P.LseProblem(A, B, b, d), P.RefinementConfig(maxit=40), precond="bd_split")
print(r.trace.iterations, r.trace.inner_iterations, r.trace.timing)
