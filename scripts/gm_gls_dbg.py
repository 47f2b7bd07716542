import sys; sys.path.insert(0, '.')
import numpy as np
import paper_2406_16499_b200 as P
from paper_2406_16499_b200 import generate as G
from oracle.oracle import Oracle
ref = Oracle('ref')
for shape, kappa, pc in [((40, 40, 40), 1e2, 'bd_split'), ((40, 40, 60), 1e2, 'bd_split'), ((40, 40, 30), 1e2, 'bd_split'), ((40, 39, 40), 1e2, 'bd_split')]:
    n, m, p = shape
    W, V, d = G.gls_problem(n, m, p, kappa, 1e2, seed=7 + n + p)
    res = P.gmres_refine_gls(P.GlsProblem(W, V, d), P.RefinementConfig(maxit=10), precond=pc)
    rr = ref.gmres_gls(W, V, d, maxit=10, precond=pc)
    print(shape, pc, 'gpu', res.trace.status, res.trace.iterations, res.trace.inner_iterations, 'ref', rr.status, rr.iterations, rr.inner,
          '|x-xr| %.2e |xr| %.2e |y| %.2e |yr| %.2e |z| %.2e |zr| %.2e' % (np.linalg.norm(res.state.x - rr.x), np.linalg.norm(rr.x), np.linalg.norm(res.state.y), np.linalg.norm(rr.r), np.linalg.norm(res.state.z), np.linalg.norm(rr.v)))
    print('  hist gpu', np.array(res.trace.residual_history)[:3].tolist())
    print('  hist ref', rr.history[:3].tolist())
