"""GMRES-IR for LSE on the GPU (mlsb_gmres_lse) against the unmodified
reference's gmres_refine_lse (inc/krylov.hpp:545-689, via oracle/_ref).

Parity bar as for classical IR: same status, outer passes
within 1, forward error within c N u kappa, backward error at the converged
level; the inner GMRES iteration count is reported and must be of the
reference's order (the preconditioned systems are applied in a different
summation order, so exact Krylov iteration counts can differ by a few)."""
import numpy as np
import pytest

from paper_2406_16499_b200 import generate as G

from .helpers import check_parity, fwd_bound, lse_backward, rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precond", ["bd_split", "left"])
@pytest.mark.parametrize("shape,kappa", [((200, 100, 50), 1e3), ((60, 40, 10), 1e6),
                                         ((120, 80, 30), 1e7), ((40, 40, 8), 1e2)])
def test_gmres_lse_parity(gpu, ref, precond, shape, kappa):
    m, n, p = shape
    A, B, b, d = G.lse_problem(m, n, p, kappa, 1e2, seed=21 + m + n)
    cfg = gpu.RefinementConfig(maxit=10)
    res = gpu.gmres_refine_lse(gpu.LseProblem(A, B, b, d), cfg, precond=precond)
    rr = ref.gmres_lse(A, B, b, d, maxit=10, precond=precond)
    kap = np.linalg.cond(np.vstack([A, B])) * 1e2
    msgs = check_parity("lse", rel(res.state.x, rr.x), fwd_bound(m, n, p, kap),
                        res.trace.iterations, rr.iterations,
                        lse_backward(A, B, b, d, res.state.x, res.state.r, res.state.v),
                        lse_backward(A, B, b, d, rr.x, rr.r, rr.v), res.trace.status, rr.status)
    assert res.trace.status == rr.status, (res.trace, rr.status)
    assert not msgs, msgs
    assert res.trace.inner_iterations >= 1
    assert res.trace.inner_iterations <= 2 * rr.inner + 10, (res.trace.inner_iterations, rr.inner)


def test_gmres_rescues_ill_conditioned(gpu, ref):
    """kappa(A) beyond u_f^-1: classical IR stagnates or diverges, GMRES-IR converges
    (PAPER §5)."""
    A, B, b, d = G.lse_problem(200, 100, 50, 1e9, 1e2, 3)
    cfg = gpu.RefinementConfig(maxit=20)
    res = gpu.gmres_refine_lse(gpu.LseProblem(A, B, b, d), cfg)
    rr = ref.gmres_lse(A, B, b, d, maxit=20)
    assert res.trace.status == rr.status
    if rr.status == "converged":
        assert abs(res.trace.iterations - rr.iterations) <= 1


def test_gmres_unsupported_shapes(gpu):
    A, B, b, d = G.lse_problem(20, 30, 15, 1e2, 1e1, 1)  # m < n
    with pytest.raises(gpu.Unsupported):
        gpu.gmres_refine_lse(gpu.LseProblem(A, B, b, d))
