"""binary64 direct solvers on the GPU (mlsb_lse_direct / mlsb_gls_direct)
against the oracle's restatement of detail::lse_direct_reference /
gls_direct_reference (inc/experiment.hpp:50-73).

Both sides are backward-stable binary64 solutions computed in different
orders, so the bar is the forward-error bound c N u kappa
on every output, plus the binary64 backward error at rounding level."""
import numpy as np
import pytest

from paper_2406_16499_b200 import generate as G

from .helpers import U53, fwd_bound, gls_backward, lse_backward, rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape,kappa", [((200, 100, 50), 1e3), ((20, 10, 4), 1e2),
                                         ((256, 128, 32), 1e5), ((64, 32, 32), 1e1),
                                         ((7, 5, 3), 1e2)])
def test_lse_direct_parity(gpu, port, shape, kappa):
    m, n, p = shape
    A, B, b, d = G.lse_problem(m, n, p, kappa, 1e2, seed=3 + m)
    st = gpu.lse_direct(gpu.LseProblem(A, B, b, d))
    x, r, v = port.lse_direct(A, B, b, d)
    kap = np.linalg.cond(np.vstack([A, B])) * 1e2
    bound = fwd_bound(m, n, p, kap)
    assert rel(st.x, x) <= bound, (rel(st.x, x), bound)
    assert rel(st.r, r) <= bound, (rel(st.r, r), bound)
    assert rel(st.v, v) <= bound, (rel(st.v, v), bound)
    assert lse_backward(A, B, b, d, st.x, st.r, st.v) <= 1e3 * (m + n + p) * U53


@pytest.mark.parametrize("shape,kappa", [((200, 100, 150), 1e4), ((12, 3, 11), 1e2),
                                         ((20, 10, 15), 1e3), ((24, 24, 4), 1e1)])
def test_gls_direct_parity(gpu, port, shape, kappa):
    n, m, p = shape
    W, V, d = G.gls_problem(n, m, p, kappa, 1e2, seed=5 + n)
    st = gpu.gls_direct(gpu.GlsProblem(W, V, d))
    x, y, z = port.gls_direct(W, V, d)
    kap = np.linalg.cond(np.hstack([W, V])) * 1e2
    bound = fwd_bound(n, m, p, kap)
    assert rel(st.x, x) <= bound, (rel(st.x, x), bound)
    assert rel(st.y, y) <= bound, (rel(st.y, y), bound)
    assert rel(st.z, z) <= bound, (rel(st.z, z), bound)
    assert gls_backward(W, V, d, st.x, st.y, st.z) <= 1e3 * (n + m + p) * U53


def test_lse_direct_matches_reference_build(gpu, ref):
    """Against the unmodified reference headers (oracle/_ref) when present."""
    A, B, b, d = G.lse_problem(200, 100, 50, 1e3, 1e2, 1)
    st = gpu.lse_direct(gpu.LseProblem(A, B, b, d))
    x, r, v = ref.lse_direct(A, B, b, d)
    assert rel(st.x, x) <= fwd_bound(200, 100, 50, 1e5)


def test_direct_singular_index(gpu, port):
    """A zero row of B gives the reference's singular_triangular index."""
    A, B, b, d = G.lse_problem(20, 10, 4, 1e2, 1e1, seed=9)
    B[2, :] = 0.0
    with pytest.raises(gpu.SingularTriangular) as ei:
        gpu.lse_direct(gpu.LseProblem(A, B, b, d))
    from oracle.oracle import OracleError

    with pytest.raises(OracleError) as eo:
        port.lse_direct(A, B, b, d)
    assert ei.value.index == eo.value.index


def test_direct_device_pointers(gpu):
    import torch

    A, B, b, d = G.lse_problem(200, 100, 50, 1e3, 1e2, 1)
    host = gpu.lse_direct(gpu.LseProblem(A, B, b, d))
    t = lambda a: torch.from_numpy(np.asfortranarray(a)).cuda() if a.ndim == 1 else \
        torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()  # noqa: E731
    dev = gpu.lse_direct(gpu.LseProblem(t(A), t(B), t(b), t(d)))
    torch.cuda.synchronize()
    assert np.array_equal(dev.x.cpu().numpy(), host.x)
