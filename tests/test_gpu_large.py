"""Parity of the whole-GPU large-problem path (blocked GRQ/GQR with cluster
panels + compact-WY GEMMs, host-driven IR) against the CPU oracle.  Shapes are
kept where the scalar oracle finishes in seconds; MLSB_FORCE_LARGE routes small
shapes through the large path too, so its edge cases are covered."""
import os

import numpy as np
import pytest

from paper_2406_16499_b200 import generate as G
from tests.helpers import check_parity, fwd_bound, gls_backward, lse_backward, rel

pytestmark = pytest.mark.gpu


@pytest.fixture
def force_large():
    os.environ["MLSB_FORCE_LARGE"] = "1"
    yield
    del os.environ["MLSB_FORCE_LARGE"]


def _cfg(P, us="low", maxit=40):
    return P.RefinementConfig(maxit=maxit, precisions=P.PrecisionConfig("low", us))


def _lse(P, port, A, B, b, d, kappa, us="low"):
    res = P.mplse(P.LseProblem(A, B, b, d), _cfg(P, us))
    ref = port.mplse(A, B, b, d, prec=("s", "s" if us == "low" else "d", "d"))
    m, n = A.shape
    p = B.shape[0]
    msgs = check_parity("lse", rel(res.state.x, ref.x), fwd_bound(m, n, p, kappa), res.trace.iterations,
                        ref.iterations, lse_backward(A, B, b, d, res.state.x, res.state.r, res.state.v),
                        lse_backward(A, B, b, d, ref.x, ref.r, ref.v), res.trace.status, ref.status)
    return res, ref, msgs


def _gls(P, port, W, V, d, kappa, us="low", cplx=False):
    res = P.mpgls(P.GlsProblem(W, V, d), _cfg(P, us))
    ref = port.mpgls(W, V, d, prec=("s", "s" if us == "low" else "d", "d"), cplx=cplx)
    n, m = W.shape
    p = V.shape[1]
    fwd = max(rel(res.state.x, ref.x), rel(res.state.y, ref.r))
    msgs = check_parity("gls", fwd, fwd_bound(m, n, p, kappa), res.trace.iterations, ref.iterations,
                        gls_backward(W, V, d, res.state.x, res.state.y, res.state.z),
                        gls_backward(W, V, d, ref.x, ref.r, ref.v), res.trace.status, ref.status)
    return res, ref, msgs


@pytest.mark.parametrize("shape", [(20, 10, 4), (70, 40, 33), (7, 5, 3), (100, 64, 64), (45, 45, 1)])
@pytest.mark.parametrize("us", ["low", "working"])
def test_lse_large_path_small_shapes(gpu, port, force_large, shape, us):
    m, n, p = shape
    A, B, b, d = G.lse_problem(m, n, p, 1e3, 1e2, seed=m + n + p)
    kappa = np.linalg.cond(np.vstack([A, B])) * 1e3
    res, ref, msgs = _lse(gpu, port, A, B, b, d, kappa, us)
    assert res.trace.status == ref.status
    assert not msgs, msgs


@pytest.mark.parametrize("shape", [(12, 3, 11), (40, 20, 30), (64, 33, 40), (24, 24, 4), (50, 10, 70)])
@pytest.mark.parametrize("us", ["low", "working"])
def test_gls_large_path_small_shapes(gpu, port, force_large, shape, us):
    n, m, p = shape
    W, V, d = G.gls_problem(n, m, p, 1e3, 1e2, seed=n + m + p)
    kappa = np.linalg.cond(np.hstack([W, V])) * 1e3
    res, ref, msgs = _gls(gpu, port, W, V, d, kappa, us)
    assert res.trace.status == ref.status
    assert not msgs, msgs


@pytest.mark.parametrize("shape", [(1024, 512, 128), (600, 400, 50)])
def test_lse_large_sizes(gpu, port, shape):
    m, n, p = shape
    A, B, b, d = G.lse_problem(m, n, p, 1e4, 1e2, seed=3)
    res, ref, msgs = _lse(gpu, port, A, B, b, d, 1e4 * 10)
    assert res.trace.status == ref.status == "converged"
    assert not msgs, msgs


def test_gls_large_size(gpu, port):
    W, V, d = G.gls_problem(512, 256, 384, 1e4, 1e2, seed=5)
    res, ref, msgs = _gls(gpu, port, W, V, d, 1e4 * 10)
    assert res.trace.status == ref.status == "converged"
    assert not msgs, msgs


# several outer WY blocks (NBO = 128 reflectors per trailing update) with a
# ragged last block and a ragged last panel, in both the RQ and the QR stage
@pytest.mark.parametrize("shape", [(700, 300, 200), (520, 270, 161), (400, 129, 33)])
def test_lse_outer_blocks(gpu, port, force_large, shape):
    m, n, p = shape
    A, B, b, d = G.lse_problem(m, n, p, 1e4, 1e2, seed=m + p)
    res, ref, msgs = _lse(gpu, port, A, B, b, d, 1e4 * 10)
    assert res.trace.status == ref.status == "converged"
    assert not msgs, msgs


@pytest.mark.parametrize("shape", [(600, 260, 400), (300, 140, 290)])
def test_gls_outer_blocks(gpu, port, force_large, shape):
    n, m, p = shape
    W, V, d = G.gls_problem(n, m, p, 1e4, 1e2, seed=n + p)
    res, ref, msgs = _gls(gpu, port, W, V, d, 1e4 * 10)
    assert res.trace.status == ref.status == "converged"
    assert not msgs, msgs


def test_complex_gls_outer_blocks(gpu, port):
    W, V, d = G.gls_problem(330, 150, 270, 1e3, 1e2, seed=33, cplx=True)
    res, ref, msgs = _gls(gpu, port, W, V, d, 1e3 * 10, cplx=True)
    assert res.trace.status == ref.status == "converged"
    assert not msgs, msgs


@pytest.mark.parametrize("shape", [(12, 4, 10), (64, 32, 48), (200, 100, 150)])
def test_complex_gls(gpu, port, shape):
    n, m, p = shape
    W, V, d = G.gls_problem(n, m, p, 1e3, 1e2, seed=n, cplx=True)
    kappa = np.linalg.cond(np.hstack([W, V])) * 1e3
    res, ref, msgs = _gls(gpu, port, W, V, d, kappa, cplx=True)
    assert res.trace.status == ref.status
    assert not msgs, msgs


def test_complex_lse(gpu, port):
    A, B, b, d = G.lse_problem(80, 40, 10, 1e3, 1e2, seed=9, cplx=True)
    res = gpu.mplse(gpu.LseProblem(A, B, b, d))
    ref = port.mplse(A, B, b, d, cplx=True)
    assert res.trace.status == ref.status == "converged"
    assert rel(res.state.x, ref.x) <= fwd_bound(80, 40, 10, 1e4)


def test_large_singular_and_zero_rhs(gpu, force_large):
    P = gpu
    W, V, d = G.gls_problem(7, 3, 6, 10.0, 10.0, 92)
    W[:, 1] = 0.0
    with pytest.raises(P.SingularTriangular):
        P.mpgls(P.GlsProblem(W, V, d))
    W, V, _ = G.gls_problem(8, 3, 7, 10.0, 10.0, 717)
    res = P.mpgls(P.GlsProblem(W, V, np.zeros(8)))
    assert res.trace.status == "converged" and res.trace.iterations == 1
    assert not np.any(res.state.x) and not np.any(res.state.y)


def test_large_determinism(gpu):
    P = gpu
    A, B, b, d = G.lse_problem(700, 400, 60, 1e3, 1e2, 11)
    r1 = P.mplse(P.LseProblem(A, B, b, d))
    r2 = P.mplse(P.LseProblem(A, B, b, d))
    assert np.array_equal(r1.state.x, r2.state.x)
    assert np.array_equal(r1.trace.residual_history, r2.trace.residual_history)


# u_r = extended (double-double residuals, lse.hpp:200-257 / gls.hpp:178-231) on the large path
def _cfg_ext(P, maxit=40):
    return P.RefinementConfig(maxit=maxit, precisions=P.PrecisionConfig("low", "low", "working",
                                                                        "extended"))


@pytest.mark.parametrize("shape", [(20, 10, 4), (70, 40, 33), (100, 64, 64)])
def test_lse_large_path_extended(gpu, port, force_large, shape):
    m, n, p = shape
    A, B, b, d = G.lse_problem(m, n, p, 1e4, 1e2, seed=m + 2 * n + p)
    res = gpu.mplse(gpu.LseProblem(A, B, b, d), _cfg_ext(gpu))
    ref = port.mplse(A, B, b, d, prec=("s", "s", "dd"))
    kappa = np.linalg.cond(np.vstack([A, B])) * 1e2
    msgs = check_parity("lse", rel(res.state.x, ref.x), fwd_bound(m, n, p, kappa),
                        res.trace.iterations, ref.iterations,
                        lse_backward(A, B, b, d, res.state.x, res.state.r, res.state.v),
                        lse_backward(A, B, b, d, ref.x, ref.r, ref.v), res.trace.status, ref.status)
    assert res.trace.status == ref.status
    assert not msgs, msgs


@pytest.mark.parametrize("shape", [(40, 20, 30), (64, 33, 40)])
def test_gls_large_path_extended(gpu, port, force_large, shape):
    n, m, p = shape
    W, V, d = G.gls_problem(n, m, p, 1e4, 1e2, seed=n + 2 * m + p)
    res = gpu.mpgls(gpu.GlsProblem(W, V, d), _cfg_ext(gpu))
    ref = port.mpgls(W, V, d, prec=("s", "s", "dd"))
    kappa = np.linalg.cond(np.hstack([W, V])) * 1e2
    fwd = max(rel(res.state.x, ref.x), rel(res.state.y, ref.r))
    msgs = check_parity("gls", fwd, fwd_bound(m, n, p, kappa), res.trace.iterations, ref.iterations,
                        gls_backward(W, V, d, res.state.x, res.state.y, res.state.z),
                        gls_backward(W, V, d, ref.x, ref.r, ref.v), res.trace.status, ref.status)
    assert res.trace.status == ref.status
    assert not msgs, msgs


def test_lse_large_size_extended(gpu, port):
    """A size the large path takes on its own, u_r = extended."""
    A, B, b, d = G.lse_problem(1024, 512, 128, 1e5, 1e2, seed=4)
    res = gpu.mplse(gpu.LseProblem(A, B, b, d), _cfg_ext(gpu))
    ref = port.mplse(A, B, b, d, prec=("s", "s", "dd"))
    assert res.trace.status == ref.status == "converged"
    assert abs(res.trace.iterations - ref.iterations) <= 1
    assert rel(res.state.x, ref.x) <= fwd_bound(1024, 512, 128, 1e5 * 10)


# u_f = working on the large path: binary64 panels and WY GEMMs, no pre-scaling
# (lse.hpp:315-318), correction without demotion (lse.hpp:399-411)
@pytest.mark.parametrize("shape", [(20, 10, 4), (70, 40, 33), (300, 170, 40)])
def test_lse_large_path_working_factor(gpu, port, force_large, shape):
    m, n, p = shape
    A, B, b, d = G.lse_problem(m, n, p, 1e6, 1e2, seed=m + 3 * n + p)
    cfg = gpu.RefinementConfig(maxit=10, precisions=gpu.PrecisionConfig("working", "working"))
    res = gpu.mplse(gpu.LseProblem(A, B, b, d), cfg)
    ref = port.mplse(A, B, b, d, maxit=10, prec=("d", "d", "d"))
    kappa = np.linalg.cond(np.vstack([A, B])) * 1e2
    msgs = check_parity("lse", rel(res.state.x, ref.x), fwd_bound(m, n, p, kappa), res.trace.iterations,
                        ref.iterations, lse_backward(A, B, b, d, res.state.x, res.state.r, res.state.v),
                        lse_backward(A, B, b, d, ref.x, ref.r, ref.v), res.trace.status, ref.status)
    assert res.trace.status == ref.status
    assert not msgs, msgs


@pytest.mark.parametrize("shape", [(40, 20, 30), (260, 120, 200)])
def test_gls_large_path_working_factor(gpu, port, force_large, shape):
    n, m, p = shape
    W, V, d = G.gls_problem(n, m, p, 1e6, 1e2, seed=n + 3 * m + p)
    cfg = gpu.RefinementConfig(maxit=10, precisions=gpu.PrecisionConfig("working", "working"))
    res = gpu.mpgls(gpu.GlsProblem(W, V, d), cfg)
    ref = port.mpgls(W, V, d, maxit=10, prec=("d", "d", "d"))
    kappa = np.linalg.cond(np.hstack([W, V])) * 1e2
    fwd = max(rel(res.state.x, ref.x), rel(res.state.y, ref.r))
    msgs = check_parity("gls", fwd, fwd_bound(m, n, p, kappa), res.trace.iterations, ref.iterations,
                        gls_backward(W, V, d, res.state.x, res.state.y, res.state.z),
                        gls_backward(W, V, d, ref.x, ref.r, ref.v), res.trace.status, ref.status)
    assert res.trace.status == ref.status
    assert not msgs, msgs


def test_lse_direct_large(gpu, port):
    """binary64 direct solve (lse_direct, lse.hpp:132-152) at a size beyond the tile solver."""
    A, B, b, d = G.lse_problem(1024, 512, 128, 1e4, 1e2, seed=21)
    st = gpu.lse_direct(gpu.LseProblem(A, B, b, d))
    xr, rr, vr = port.lse_direct(A, B, b, d)
    assert rel(st.x, xr) <= fwd_bound(1024, 512, 128, 1e4 * 10)
    assert rel(st.r, rr) <= fwd_bound(1024, 512, 128, 1e4 * 10)
