"""Input validation of the CUDA-tensor paths (the checks that keep bad input
away from out-of-bounds device reads): dtype, device, shapes, strides."""
import numpy as np
import pytest

from paper_2406_16499_b200 import generate as G

pytestmark = pytest.mark.gpu


def _dev(P):
    import torch

    A, B, b, d = G.lse_problem(30, 12, 4, 1e2, 1e1, 3)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t() if a.ndim == 2 else \
        torch.from_numpy(a).cuda()  # noqa: E731
    return (A, B, b, d), tuple(t(x) for x in (A, B, b, d))


def test_single_solve_rejects_wrong_dtype_and_shapes(gpu):
    import torch

    P = gpu
    _, (A, B, b, d) = _dev(P)
    with pytest.raises(P.InvalidInput):
        P.mplse(P.LseProblem(A.float(), B, b, d))
    with pytest.raises(P.InvalidInput):
        P.mplse(P.LseProblem(A, B, b.cpu(), d))
    with pytest.raises(P.DimensionError):
        P.mplse(P.LseProblem(A, B, b[:-1], d))
    with pytest.raises(P.DimensionError):
        P.mplse(P.LseProblem(A, B[:, :-1], b, d))
    W = torch.randn(20, 6, dtype=torch.float64, device="cuda")
    V = torch.randn(19, 9, dtype=torch.float64, device="cuda")
    with pytest.raises(P.DimensionError):
        P.mpgls(P.GlsProblem(W, V, torch.randn(20, dtype=torch.float64, device="cuda")))


def test_strided_rhs_is_accepted_and_equal(gpu):
    import torch

    P = gpu
    (An, Bn, bn, dn), (A, B, b, d) = _dev(P)
    host = P.mplse(P.LseProblem(An, Bn, bn, dn))
    b2 = torch.zeros(2 * b.numel(), dtype=torch.float64, device="cuda")[::2]
    b2.copy_(b)
    dev = P.mplse(P.LseProblem(A, B, b2, d))
    assert np.array_equal(dev.state.x.cpu().numpy(), host.state.x)


def test_batched_rejects_wrong_dtype_and_shapes(gpu):
    import torch

    P = gpu
    A, B, b, d, _ = G.lse_batch_torch(8, 20, 10, 4, seed=5, device="cuda")
    with pytest.raises(P.InvalidInput):
        P.mplse_batched(A.float(), B, b, d)
    with pytest.raises(P.DimensionError):
        P.mplse_batched(A, B, b[:, :-1], d)
    with pytest.raises(P.DimensionError):
        P.mplse_batched(A, B[:, :, :-1], b, d)
    out = P.mplse_batched(A, B, b, d, history=True)
    torch.cuda.synchronize()
    h = out.history.cpu().numpy()
    it = out.iterations.cpu().numpy()
    for i in range(8):  # rows past a problem's pass count are zero (defined output)
        assert not h[i, it[i]:].any()
