"""The seeded BASELINE-spec generator (input preparation, not parity-critical)."""
import numpy as np
import pytest

from paper_2406_16499_b200 import generate as G


@pytest.mark.parametrize("cplx", [False, True])
def test_haar_orthonormal(cplx):
    rng = np.random.default_rng(0)
    Q = G.haar(rng, 40, 25, cplx)
    assert np.abs(Q.conj().T @ Q - np.eye(25)).max() < 1e-13


@pytest.mark.parametrize("shape,kappa", [((200, 100), 1e3), ((50, 100), 1e2), ((64, 64), 1e6)])
def test_svd_matrix_has_requested_spectrum(shape, kappa):
    rng = np.random.default_rng(1)
    X = G.svd_matrix(rng, *shape, kappa)
    s = np.linalg.svd(X, compute_uv=False)
    k = min(shape)
    assert np.allclose(s, kappa ** (-np.arange(k) / (k - 1)), rtol=1e-9)
    assert X.flags["F_CONTIGUOUS"]


def test_problems_are_seeded():
    a = G.lse_problem(20, 10, 4, 1e3, 1e2, 7)
    b = G.lse_problem(20, 10, 4, 1e3, 1e2, 7)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    W, V, d = G.gls_problem(12, 4, 10, 1e4, 1e2, 2)
    assert W.shape == (12, 4) and V.shape == (12, 4 + 6) and d.shape == (12,)


def test_batch_numpy_kappa_range():
    A, B, b, d, kA = G.lse_batch_numpy(6, 16, 8, 2, seed=1000)
    assert A.shape == (6, 16, 8) and B.shape == (6, 2, 8)
    assert np.all((kA >= 10.0) & (kA <= 1e5))
    for i in range(6):
        s = np.linalg.svd(A[i], compute_uv=False)
        assert s[0] / s[-1] == pytest.approx(kA[i], rel=1e-8)


def test_configs_match_baseline():
    c = G.CONFIGS
    assert (c["C1"]["m"], c["C1"]["n"], c["C1"]["p"]) == (200, 100, 50)
    assert (c["C2"]["n"], c["C2"]["m"], c["C2"]["p"]) == (200, 100, 150)
    assert (c["C3"]["m"], c["C3"]["n"], c["C3"]["p"]) == (8192, 4096, 1024)
    assert (c["C4"]["batch"], c["C4"]["m"], c["C4"]["n"], c["C4"]["p"]) == (65536, 256, 128, 32)
    assert (c["C5"]["n"], c["C5"]["m"], c["C5"]["p"]) == (4096, 2048, 3072)


def test_batch_torch_slices_are_the_same_problems():
    """Per-block seeds: any slice [start, start + count) of a batch regenerates
    bitwise the same problems as the whole batch (what the sharded bench and
    the reference arm rely on)."""
    import torch

    A, B, b, d, kA = G.lse_batch_torch(G.GEN_BLOCK + 300, 12, 6, 2, seed=11, device="cpu")
    for start, count in ((0, 5), (G.GEN_BLOCK - 7, 20), (500, G.GEN_BLOCK - 200)):
        A2, B2, b2, d2, k2 = G.lse_batch_torch(count, 12, 6, 2, seed=11, device="cpu", start=start)
        sl = slice(start, start + count)
        for full, part in ((A, A2), (B, B2), (b, b2), (d, d2), (kA, k2)):
            assert torch.equal(full[sl], part)
    assert A.stride() == (72, 1, 12)  # column-major per problem
    assert np.all((kA.numpy() >= 10.0) & (kA.numpy() <= 1e5))
    s = torch.linalg.svdvals(A[3])
    assert float(s[0] / s[-1]) == pytest.approx(float(kA[3]), rel=1e-8)
