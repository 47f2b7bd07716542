"""Seeded synthetic inputs to the BASELINE.json spec.

Each matrix is X = U diag(sigma) V^H with Haar U, V (Q of the QR of an i.i.d.
Gaussian matrix times diag(sign(diag R)) -- phase of diag R for complex) and
sigma_i = kappa^(-i/(k-1)), k = min(rows, cols), so kappa(X) = kappa exactly.
Right-hand sides are N(0,1) (real and imaginary parts N(0,1) for complex).

This stands in for the paper's DLATM1-based generator; it is input
preparation, not part of the measured or parity-checked path: both the GPU
and the CPU oracle receive the identical arrays.
"""
from __future__ import annotations

import numpy as np

__all__ = ["haar", "svd_matrix", "lse_problem", "gls_problem", "lse_batch_torch", "lse_batch_numpy",
           "block_seed", "GEN_BLOCK", "CONFIGS"]


def haar(rng: np.random.Generator, rows: int, cols: int, cplx: bool = False) -> np.ndarray:
    """rows x cols (rows >= cols) with Haar-distributed orthonormal columns."""
    if cplx:
        G = (rng.standard_normal((rows, cols)) + 1j * rng.standard_normal((rows, cols))) / np.sqrt(2)
    else:
        G = rng.standard_normal((rows, cols))
    Q, R = np.linalg.qr(G)
    dg = np.diag(R)
    ph = dg / np.abs(dg) if cplx else np.sign(dg)
    ph[dg == 0] = 1
    return Q * ph[None, :]


def sigma_profile(k: int, kappa: float) -> np.ndarray:
    if k == 1:
        return np.ones(1)
    return kappa ** (-np.arange(k) / (k - 1))


def svd_matrix(rng, rows: int, cols: int, kappa: float, cplx: bool = False) -> np.ndarray:
    k = min(rows, cols)
    U = haar(rng, rows, k, cplx)
    V = haar(rng, cols, k, cplx)
    X = (U * sigma_profile(k, kappa)[None, :]) @ V.conj().T
    return np.asfortranarray(X)


def _rhs(rng, n, cplx):
    if cplx:
        return rng.standard_normal(n) + 1j * rng.standard_normal(n)
    return rng.standard_normal(n)


def lse_problem(m, n, p, kappa_A, kappa_B, seed, cplx=False):
    """min ||Ax - b|| s.t. Bx = d; A m x n, B p x n."""
    rng = np.random.default_rng(seed)
    A = svd_matrix(rng, m, n, kappa_A, cplx)
    B = svd_matrix(rng, p, n, kappa_B, cplx)
    return A, B, _rhs(rng, m, cplx), _rhs(rng, p, cplx)


def gls_problem(n, m, p, kappa_A, kappa_B, seed, cplx=False):
    """min ||y|| s.t. W x + V y = d; W n x m, V n x p."""
    rng = np.random.default_rng(seed)
    W = svd_matrix(rng, n, m, kappa_A, cplx)
    V = svd_matrix(rng, n, p, kappa_B, cplx)
    return W, V, _rhs(rng, n, cplx)


GEN_BLOCK = 1024  # problems per generator block (lse_batch_torch)


def block_seed(seed: int, block: int) -> int:
    """Seed of generator block `block` (problems block*GEN_BLOCK ...) of a batch
    with base seed `seed`: any slice of the batch can be regenerated on its own."""
    return seed * 1_000_003 + block


def lse_batch_torch(batch, m, n, p, log10_kappa_range=(1.0, 5.0), kappa_B=10.0, seed=1000,
                    device="cuda", start=0):
    """Batched BASELINE config 4: per problem kappa(A) = 10^U(1,5), kappa(B) = 10.
    Returns problems [start, start + batch) of the batch with base seed `seed`:
    A (batch, m, n), B (batch, p, n) column-major per problem, b (batch, m),
    d (batch, p), kappa_A (batch,).

    The batch is cut into fixed blocks of GEN_BLOCK problems; block j draws
    everything from its own generator (block_seed(seed, j)) with the same call
    shapes whatever the slice, so a slice is bitwise the same problems as in
    the whole batch on the same device type.  That is what lets a rank of the
    sharded bench generate only its shard, and the reference arm regenerate
    the GPU arm's first problems (SURVEY.md §8(e) seed rule, per block rather
    than per problem)."""
    import torch

    f64 = torch.float64
    A = torch.empty((batch, n, m), dtype=f64, device=device).transpose(1, 2)
    B = torch.empty((batch, n, p), dtype=f64, device=device).transpose(1, 2)
    b = torch.empty((batch, m), dtype=f64, device=device)
    d = torch.empty((batch, p), dtype=f64, device=device)
    kA = torch.empty(batch, dtype=f64, device=device)
    lo, hi = log10_kappa_range
    nb = GEN_BLOCK

    def haar_t(g, rows, cols):
        G = torch.randn((nb, rows, cols), generator=g, device=device, dtype=f64)
        Q, R = torch.linalg.qr(G)
        s = torch.sign(torch.diagonal(R, dim1=-2, dim2=-1))
        s[s == 0] = 1
        return Q * s[:, None, :]

    def sig(k, kap):
        if k == 1:
            return torch.ones((kap.shape[0], 1), dtype=f64, device=device)
        t = torch.arange(k, dtype=f64, device=device) / (k - 1)
        return kap[:, None] ** (-t[None, :])

    for blk in range(start // nb, (start + batch + nb - 1) // nb):
        g = torch.Generator(device=device)
        g.manual_seed(block_seed(seed, blk))
        ka_blk = 10.0 ** (lo + (hi - lo) * torch.rand(nb, generator=g, device=device, dtype=f64))
        ka = min(m, n)
        UA, VA = haar_t(g, m, ka), haar_t(g, n, ka)
        A_blk = (UA * sig(ka, ka_blk)[:, None, :]) @ VA.transpose(1, 2)
        kb = min(p, n)
        UB, VB = haar_t(g, p, kb), haar_t(g, n, kb)
        kBv = torch.full((nb,), float(kappa_B), dtype=f64, device=device)
        B_blk = (UB * sig(kb, kBv)[:, None, :]) @ VB.transpose(1, 2)
        b_blk = torch.randn((nb, m), generator=g, device=device, dtype=f64)
        d_blk = torch.randn((nb, p), generator=g, device=device, dtype=f64)
        g0 = blk * nb                       # global index of the block's first problem
        s0, s1 = max(start, g0), min(start + batch, g0 + nb)
        o, i = s0 - start, s0 - g0          # output / in-block offsets
        c = s1 - s0
        A[o:o + c] = A_blk[i:i + c]
        B[o:o + c] = B_blk[i:i + c]
        b[o:o + c] = b_blk[i:i + c]
        d[o:o + c] = d_blk[i:i + c]
        kA[o:o + c] = ka_blk[i:i + c]
    return A, B, b, d, kA


# BASELINE.json configs (SURVEY.md §8 legend).  prec = (u_f, u_s, u_r).
CONFIGS = {
    "C1": dict(kind="lse", m=200, n=100, p=50, kappa_A=1e3, kappa_B=1e2, seed=1,
               prec=("low", "working", "working"), maxit=10),
    "C2": dict(kind="gls", n=200, m=100, p=150, kappa_A=1e4, kappa_B=1e2, seed=2,
               prec=("low", "low", "working"), maxit=10),
    "C3": dict(kind="lse", m=8192, n=4096, p=1024, kappa_A=1e4, kappa_B=1e2, seed=3,
               prec=("low", "low", "working"), maxit=40, kappa_sweep=(1e2, 1e4, 1e6)),
    "C4": dict(kind="lse_batch", batch=65536, m=256, n=128, p=32, log10_kappa_A=(1.0, 5.0),
               kappa_B=1e1, seed=1000, prec=("low", "low", "working"), maxit=40),
    "C5": dict(kind="gls_complex", n=4096, m=2048, p=3072, kappa_A=1e6, kappa_B=1e3, seed=5,
               prec=("low", "low", "working"), maxit=40),
}


def lse_batch_numpy(batch, m, n, p, log10_kappa_range=(1.0, 5.0), kappa_B=10.0, seed=1000):
    """CPU twin of lse_batch_torch (same distribution, numpy streams): per
    problem i the stream is seeded with seed + i (SURVEY.md §8(d) seed rule)."""
    A = np.empty((batch, m, n), order="C")
    B = np.empty((batch, p, n), order="C")
    b = np.empty((batch, m))
    d = np.empty((batch, p))
    kA = np.empty(batch)
    lo, hi = log10_kappa_range
    for i in range(batch):
        rng = np.random.default_rng(seed + i)
        kA[i] = 10.0 ** rng.uniform(lo, hi)
        A[i] = svd_matrix(rng, m, n, kA[i])
        B[i] = svd_matrix(rng, p, n, kappa_B)
        b[i] = rng.standard_normal(m)
        d[i] = rng.standard_normal(p)
    return A, B, b, d, kA
