"""Parity checker math (SURVEY.md §8(d) 'Parity checks per config').

* forward error   ||x_gpu - x_ref|| / ||x_ref||  <=  c * N * u * kappa,  c = 40,
                  N = m + n + p + 1, u = 2^-53 (u_r = working)
* iterations      |it_gpu - it_ref| <= 1
* backward error  the stop-test max ratio (lse.hpp:281-290, gls.hpp:255-264)
                  recomputed in fp64 from each returned state; GPU within 2x
                  of the oracle's, floored at 10 u (rounding noise) and -- when
                  both runs converged -- at 2 tol: a run allowed to stop one
                  pass earlier (iterations +-1) ends anywhere below tol, while
                  the oracle's extra correction can take it to ~u
"""
import numpy as np

U53 = 2.0 ** -53


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    if nb == 0:
        return float(np.linalg.norm(a))
    return float(np.linalg.norm(a - b) / nb)


def lse_backward(A, B, b, d, x, r, v):
    f1 = b - r - A @ x
    f2 = d - B @ x
    f3 = B.conj().T @ v - A.conj().T @ r
    nA, nB = np.linalg.norm(A), np.linalg.norm(B)
    nr, nv, nx = np.linalg.norm(r), np.linalg.norm(v), np.linalg.norm(x)

    def ratio(num, den):
        return num / den if den > 0 else (0.0 if num == 0 else np.inf)

    return max(ratio(np.linalg.norm(f1), np.linalg.norm(b) + nr + nA * nx),
               ratio(np.linalg.norm(f2), np.linalg.norm(d) + nB * nx),
               ratio(np.linalg.norm(f3), nA * nr + nB * nv))


def gls_backward(W, V, d, x, y, z):
    f1 = V.conj().T @ z - y
    f2 = d - W @ x - V @ y
    f3 = W.conj().T @ z
    nW, nV = np.linalg.norm(W), np.linalg.norm(V)
    nx, ny, nz = np.linalg.norm(x), np.linalg.norm(y), np.linalg.norm(z)

    def ratio(num, den):
        return num / den if den > 0 else (0.0 if num == 0 else np.inf)

    return max(ratio(np.linalg.norm(f1), ny + nV * nz),
               ratio(np.linalg.norm(f2), np.linalg.norm(d) + nW * nx + nV * ny),
               ratio(np.linalg.norm(f3), nW * nz))


def fwd_bound(m, n, p, kappa, c=40.0, u=U53):
    return c * (m + n + p + 1) * u * kappa


def check_parity(name, fwd, bound, it_gpu, it_ref, be_gpu, be_ref, status_gpu=None, status_ref=None,
                 tol=1e-13):
    msgs = []
    floor = 10 * U53
    if status_gpu == "converged" and status_ref == "converged":
        floor = max(floor, 2 * tol)
    if not fwd <= bound:
        msgs.append(f"{name}: forward error {fwd:.3e} > bound {bound:.3e}")
    if abs(int(it_gpu) - int(it_ref)) > 1:
        msgs.append(f"{name}: iterations gpu {it_gpu} vs oracle {it_ref}")
    if not be_gpu <= max(2.0 * be_ref, floor):
        msgs.append(f"{name}: backward error gpu {be_gpu:.3e} vs oracle {be_ref:.3e}")
    return msgs


def lse_kkt(A, B, b, d):
    """dense KKT solve of [0 B^T A^T; B 0 0; A 0 -I] style system (oracles.hpp:185-199 restated):
    A^T A x - B^T v... we solve the augmented system [[I, 0, A], [0, 0, B], [A^T, B^T, 0]]
    [r; -v; x] = [b; d; 0]."""
    m, n = A.shape
    p = B.shape[0]
    K = np.zeros((m + p + n, m + p + n), dtype=np.result_type(A, B))
    K[:m, :m] = np.eye(m)
    K[:m, m + p:] = A
    K[m:m + p, m + p:] = B
    K[m + p:, :m] = A.conj().T
    K[m + p:, m:m + p] = B.conj().T
    rhs = np.concatenate([b, d, np.zeros(n, dtype=K.dtype)])
    s = np.linalg.solve(K, rhs)
    return s[m + p:], s[:m], -s[m:m + p]


def gls_kkt(W, V, d):
    """[[I, V^H, 0], [V, 0, W], [0, W^H, 0]] [y; -z; x] = [0; d; 0] (oracles.hpp:206-219 restated)."""
    n, m = W.shape
    p = V.shape[1]
    K = np.zeros((p + n + m, p + n + m), dtype=np.result_type(W, V))
    K[:p, :p] = np.eye(p)
    K[:p, p:p + n] = V.conj().T
    K[p:p + n, :p] = V
    K[p:p + n, p + n:] = W
    K[p + n:, p:p + n] = W.conj().T
    rhs = np.concatenate([np.zeros(p, dtype=K.dtype), d, np.zeros(m, dtype=K.dtype)])
    s = np.linalg.solve(K, rhs)
    return s[p + n:], s[:p], -s[p:p + n]
