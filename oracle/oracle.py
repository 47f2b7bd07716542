"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY.

numpy front-end over the two CPU checkers (see oracle/orc_api.h):

* ``Oracle("ref")``  -> oracle/_ref/libmixedls_ref.so, the unmodified
  reference headers (/root/reference/proj/include/mixedls) behind a C shim;
* ``Oracle("port")`` -> oracle/_build/libmixedls_port.so, our restatement
  (real path bitwise-identical to "ref"; complex path for config C5).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg use
this module.  The product never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "ref": os.path.join(HERE, "_ref", "libmixedls_ref.so"),
    "port": os.path.join(HERE, "_build", "libmixedls_port.so"),
}
STATUS = {0: "converged", 1: "max_iterations", 2: "diverged"}
ERRORS = {1: "dimension_error", 2: "invalid_input", 3: "singular_triangular", 9: "error"}
LEVEL = {"low": 0, "working": 1, "extended": 2, "s": 0, "d": 1, "dd": 2}


class OracleError(RuntimeError):
    def __init__(self, code: int, index: int = -1):
        super().__init__(f"{ERRORS.get(code, code)}" + (f" (index {index})" if code == 3 else ""))
        self.code = code
        self.kind = ERRORS.get(code, "error")
        self.index = index


@dataclass
class OracleResult:
    x: np.ndarray
    r: np.ndarray  # LSE: r ; GLS: y
    v: np.ndarray  # LSE: v ; GLS: z
    status: str
    iterations: int
    history: np.ndarray
    phases: np.ndarray = field(default_factory=lambda: np.zeros(6))
    inner: int = 0  # GMRES iterations (gmres_lse)


_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_i64 = C.c_int64


def _p(a):
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


def _f(a, dtype=np.float64):
    return np.asfortranarray(np.asarray(a, dtype=dtype))


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])


def build(kind: str = "all") -> None:
    subprocess.run(["make", "-s", "-C", HERE, kind], check=True)


class Oracle:
    def __init__(self, kind: str = "port"):
        if kind not in LIBS:
            raise ValueError(kind)
        path = LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} (run `make -C oracle {kind}`)")
        self.kind = kind
        self.lib = C.CDLL(path)
        self.lib.orc_extended_dot.restype = C.c_double

    # -- drivers ------------------------------------------------------------
    def _solve(self, fn, dims, mats, vecs, outs_len, tol, maxit, prec, cplx=False):
        uf, us, ur = (LEVEL[p] if isinstance(p, str) else int(p) for p in prec)
        dt = np.complex128 if cplx else np.float64
        mats = [_f(M, dt) for M in mats]
        vecs = [np.ascontiguousarray(v, dtype=dt) for v in vecs]
        outs = [np.zeros(n, dtype=dt) for n in outs_len]
        st = C.c_int32(0)
        it = C.c_int64(0)
        hist = np.zeros(3 * max(int(maxit), 1))
        ph = np.zeros(6)
        sing = C.c_int64(-1)
        rc = fn(*[_i64(d) for d in dims], *[M.ctypes.data_as(_dp) for M in mats],
                *[v.ctypes.data_as(_dp) for v in vecs], C.c_double(tol), _i64(maxit),
                C.c_int(uf), C.c_int(us), C.c_int(ur), *[o.ctypes.data_as(_dp) for o in outs],
                C.byref(st), C.byref(it), _p(hist), _p(ph), C.byref(sing))
        if rc:
            raise OracleError(rc, sing.value)
        n_it = it.value
        return OracleResult(outs[0], outs[1], outs[2], STATUS[st.value], n_it,
                            hist[: 3 * n_it].reshape(n_it, 3).copy(), ph)

    def mplse(self, A, B, b, d, tol=1e-13, maxit=40, prec=("s", "s", "d"), cplx=False):
        m, n = np.shape(A)
        p = np.shape(B)[0]
        fn = self.lib.orc_mplse_z if cplx else self.lib.orc_mplse
        return self._solve(fn, (m, n, p), (A, B), (b, d), (n, m, p), tol, maxit, prec, cplx)

    def mpgls(self, W, V, d, tol=1e-13, maxit=40, prec=("s", "s", "d"), cplx=False):
        n, m = np.shape(W)
        p = np.shape(V)[1]
        fn = self.lib.orc_mpgls_z if cplx else self.lib.orc_mpgls
        return self._solve(fn, (n, m, p), (W, V), (d,), (m, p, n), tol, maxit, prec, cplx)

    def mplse_batch(self, A, B, b, d, tol=1e-13, maxit=40, prec=("s", "s", "d"), nthreads=1):
        """A: (batch, m, n) with each problem column-major (i.e. A[i].T contiguous)."""
        batch, m, n = A.shape
        p = B.shape[1]
        Ac = np.ascontiguousarray(np.transpose(A, (0, 2, 1)))
        Bc = np.ascontiguousarray(np.transpose(B, (0, 2, 1)))
        bc = np.ascontiguousarray(b, dtype=np.float64)
        dc = np.ascontiguousarray(d, dtype=np.float64)
        x = np.zeros((batch, n))
        r = np.zeros((batch, m))
        v = np.zeros((batch, p))
        st = np.zeros(batch, np.int32)
        it = np.zeros(batch, np.int64)
        err = np.zeros(batch, np.int32)
        uf, us, ur = (LEVEL[q] for q in prec)
        self.lib.orc_mplse_batch(_i64(batch), _i64(m), _i64(n), _i64(p), _p(Ac), _p(Bc), _p(bc),
                                 _p(dc), C.c_double(tol), _i64(maxit), C.c_int(uf), C.c_int(us),
                                 C.c_int(ur), _p(x), _p(r), _p(v), st.ctypes.data_as(_i32p),
                                 it.ctypes.data_as(_i64p), err.ctypes.data_as(_i32p),
                                 C.c_int(nthreads))
        return x, r, v, st, it, err

    # -- generator -------------------------------------------------------------
    def gen_lse(self, m, n, p, cond, seed, dist=0):
        A = np.zeros((m, n), order="F")
        B = np.zeros((p, n), order="F")
        b = np.zeros(m)
        d = np.zeros(p)
        rc = self.lib.orc_gen_lse(_i64(m), _i64(n), _i64(p), C.c_double(cond), C.c_uint64(seed),
                                  C.c_int(dist), _p(A), _p(B), _p(b), _p(d))
        if rc:
            raise OracleError(rc)
        return A, B, b, d

    def gen_gls(self, n, m, p, cond, seed, dist=0):
        W = np.zeros((n, m), order="F")
        V = np.zeros((n, p), order="F")
        d = np.zeros(n)
        rc = self.lib.orc_gen_gls(_i64(n), _i64(m), _i64(p), C.c_double(cond), C.c_uint64(seed),
                                  C.c_int(dist), _p(W), _p(V), _p(d))
        if rc:
            raise OracleError(rc)
        return W, V, d

    # -- components ------------------------------------------------------------
    def lse_residuals(self, A, B, b, d, x, r, v, ur="d"):
        m, n = A.shape
        p = B.shape[0]
        A, B = _f(A), _f(B)
        vs = [np.ascontiguousarray(t, np.float64) for t in (b, d, x, r, v)]
        f1, f2, f3 = np.zeros(m), np.zeros(p), np.zeros(n)
        rc = self.lib.orc_lse_residuals(_i64(m), _i64(n), _i64(p), _p(A), _p(B),
                                        *[_p(t) for t in vs], C.c_int(LEVEL[ur]), _p(f1), _p(f2),
                                        _p(f3))
        if rc:
            raise OracleError(rc)
        return f1, f2, f3

    def gls_residuals(self, W, V, d, x, y, z, ur="d"):
        n, m = W.shape
        p = V.shape[1]
        W, V = _f(W), _f(V)
        vs = [np.ascontiguousarray(t, np.float64) for t in (d, x, y, z)]
        f1, f2, f3 = np.zeros(p), np.zeros(n), np.zeros(m)
        rc = self.lib.orc_gls_residuals(_i64(n), _i64(m), _i64(p), _p(W), _p(V),
                                        *[_p(t) for t in vs], C.c_int(LEVEL[ur]), _p(f1), _p(f2),
                                        _p(f3))
        if rc:
            raise OracleError(rc)
        return f1, f2, f3

    def lse_correction(self, A, B, f1, f2, f3, uf="d"):
        m, n = A.shape
        p = B.shape[0]
        A, B = _f(A), _f(B)
        fs = [np.ascontiguousarray(t, np.float64) for t in (f1, f2, f3)]
        dr, dv, dx = np.zeros(m), np.zeros(p), np.zeros(n)
        sing = C.c_int64(-1)
        rc = self.lib.orc_lse_correction(_i64(m), _i64(n), _i64(p), _p(A), _p(B),
                                         *[_p(t) for t in fs], C.c_int(LEVEL[uf]), _p(dr), _p(dv),
                                         _p(dx), C.byref(sing))
        if rc:
            raise OracleError(rc, sing.value)
        return dr, dv, dx

    def gls_correction(self, W, V, f1, f2, f3, uf="d"):
        n, m = W.shape
        p = V.shape[1]
        W, V = _f(W), _f(V)
        fs = [np.ascontiguousarray(t, np.float64) for t in (f1, f2, f3)]
        dy, dz, dx = np.zeros(p), np.zeros(n), np.zeros(m)
        sing = C.c_int64(-1)
        rc = self.lib.orc_gls_correction(_i64(n), _i64(m), _i64(p), _p(W), _p(V),
                                         *[_p(t) for t in fs], C.c_int(LEVEL[uf]), _p(dy), _p(dz),
                                         _p(dx), C.byref(sing))
        if rc:
            raise OracleError(rc, sing.value)
        return dy, dz, dx

    def gmres_lse(self, A, B, b, d, tol=1e-13, maxit=40, prec=("s", "s", "d"), precond="bd_split",
                  alpha_scale=1.0):
        """gmres_refine_lse (krylov.hpp:545) -- reference build only."""
        if not hasattr(self.lib, "orc_gmres_lse"):
            raise OracleError(9)
        m, n = A.shape
        p = B.shape[0]
        A, B = _f(A), _f(B)
        b = np.ascontiguousarray(b, np.float64)
        d = np.ascontiguousarray(d, np.float64)
        x, r, v = np.zeros(n), np.zeros(m), np.zeros(p)
        st, it, inner = C.c_int32(0), C.c_int64(0), C.c_int64(0)
        hist = np.zeros(3 * max(maxit, 1))
        sing = C.c_int64(-1)
        uf, us, ur = (LEVEL[q] for q in prec)
        f = self.lib.orc_gmres_lse
        f.restype = C.c_int
        rc = f(_i64(m), _i64(n), _i64(p), _p(A), _p(B), _p(b), _p(d), C.c_double(tol), _i64(maxit),
               C.c_int(uf), C.c_int(us), C.c_int(ur), C.c_int(0 if precond == "left" else 1),
               C.c_double(alpha_scale), _p(x), _p(r), _p(v), C.byref(st), C.byref(it),
               C.byref(inner), _p(hist), C.byref(sing))
        if rc:
            raise OracleError(rc, sing.value)
        return OracleResult(x, r, v, STATUS[st.value], it.value,
                            hist[: 3 * it.value].reshape(-1, 3), inner=inner.value)

    def gmres_gls(self, W, V, d, tol=1e-13, maxit=40, prec=("s", "s", "d"), precond="bd_split",
                  alpha_scale=1.0):
        """gmres_refine_gls (krylov.hpp:673) -- reference build only.  Returns
        (x, y, z) as OracleResult(x, r=y, v=z)."""
        if not hasattr(self.lib, "orc_gmres_gls"):
            raise OracleError(9)
        n, m = W.shape
        p = V.shape[1]
        W, V = _f(W), _f(V)
        d = np.ascontiguousarray(d, np.float64)
        x, y, z = np.zeros(m), np.zeros(p), np.zeros(n)
        st, it, inner = C.c_int32(0), C.c_int64(0), C.c_int64(0)
        hist = np.zeros(3 * max(maxit, 1))
        sing = C.c_int64(-1)
        uf, us, ur = (LEVEL[q] for q in prec)
        f = self.lib.orc_gmres_gls
        f.restype = C.c_int
        rc = f(_i64(n), _i64(m), _i64(p), _p(W), _p(V), _p(d), C.c_double(tol), _i64(maxit), C.c_int(uf),
               C.c_int(us), C.c_int(ur), C.c_int(0 if precond == "left" else 1), C.c_double(alpha_scale),
               _p(x), _p(y), _p(z), C.byref(st), C.byref(it), C.byref(inner), _p(hist), C.byref(sing))
        if rc:
            raise OracleError(rc, sing.value)
        return OracleResult(x, y, z, STATUS[st.value], it.value,
                            hist[: 3 * it.value].reshape(-1, 3), inner=inner.value)

    def lse_direct(self, A, B, b, d):
        m, n = A.shape
        p = B.shape[0]
        A, B = _f(A), _f(B)
        b = np.ascontiguousarray(b, np.float64)
        d = np.ascontiguousarray(d, np.float64)
        x, r, v = np.zeros(n), np.zeros(m), np.zeros(p)
        sing = C.c_int64(-1)
        rc = self.lib.orc_lse_direct(_i64(m), _i64(n), _i64(p), _p(A), _p(B), _p(b), _p(d), _p(x),
                                     _p(r), _p(v), C.byref(sing))
        if rc:
            raise OracleError(rc, sing.value)
        return x, r, v

    def gls_direct(self, W, V, d):
        n, m = W.shape
        p = V.shape[1]
        W, V = _f(W), _f(V)
        d = np.ascontiguousarray(d, np.float64)
        x, y, z = np.zeros(m), np.zeros(p), np.zeros(n)
        sing = C.c_int64(-1)
        rc = self.lib.orc_gls_direct(_i64(n), _i64(m), _i64(p), _p(W), _p(V), _p(d), _p(x),
                                     _p(y), _p(z), C.byref(sing))
        if rc:
            raise OracleError(rc, sing.value)
        return x, y, z

    def extended_dot(self, x, y):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        return self.lib.orc_extended_dot(_i64(len(x)), _p(x), _p(y))

    def trsv(self, T, rhs, transpose=False):
        n = T.shape[0]
        T = _f(T)
        rhs = np.ascontiguousarray(rhs, np.float64)
        x = np.zeros(n)
        sing = C.c_int64(-1)
        rc = self.lib.orc_trsv(_i64(n), _p(T), _p(rhs), C.c_int(int(transpose)), _p(x),
                               C.byref(sing))
        if rc:
            raise OracleError(rc, sing.value)
        return x
