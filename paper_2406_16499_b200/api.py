"""Reference-shaped Python API over the C ABI (include/mixedls_b200.h).

Host numpy inputs are copied to the device inside the call (the end-to-end
path); CUDA tensors (anything exposing ``data_ptr()`` and ``is_cuda``) are
used in place with MLSB_DEVICE pointers.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import Config, Exec, Trace, lib, raise_for

_STATUS = {0: "converged", 1: "max_iterations", 2: "diverged"}
_LEVELS = {"low": 0, "working": 1, "extended": 2}


# ---------------------------------------------------------------------------
# configuration (precision.hpp:57-90, refine.hpp:28-38)
@dataclass
class PrecisionConfig:
    factor: str = "low"
    solve: str = "low"
    working: str = "working"
    residual: str = "working"

    @staticmethod
    def classical() -> "PrecisionConfig":
        return PrecisionConfig()

    @staticmethod
    def classical_extended() -> "PrecisionConfig":
        return PrecisionConfig(residual="extended")

    @staticmethod
    def all_working(residual: str = "working") -> "PrecisionConfig":
        return PrecisionConfig("working", "working", "working", residual)


@dataclass
class RefinementConfig:
    tol: float = 1e-13
    maxit: int = 40
    precisions: PrecisionConfig = field(default_factory=PrecisionConfig)

    def to_c(self) -> Config:
        p = self.precisions

        def lv(s):
            return _LEVELS.get(s, -1) if isinstance(s, str) else int(s)

        return Config(float(self.tol), int(self.maxit), lv(p.factor), lv(p.solve), lv(p.working),
                      lv(p.residual))


# ---------------------------------------------------------------------------
# problems / states / results (lse.hpp:17-42, gls.hpp:17-39, refine.hpp:56-61)
@dataclass
class LseProblem:
    A: np.ndarray  # m x n
    B: np.ndarray  # p x n
    b: np.ndarray  # m
    d: np.ndarray  # p


@dataclass
class GlsProblem:
    W: np.ndarray  # n x m
    V: np.ndarray  # n x p
    d: np.ndarray  # n


@dataclass
class LseState:
    x: np.ndarray
    r: np.ndarray
    v: np.ndarray


@dataclass
class GlsState:
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray


@dataclass
class RefinementTrace:
    status: str
    iterations: int
    residual_history: np.ndarray  # (iterations, 3), unscaled
    inner_iterations: int = 0
    timing: dict = field(default_factory=dict)


@dataclass
class MplseResult:
    state: LseState
    trace: RefinementTrace


@dataclass
class MpglsResult:
    state: GlsState
    trace: RefinementTrace


_PHASES = ("factorization", "init", "residual", "correction", "gmres", "other")


def _is_cuda(t) -> bool:
    return bool(getattr(t, "is_cuda", False)) and hasattr(t, "data_ptr")


def _ptr(a):
    if a is None:
        return None
    if _is_cuda(a):
        return C.c_void_p(a.data_ptr())
    return C.c_void_p(a.ctypes.data)


def _exec(device_mode: bool, stream=None, device: int = -1) -> Exec:
    s = None
    if stream is not None:
        s = getattr(stream, "cuda_stream", stream)
    return Exec(_capi.MLSB_DEVICE if device_mode else _capi.MLSB_HOST, int(device),
                C.c_void_p(s) if s else None)


def _matrix_ld(M):
    """(rows, cols, ld) of a column-major 2-D host array or CUDA tensor."""
    rows, cols = M.shape
    if _is_cuda(M):
        s0, s1 = M.stride()
        if s0 != 1 and rows > 1:
            raise _capi.DimensionError("device matrices must be column-major (stride(0) == 1)")
        return rows, cols, max(s1, rows, 1)
    return rows, cols, max(rows, 1)


def _dev_inputs(mats, vecs, shapes, what):
    """Validate the CUDA-tensor inputs of a single solve before they reach the C
    ABI: binary64, one device, 2-D column-major matrices, vectors of the right
    length with unit stride (made contiguous).  Wrong input here would be read
    out of bounds on the device.  Returns the (possibly contiguous) vectors."""
    import torch

    dev = mats[0].device
    for t in list(mats) + list(vecs):
        if not _is_cuda(t):
            raise _capi.InvalidInput(f"{what}: mixing CUDA tensors and host arrays")
        if t.device != dev:
            raise _capi.InvalidInput(f"{what}: inputs on different devices")
        if t.dtype != torch.float64:
            raise _capi.InvalidInput(f"{what}: CUDA inputs must be torch.float64 (got {t.dtype})")
    for M in mats:
        if M.dim() != 2:
            raise _capi.DimensionError(f"{what}: matrices must be 2-D")
    out = []
    for v, n in zip(vecs, shapes):
        if v.dim() != 1 or v.shape[0] != n:
            raise _capi.DimensionError(f"{what}: rhs length mismatch")
        out.append(v if v.stride(0) == 1 else v.contiguous())
    return out


def _dev_lse(pb, what="lse_problem"):
    A, B = pb.A, pb.B
    if A.dim() != 2 or B.dim() != 2 or A.shape[1] != B.shape[1]:
        raise _capi.DimensionError(f"{what}: A and B column counts differ")
    b, d = _dev_inputs((A, B), (pb.b, pb.d), (A.shape[0], B.shape[0]), what)
    m, n, lda = _matrix_ld(A)
    p, _, ldb = _matrix_ld(B)
    return A, B, b, d, m, n, p, lda, ldb


def _dev_gls(pb, what="gls_problem"):
    W, V = pb.W, pb.V
    if W.dim() != 2 or V.dim() != 2 or W.shape[0] != V.shape[0]:
        raise _capi.DimensionError(f"{what}: W and V row counts differ")
    (d,) = _dev_inputs((W, V), (pb.d,), (W.shape[0],), what)
    n, m, ldw = _matrix_ld(W)
    _, p, ldv = _matrix_ld(V)
    return W, V, d, n, m, p, ldw, ldv


def _trace_from(tr: Trace, hist: np.ndarray) -> RefinementTrace:
    it = int(tr.iterations)
    return RefinementTrace(_STATUS.get(tr.status, str(tr.status)), it,
                           hist[: 3 * it].reshape(it, 3).copy(), int(tr.inner_iterations),
                           {k: float(tr.phase_seconds[i]) for i, k in enumerate(_PHASES)})


# ---------------------------------------------------------------------------
def mplse(pb: LseProblem, cfg: RefinementConfig | None = None, stream=None) -> MplseResult:
    """Four-precision classical IR for LSE (lse.hpp:303-429) on the GPU."""
    cfg = cfg or RefinementConfig()
    ccfg = cfg.to_c()
    dev = _is_cuda(pb.A)
    if dev:
        import torch

        A, B, b, d, m, n, p, lda, ldb = _dev_lse(pb)
        x = torch.empty(n, dtype=torch.float64, device=A.device)
        r = torch.empty(m, dtype=torch.float64, device=A.device)
        v = torch.empty(p, dtype=torch.float64, device=A.device)
    else:
        cplx = any(np.iscomplexobj(t) for t in (pb.A, pb.B, pb.b, pb.d))
        dt = np.complex128 if cplx else np.float64
        A = np.asfortranarray(pb.A, dtype=dt)
        B = np.asfortranarray(pb.B, dtype=dt)
        if A.ndim != 2 or B.ndim != 2 or B.shape[1] != A.shape[1]:
            raise _capi.DimensionError("lse_problem: A and B column counts differ")
        b = np.ascontiguousarray(pb.b, dtype=dt)
        d = np.ascontiguousarray(pb.d, dtype=dt)
        m, n = A.shape
        p = B.shape[0]
        if b.shape != (m,) or d.shape != (p,):
            raise _capi.DimensionError("lse_problem: rhs length mismatch")
        lda, ldb = max(m, 1), max(p, 1)
        x, r, v = np.zeros(n, dt), np.zeros(m, dt), np.zeros(p, dt)
    hist = np.zeros(3 * max(int(cfg.maxit), 1))
    tr = Trace()
    tr.residual_history = hist.ctypes.data_as(C.POINTER(C.c_double))
    sing = C.c_int64(-1)
    ex = _exec(dev, stream)
    fn = lib.mlsb_mplse_z if (not dev and np.iscomplexobj(A)) else lib.mlsb_mplse
    rc = fn(_ptr(A), lda, _ptr(B), ldb, _ptr(b), _ptr(d), m, n, p, C.byref(ccfg),
                        _ptr(x), _ptr(r), _ptr(v), C.byref(tr), C.byref(sing), C.byref(ex))
    raise_for(rc, sing.value)
    return MplseResult(LseState(x, r, v), _trace_from(tr, hist))


def mpgls(pb: GlsProblem, cfg: RefinementConfig | None = None, stream=None) -> MpglsResult:
    """Four-precision classical IR for GLS (gls.hpp:276-387) on the GPU."""
    cfg = cfg or RefinementConfig()
    ccfg = cfg.to_c()
    dev = _is_cuda(pb.W)
    if dev:
        import torch

        W, V, d, n, m, p, ldw, ldv = _dev_gls(pb)
        x = torch.empty(m, dtype=torch.float64, device=W.device)
        y = torch.empty(p, dtype=torch.float64, device=W.device)
        z = torch.empty(n, dtype=torch.float64, device=W.device)
    else:
        cplx = any(np.iscomplexobj(t) for t in (pb.W, pb.V, pb.d))
        dt = np.complex128 if cplx else np.float64
        W = np.asfortranarray(pb.W, dtype=dt)
        V = np.asfortranarray(pb.V, dtype=dt)
        if W.ndim != 2 or V.ndim != 2 or V.shape[0] != W.shape[0]:
            raise _capi.DimensionError("gls_problem: W and V row counts differ")
        d = np.ascontiguousarray(pb.d, dtype=dt)
        n, m = W.shape
        p = V.shape[1]
        if d.shape != (n,):
            raise _capi.DimensionError("gls_problem: rhs length mismatch")
        ldw = ldv = max(n, 1)
        x, y, z = np.zeros(m, dt), np.zeros(p, dt), np.zeros(n, dt)
    hist = np.zeros(3 * max(int(cfg.maxit), 1))
    tr = Trace()
    tr.residual_history = hist.ctypes.data_as(C.POINTER(C.c_double))
    sing = C.c_int64(-1)
    ex = _exec(dev, stream)
    fn = lib.mlsb_mpgls_z if (not dev and np.iscomplexobj(W)) else lib.mlsb_mpgls
    rc = fn(_ptr(W), ldw, _ptr(V), ldv, _ptr(d), n, m, p, C.byref(ccfg), _ptr(x),
                        _ptr(y), _ptr(z), C.byref(tr), C.byref(sing), C.byref(ex))
    raise_for(rc, sing.value)
    return MpglsResult(GlsState(x, y, z), _trace_from(tr, hist))


def gmres_refine_lse(pb: LseProblem, cfg: RefinementConfig | None = None,
                     precond: str = "bd_split", alpha_scale: float = 1.0,
                     stream=None) -> MplseResult:
    """GMRES-IR for LSE (gmres_refine_lse, inc/krylov.hpp:545-689) on the GPU:
    precond "left" or "bd_split"; trace.inner_iterations = total GMRES steps."""
    cfg = cfg or RefinementConfig()
    ccfg = cfg.to_c()
    if precond not in ("left", "bd_split"):
        raise _capi.InvalidInput("gmres: precond must be 'left' or 'bd_split'")
    dev = _is_cuda(pb.A)
    if dev:
        import torch

        A, B, b, d, m, n, p, lda, ldb = _dev_lse(pb)
        x = torch.empty(n, dtype=torch.float64, device=A.device)
        r = torch.empty(m, dtype=torch.float64, device=A.device)
        v = torch.empty(p, dtype=torch.float64, device=A.device)
    else:
        A = np.asfortranarray(pb.A, dtype=np.float64)
        B = np.asfortranarray(pb.B, dtype=np.float64)
        if A.ndim != 2 or B.ndim != 2 or B.shape[1] != A.shape[1]:
            raise _capi.DimensionError("lse_problem: A and B column counts differ")
        b = np.ascontiguousarray(pb.b, dtype=np.float64)
        d = np.ascontiguousarray(pb.d, dtype=np.float64)
        m, n = A.shape
        p = B.shape[0]
        if b.shape != (m,) or d.shape != (p,):
            raise _capi.DimensionError("lse_problem: rhs length mismatch")
        lda, ldb = max(m, 1), max(p, 1)
        x, r, v = np.zeros(n), np.zeros(m), np.zeros(p)
    hist = np.zeros(3 * max(int(cfg.maxit), 1))
    tr = Trace()
    tr.residual_history = hist.ctypes.data_as(C.POINTER(C.c_double))
    sing = C.c_int64(-1)
    ex = _exec(dev, stream)
    rc = lib.mlsb_gmres_lse(_ptr(A), lda, _ptr(B), ldb, _ptr(b), _ptr(d), m, n, p, C.byref(ccfg),
                            0 if precond == "left" else 1, float(alpha_scale), _ptr(x), _ptr(r),
                            _ptr(v), C.byref(tr), C.byref(sing), C.byref(ex))
    raise_for(rc, sing.value)
    return MplseResult(LseState(x, r, v), _trace_from(tr, hist))


def gmres_refine_gls(pb: GlsProblem, cfg: RefinementConfig | None = None,
                     precond: str = "bd_split", alpha_scale: float = 1.0,
                     stream=None) -> MpglsResult:
    """GMRES-IR for GLS (gmres_refine_gls, inc/krylov.hpp:673-784) on the GPU:
    precond "left" or "bd_split"; trace.inner_iterations = total GMRES steps."""
    cfg = cfg or RefinementConfig()
    ccfg = cfg.to_c()
    if precond not in ("left", "bd_split"):
        raise _capi.InvalidInput("gmres: precond must be 'left' or 'bd_split'")
    dev = _is_cuda(pb.W)
    if dev:
        import torch

        W, V, d, n, m, p, ldw, ldv = _dev_gls(pb)
        x = torch.empty(m, dtype=torch.float64, device=W.device)
        y = torch.empty(p, dtype=torch.float64, device=W.device)
        z = torch.empty(n, dtype=torch.float64, device=W.device)
    else:
        W = np.asfortranarray(pb.W, dtype=np.float64)
        V = np.asfortranarray(pb.V, dtype=np.float64)
        if W.ndim != 2 or V.ndim != 2 or V.shape[0] != W.shape[0]:
            raise _capi.DimensionError("gls_problem: W and V row counts differ")
        d = np.ascontiguousarray(pb.d, dtype=np.float64)
        n, m = W.shape
        p = V.shape[1]
        if d.shape != (n,):
            raise _capi.DimensionError("gls_problem: rhs length mismatch")
        ldw = ldv = max(n, 1)
        x, y, z = np.zeros(m), np.zeros(p), np.zeros(n)
    hist = np.zeros(3 * max(int(cfg.maxit), 1))
    tr = Trace()
    tr.residual_history = hist.ctypes.data_as(C.POINTER(C.c_double))
    sing = C.c_int64(-1)
    ex = _exec(dev, stream)
    rc = lib.mlsb_gmres_gls(_ptr(W), ldw, _ptr(V), ldv, _ptr(d), n, m, p, C.byref(ccfg),
                            0 if precond == "left" else 1, float(alpha_scale), _ptr(x), _ptr(y),
                            _ptr(z), C.byref(tr), C.byref(sing), C.byref(ex))
    raise_for(rc, sing.value)
    return MpglsResult(GlsState(x, y, z), _trace_from(tr, hist))


def lse_direct(pb: LseProblem, stream=None) -> LseState:
    """binary64 direct LSE solve on the GPU: the err-2 reference of the experiment
    harness (detail::lse_direct_reference, inc/experiment.hpp:50-59)."""
    dev = _is_cuda(pb.A)
    if dev:
        import torch

        A, B, b, d, m, n, p, lda, ldb = _dev_lse(pb)
        x = torch.empty(n, dtype=torch.float64, device=A.device)
        r = torch.empty(m, dtype=torch.float64, device=A.device)
        v = torch.empty(p, dtype=torch.float64, device=A.device)
    else:
        A = np.asfortranarray(pb.A, dtype=np.float64)
        B = np.asfortranarray(pb.B, dtype=np.float64)
        if A.ndim != 2 or B.ndim != 2 or B.shape[1] != A.shape[1]:
            raise _capi.DimensionError("lse_problem: A and B column counts differ")
        b = np.ascontiguousarray(pb.b, dtype=np.float64)
        d = np.ascontiguousarray(pb.d, dtype=np.float64)
        m, n = A.shape
        p = B.shape[0]
        if b.shape != (m,) or d.shape != (p,):
            raise _capi.DimensionError("lse_problem: rhs length mismatch")
        lda, ldb = max(m, 1), max(p, 1)
        x, r, v = np.zeros(n), np.zeros(m), np.zeros(p)
    sing = C.c_int64(-1)
    ex = _exec(dev, stream)
    rc = lib.mlsb_lse_direct(_ptr(A), lda, _ptr(B), ldb, _ptr(b), _ptr(d), m, n, p, _ptr(x),
                             _ptr(r), _ptr(v), C.byref(sing), C.byref(ex))
    raise_for(rc, sing.value)
    return LseState(x, r, v)


def gls_direct(pb: GlsProblem, stream=None) -> GlsState:
    """binary64 direct GLS solve on the GPU: the er-2 reference of the experiment
    harness (detail::gls_direct_reference, inc/experiment.hpp:65-73)."""
    dev = _is_cuda(pb.W)
    if dev:
        import torch

        W, V, d, n, m, p, ldw, ldv = _dev_gls(pb)
        x = torch.empty(m, dtype=torch.float64, device=W.device)
        y = torch.empty(p, dtype=torch.float64, device=W.device)
        z = torch.empty(n, dtype=torch.float64, device=W.device)
    else:
        W = np.asfortranarray(pb.W, dtype=np.float64)
        V = np.asfortranarray(pb.V, dtype=np.float64)
        if W.ndim != 2 or V.ndim != 2 or V.shape[0] != W.shape[0]:
            raise _capi.DimensionError("gls_problem: W and V row counts differ")
        d = np.ascontiguousarray(pb.d, dtype=np.float64)
        n, m = W.shape
        p = V.shape[1]
        if d.shape != (n,):
            raise _capi.DimensionError("gls_problem: rhs length mismatch")
        ldw = ldv = max(n, 1)
        x, y, z = np.zeros(m), np.zeros(p), np.zeros(n)
    sing = C.c_int64(-1)
    ex = _exec(dev, stream)
    rc = lib.mlsb_gls_direct(_ptr(W), ldw, _ptr(V), ldv, _ptr(d), n, m, p, _ptr(x), _ptr(y),
                             _ptr(z), C.byref(sing), C.byref(ex))
    raise_for(rc, sing.value)
    return GlsState(x, y, z)


# ---------------------------------------------------------------------------
@dataclass
class BatchResult:
    x: object
    r: object  # LSE r ; GLS y
    v: object  # LSE v ; GLS z
    status: object
    iterations: object
    errcode: object
    history: object = None


def _batched_layout(A):
    """A batch of column-major matrices as a (batch, rows, cols) array/tensor with
    stride(1) == 1.  Returns (batch, rows, cols, ld, batch_stride)."""
    bt, rows, cols = A.shape
    if _is_cuda(A):
        s = A.stride()
    else:
        s = tuple(x // A.itemsize for x in A.strides)
    if s[1] != 1 and rows > 1:
        raise _capi.DimensionError("batched matrices must be column-major per problem")
    return bt, rows, cols, max(s[2], rows), s[0]


def _batch_common(kind, A, B, rhs1, rhs2, cfg, stream, history):
    cfg = cfg or RefinementConfig()
    ccfg = cfg.to_c()
    dev = _is_cuda(A)
    if not dev:
        A = np.asarray(A, dtype=np.float64)
        B = np.asarray(B, dtype=np.float64)
        # column-major per problem
        A = np.ascontiguousarray(A.transpose(0, 2, 1)).transpose(0, 2, 1)
        B = np.ascontiguousarray(B.transpose(0, 2, 1)).transpose(0, 2, 1)
        rhs2 = np.ascontiguousarray(rhs2, dtype=np.float64)
        if rhs1 is not None:
            rhs1 = np.ascontiguousarray(rhs1, dtype=np.float64)
    if dev:
        import torch

        for t in (A, B, rhs1, rhs2):
            if t is None:
                continue
            if not _is_cuda(t) or t.device != A.device:
                raise _capi.InvalidInput("batched: all inputs must be CUDA tensors on one device")
            if t.dtype != torch.float64:
                raise _capi.InvalidInput(f"batched: CUDA inputs must be torch.float64 (got {t.dtype})")
        if A.dim() != 3 or B.dim() != 3:
            raise _capi.DimensionError("batched: matrices must be (batch, rows, cols)")
    bt, ra, ca, lda, sA = _batched_layout(A)
    bt2, rb, cb, ldb, sB = _batched_layout(B)
    if bt2 != bt:
        raise _capi.DimensionError("batch sizes differ")
    if kind == "lse":
        m, n, p = ra, ca, rb
        nx, nr, nv = n, m, p
        if cb != n:
            raise _capi.DimensionError("lse_problem: A and B column counts differ")
    else:
        n, m, p = ra, ca, cb
        nx, nr, nv = m, p, n
        if rb != n:
            raise _capi.DimensionError("gls_problem: W and V row counts differ")
    want = ((rhs1, m), (rhs2, p)) if kind == "lse" else ((rhs2, n),)
    for t, ln in want:
        if tuple(t.shape) != (bt, ln):
            raise _capi.DimensionError("batched: rhs shape mismatch")
    if dev:
        if rhs1 is not None and rhs1.stride(1) != 1:
            rhs1 = rhs1.contiguous()
        if rhs2.stride(1) != 1:
            rhs2 = rhs2.contiguous()

    def vstride(t):
        if t is None:
            return 0
        if _is_cuda(t):
            return t.stride(0)
        return t.strides[0] // t.itemsize

    if dev:
        import torch

        mk = lambda k, dt=torch.float64: torch.empty(k, dtype=dt, device=A.device)  # noqa: E731
        x, r, v = mk((bt, nx)), mk((bt, nr)), mk((bt, nv))
        status, iters, err = mk(bt, torch.int32), mk(bt, torch.int64), mk(bt, torch.int32)
        sing = mk(bt, torch.int64)
        hist = mk((bt, cfg.maxit, 3)) if history else None
    else:
        x, r, v = np.zeros((bt, nx)), np.zeros((bt, nr)), np.zeros((bt, nv))
        status, iters = np.zeros(bt, np.int32), np.zeros(bt, np.int64)
        err, sing = np.zeros(bt, np.int32), np.zeros(bt, np.int64)
        hist = np.zeros((bt, cfg.maxit, 3)) if history else None
    ex = _exec(dev, stream)
    if kind == "lse":
        rc = lib.mlsb_mplse_batched(bt, _ptr(A), lda, sA, _ptr(B), ldb, sB, _ptr(rhs1),
                                    vstride(rhs1), _ptr(rhs2), vstride(rhs2), m, n, p,
                                    C.byref(ccfg), _ptr(x), _ptr(r), _ptr(v), _ptr(status),
                                    _ptr(iters), _ptr(err), _ptr(sing), _ptr(hist), C.byref(ex))
    else:
        rc = lib.mlsb_mpgls_batched(bt, _ptr(A), lda, sA, _ptr(B), ldb, sB, _ptr(rhs2),
                                    vstride(rhs2), n, m, p, C.byref(ccfg), _ptr(x), _ptr(r),
                                    _ptr(v), _ptr(status), _ptr(iters), _ptr(err), _ptr(sing),
                                    _ptr(hist), C.byref(ex))
    raise_for(rc)
    return BatchResult(x, r, v, status, iters, err, hist)


def mplse_batched(A, B, b, d, cfg: RefinementConfig | None = None, stream=None,
                  history: bool = False) -> BatchResult:
    """Independent LSE solves, one CTA per problem.  A: (batch, m, n), B: (batch, p, n),
    column-major per problem; b: (batch, m); d: (batch, p).  CUDA inputs run
    asynchronously on `stream` (status/iterations/errcode are device tensors)."""
    return _batch_common("lse", A, B, b, d, cfg, stream, history)


def mpgls_batched(W, V, d, cfg: RefinementConfig | None = None, stream=None,
                  history: bool = False) -> BatchResult:
    """Independent GLS solves.  W: (batch, n, m), V: (batch, n, p); d: (batch, n)."""
    return _batch_common("gls", W, V, None, d, cfg, stream, history)
