"""ctypes binding of include/mixedls_b200.h (libmixedls_b200.so).

The library is loaded eagerly and loudly: if it is missing the import fails
with instructions to build it -- there is no Python fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(HERE, "lib", "libmixedls_b200.so")

MLSB_OK, MLSB_ERR_DIMENSION, MLSB_ERR_INVALID_INPUT, MLSB_ERR_SINGULAR = 0, 1, 2, 3
MLSB_ERR_CUDA, MLSB_ERR_UNSUPPORTED, MLSB_ERR_OTHER = 4, 5, 9
MLSB_HOST, MLSB_DEVICE = 0, 1


class MixedlsError(RuntimeError):
    """Base of the reference's exception hierarchy (errors.hpp:14-16)."""


class DimensionError(MixedlsError):
    pass


class InvalidInput(MixedlsError):
    pass


class SingularTriangular(MixedlsError):
    def __init__(self, msg: str, index: int):
        super().__init__(msg)
        self.index = index


class CudaError(MixedlsError):
    pass


class Unsupported(MixedlsError):
    pass


class Config(C.Structure):
    _fields_ = [("tol", C.c_double), ("maxit", C.c_int64), ("u_f", C.c_int32),
                ("u_s", C.c_int32), ("u", C.c_int32), ("u_r", C.c_int32)]


class Trace(C.Structure):
    _fields_ = [("status", C.c_int32), ("reserved", C.c_int32), ("iterations", C.c_int64),
                ("inner_iterations", C.c_int64), ("residual_history", C.POINTER(C.c_double)),
                ("phase_seconds", C.c_double * 6)]


class Exec(C.Structure):
    _fields_ = [("pointer_kind", C.c_int32), ("device", C.c_int32), ("stream", C.c_void_p)]


def _load():
    if not os.path.exists(lib_path):
        raise ImportError(
            f"{lib_path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " or `make -C paper_2406_16499_b200/csrc` (there is no CPU fallback)")
    L = C.CDLL(lib_path)
    dp, i64, i64p, i32p = C.c_void_p, C.c_int64, C.POINTER(C.c_int64), C.c_void_p
    cfgp, trp, exp_ = C.POINTER(Config), C.POINTER(Trace), C.POINTER(Exec)
    L.mlsb_default_config.restype = Config
    L.mlsb_last_error.restype = C.c_char_p
    L.mlsb_version.restype = C.c_int
    L.mlsb_mplse.argtypes = [dp, i64, dp, i64, dp, dp, i64, i64, i64, cfgp, dp, dp, dp, trp, i64p,
                             exp_]
    L.mlsb_mpgls.argtypes = [dp, i64, dp, i64, dp, i64, i64, i64, cfgp, dp, dp, dp, trp, i64p, exp_]
    L.mlsb_mplse_z.argtypes = L.mlsb_mplse.argtypes
    L.mlsb_mpgls_z.argtypes = L.mlsb_mpgls.argtypes
    L.mlsb_mplse_batched.argtypes = [i64, dp, i64, i64, dp, i64, i64, dp, i64, dp, i64, i64, i64,
                                     i64, cfgp, dp, dp, dp, i32p, dp, i32p, dp, dp, exp_]
    L.mlsb_mpgls_batched.argtypes = [i64, dp, i64, i64, dp, i64, i64, dp, i64, i64, i64, i64, cfgp,
                                     dp, dp, dp, i32p, dp, i32p, dp, dp, exp_]
    L.mlsb_gmres_lse.argtypes = [dp, i64, dp, i64, dp, dp, i64, i64, i64, cfgp, C.c_int, C.c_double,
                                 dp, dp, dp, trp, i64p, exp_]
    L.mlsb_gmres_gls.argtypes = [dp, i64, dp, i64, dp, i64, i64, i64, cfgp, C.c_int, C.c_double,
                                 dp, dp, dp, trp, i64p, exp_]
    L.mlsb_lse_direct.argtypes = [dp, i64, dp, i64, dp, dp, i64, i64, i64, dp, dp, dp, i64p, exp_]
    L.mlsb_gls_direct.argtypes = [dp, i64, dp, i64, dp, i64, i64, i64, dp, dp, dp, i64p, exp_]
    for f in ("mlsb_mplse", "mlsb_mpgls", "mlsb_mplse_batched", "mlsb_mpgls_batched",
              "mlsb_mplse_z", "mlsb_mpgls_z", "mlsb_lse_direct", "mlsb_gls_direct",
              "mlsb_gmres_lse", "mlsb_gmres_gls"):
        getattr(L, f).restype = C.c_int
    return L


lib = _load()


def raise_for(rc: int, sing: int = -1) -> None:
    if rc == MLSB_OK:
        return
    msg = lib.mlsb_last_error().decode(errors="replace")
    if rc == MLSB_ERR_DIMENSION:
        raise DimensionError(msg)
    if rc == MLSB_ERR_INVALID_INPUT:
        raise InvalidInput(msg)
    if rc == MLSB_ERR_SINGULAR:
        raise SingularTriangular(msg, sing)
    if rc == MLSB_ERR_CUDA:
        raise CudaError(msg)
    if rc == MLSB_ERR_UNSUPPORTED:
        raise Unsupported(msg)
    raise MixedlsError(msg)
