"""paper_2406_16499_b200 -- B200-native mixed-precision iterative refinement
for LSE / GLS (arXiv 2406.16499), a drop-in for the reference library's
classical-IR path.

The Python layer mirrors the reference's C++ interface
(/root/reference/proj/include/mixedls):

    reference                                   here
    -------------------------------------------  ------------------------------
    lse_problem {A, B, b, d}     lse.hpp:17-35   LseProblem(A, B, b, d)
    gls_problem {W, V, d}        gls.hpp:17-33   GlsProblem(W, V, d)
    precision_config             precision.hpp:57-90
                                                 PrecisionConfig (.classical(),
                                                 .classical_extended(), .all_working())
    refinement_config            refine.hpp:28-38 RefinementConfig(tol, maxit, precisions)
    mplse(pb, cfg) -> mplse_result  lse.hpp:303  mplse(pb, cfg) -> MplseResult
    mpgls(pb, cfg) -> mpgls_result  gls.hpp:276  mpgls(pb, cfg) -> MpglsResult
    dimension_error / invalid_input / singular_triangular (errors.hpp:14-49)
                                                 DimensionError / InvalidInput /
                                                 SingularTriangular(.index)

Every call goes through the C ABI of ``lib/libmixedls_b200.so``
(include/mixedls_b200.h) and runs on the GPU; there is no CPU fallback.
"""
from __future__ import annotations

from ._capi import (  # noqa: F401
    CudaError,
    DimensionError,
    InvalidInput,
    MixedlsError,
    SingularTriangular,
    Unsupported,
    lib,
    lib_path,
)
from .api import (  # noqa: F401
    GlsProblem,
    GlsState,
    LseProblem,
    LseState,
    MpglsResult,
    MplseResult,
    PrecisionConfig,
    RefinementConfig,
    RefinementTrace,
    gls_direct,
    gmres_refine_lse,
    gmres_refine_gls,
    lse_direct,
    mpgls,
    mpgls_batched,
    mplse,
    mplse_batched,
)

__all__ = [
    "LseProblem", "GlsProblem", "LseState", "GlsState", "PrecisionConfig", "RefinementConfig",
    "RefinementTrace", "MplseResult", "MpglsResult", "mplse", "mpgls", "mplse_batched",
    "mpgls_batched", "lse_direct", "gls_direct", "gmres_refine_lse", "gmres_refine_gls", "MixedlsError", "DimensionError", "InvalidInput", "SingularTriangular",
    "CudaError", "Unsupported", "lib", "lib_path",
]
