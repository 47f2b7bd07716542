"""C-ABI boundary tests that need no GPU: the library loads, exports every
symbol the public headers declare, validates arguments exactly where the
reference throws (lse.hpp:27-34, gls.hpp:26-32, precision.hpp:63-70,
refine.hpp:33-37), and fails loudly -- never falls back -- without a device."""
import ctypes as C
import glob
import os
import re

import numpy as np
import pytest

import paper_2406_16499_b200 as P
from paper_2406_16499_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(mlsb_\w+)\s*\(", src))
    return sorted(names)


def test_headers_declare_the_drop_in_entry_points():
    syms = declared_symbols()
    for s in ("mlsb_mplse", "mlsb_mpgls", "mlsb_mplse_batched", "mlsb_mpgls_batched",
              "mlsb_default_config", "mlsb_last_error"):
        assert s in syms


@pytest.mark.parametrize("sym", declared_symbols())
def test_library_exports_declared_symbol(sym):
    lib = C.CDLL(_capi.lib_path)
    assert getattr(lib, sym) is not None


def test_default_config_matches_reference_defaults():
    c = _capi.lib.mlsb_default_config()
    # refinement_config {tol = 1e-13, maxit = 40, classical (s, s, d, d)} (refine.hpp:28-31)
    assert (c.tol, c.maxit, c.u_f, c.u_s, c.u, c.u_r) == (1e-13, 40, 0, 0, 1, 1)


def _lse(m=6, n=4, p=2):
    rng = np.random.default_rng(0)
    return P.LseProblem(rng.standard_normal((m, n)), rng.standard_normal((p, n)),
                        rng.standard_normal(m), rng.standard_normal(p))


@pytest.mark.parametrize("shape", [(6, 4, 5), (2, 7, 3), (0, 4, 2)])
def test_lse_dimension_errors(shape):
    m, n, p = shape
    with pytest.raises(P.DimensionError):
        P.mplse(_lse(m, n, p))


@pytest.mark.parametrize("shape", [(4, 5, 2), (9, 3, 4)])
def test_gls_dimension_errors(shape):
    n, m, p = shape
    rng = np.random.default_rng(1)
    with pytest.raises(P.DimensionError):
        P.mpgls(P.GlsProblem(rng.standard_normal((n, m)), rng.standard_normal((n, p)),
                             rng.standard_normal(n)))


@pytest.mark.parametrize("cfg", [
    dict(tol=0.0), dict(tol=float("nan")), dict(maxit=0),
    dict(precisions=P.PrecisionConfig("working", "low")),            # u_f < u_s
    dict(precisions=P.PrecisionConfig("low", "low", "low")),         # working != binary64
    dict(precisions=P.PrecisionConfig("low", "extended")),           # u_s < u
    dict(precisions=P.PrecisionConfig("low", "low", "working", "low")),  # u < u_r violated
])
def test_config_validation(cfg):
    with pytest.raises(P.InvalidInput):
        P.mplse(_lse(), P.RefinementConfig(**cfg))


def test_rhs_length_mismatch():
    pb = _lse()
    pb.b = pb.b[:-1]
    with pytest.raises(P.DimensionError):
        P.mplse(pb)


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(P.CudaError):
        P.mplse(_lse())
    with pytest.raises(P.CudaError):
        P.mplse_batched(np.zeros((2, 6, 4)), np.ones((2, 2, 4)), np.zeros((2, 6)), np.zeros((2, 2)))


def test_batched_validation_before_device():
    with pytest.raises(P.DimensionError):
        P.mplse_batched(np.zeros((2, 6, 4)), np.ones((3, 2, 4)), np.zeros((2, 6)), np.zeros((2, 2)))
    with pytest.raises(P.InvalidInput):
        P.mplse_batched(np.zeros((2, 6, 4)), np.ones((2, 2, 4)), np.zeros((2, 6)), np.zeros((2, 2)),
                        P.RefinementConfig(maxit=0))


def test_product_never_imports_the_oracle():
    import ast

    for f in glob.glob(os.path.join(ROOT, "paper_2406_16499_b200", "**", "*.py"), recursive=True):
        tree = ast.parse(open(f).read())
        for node in ast.walk(tree):
            if isinstance(node, (ast.Import, ast.ImportFrom)):
                mod = getattr(node, "module", None) or ""
                names = [a.name for a in node.names]
                assert not mod.startswith("oracle") and not any(n.startswith("oracle") for n in names), f
    for f in glob.glob(os.path.join(ROOT, "paper_2406_16499_b200", "csrc", "*")):
        assert "orc_" not in open(f, errors="ignore").read(), f
