"""Experiment harness and on-disk formats of the reference,
host side, around the GPU solvers.

* ``run_experiment`` mirrors ``mixedls::run_experiment`` (inc/experiment.hpp:80-160):
  binary64 direct reference on the GPU (``lse_direct`` / ``gls_direct``), the
  requested method on the GPU, the err-1/err-2 (LSE) or er-1/er-2 (GLS)
  metrics (inc/metrics.hpp:23-56) in binary64 on the host.  Solver failures are
  captured in ``status``, never raised (experiment.hpp:155-160).
* Matrix Market dense array files (inc/io.hpp:32-75) and the JSON / CSV report
  schema (inc/io.hpp:77-142), with the reference's shortest round-trip number
  format (``std::to_chars`` without a format: shortest digits, the shorter of
  fixed / scientific, fixed on a tie).

Methods: ``"direct"``, ``"ir"`` (classical IR, mplse / mpgls) and, for LSE,
``"gmres-left"`` / ``"gmres-bd"`` (GMRES-IR, gmres_refine_lse / gmres_refine_gls,
inc/krylov.hpp:545-784), for LSE and GLS.
"""
from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import api
from ._capi import MixedlsError

METHODS = ("direct", "ir", "gmres-left", "gmres-bd")
CSV_HEADER = ("kind,m,n,p,cond,seed,distribution,method,metric1,metric2,iterations,"
              "inner_iterations,status,factorization,init,residual,correction,gmres,other")


# ------------------------------------------------------------------ numbers
def shortest_double(v: float) -> str:
    """std::to_chars(double) without a format (io.hpp:22-27): the shortest
    round-trip digits, printed as %f or %e, whichever is shorter (f on a tie)."""
    v = float(v)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    if v == 0.0:
        return "-0" if math.copysign(1.0, v) < 0 else "0"
    sign = "-" if v < 0 else ""
    r = repr(abs(v))  # shortest round-trip digits
    mant, _, exp = r.partition("e")
    e = int(exp) if exp else 0
    ip, _, fp = mant.partition(".")
    digits = (ip + fp).lstrip("0")
    # decimal exponent of the first significant digit
    if ip.strip("0"):
        point = len(ip.lstrip("0")) + e
    else:
        point = -(len(fp) - len(fp.lstrip("0"))) + e
    digits = digits.rstrip("0") or "0"
    # scientific: d[.ddd]e±XX (at least two exponent digits)
    se = point - 1
    sci = digits[0] + ("." + digits[1:] if len(digits) > 1 else "") + \
        ("e-" if se < 0 else "e+") + f"{abs(se):02d}"
    # fixed
    if point <= 0:
        fix = "0." + "0" * (-point) + digits
    elif point >= len(digits):
        # integer-valued: %f prints the exact integer (e.g. ...416, not ...420)
        fix = str(int(abs(v)))
    else:
        fix = digits[:point] + "." + digits[point:]
    return sign + (fix if len(fix) <= len(sci) else sci)


# ------------------------------------------------------------ Matrix Market
class ParseError(MixedlsError):
    def __init__(self, msg: str, line: int):
        super().__init__(f"{msg} (line {line})")
        self.line = line


def write_matrix_market(M, path: str) -> None:
    """'%%MatrixMarket matrix array real general', column-major (io.hpp:32-40)."""
    M = np.asarray(M, dtype=np.float64)
    if M.ndim != 2:
        raise ValueError("write_matrix_market: 2-D array expected")
    with open(path, "w") as out:
        out.write("%%MatrixMarket matrix array real general\n")
        out.write(f"{M.shape[0]} {M.shape[1]}\n")
        for v in M.reshape(-1, order="F"):
            out.write(shortest_double(v) + "\n")


def read_matrix_market(path: str) -> np.ndarray:
    """Dense real general array files (io.hpp:42-75), same errors and line numbers."""
    with open(path) as fh:
        lines = fh.read().split("\n")
    if not lines or (len(lines) == 1 and not lines[0]):
        raise ParseError("read_matrix_market: empty file", 1)
    head = lines[0].split()
    if head[:5] != ["%%MatrixMarket", "matrix", "array", "real", "general"]:
        raise ParseError(f"read_matrix_market: unsupported header '{lines[0]}'", 1)
    k = 1
    while True:
        if k >= len(lines):
            raise ParseError("read_matrix_market: missing size line", k)
        line = lines[k]
        k += 1
        if not (line and line[0] == "%"):
            break
    try:
        tok = line.split()
        rows, cols = int(tok[0]), int(tok[1])
        if rows <= 0 or cols <= 0:
            raise ValueError
    except (ValueError, IndexError):
        raise ParseError(f"read_matrix_market: bad size line '{line}'", k) from None
    size_line = k
    vals = " ".join(lines[k:]).split()
    if len(vals) < rows * cols:
        raise ParseError("read_matrix_market: bad or missing value", size_line + len(vals) + 1)
    out = np.empty(rows * cols)
    for q in range(rows * cols):
        try:
            out[q] = float(vals[q])
        except ValueError:
            raise ParseError("read_matrix_market: bad or missing value", size_line + q + 1) from None
    return out.reshape((rows, cols), order="F")


# ------------------------------------------------------------------ metrics
def _safe_ratio(num, den):
    return num / den if den > 0 else (0.0 if num == 0 else math.inf)


def metric_err1_lse(A, B, b, d, x):
    """err-1 = ||B x - d|| / (||B||_F ||x|| + ||d||)   (metrics.hpp:23-29)"""
    return _safe_ratio(np.linalg.norm(B @ x - d),
                       np.linalg.norm(B) * np.linalg.norm(x) + np.linalg.norm(d))


def metric_err2_lse(A, b, x, x_ref):
    """err-2 = | ||A x - b|| / ||A x_ref - b|| - 1 |   (metrics.hpp:31-43)"""
    num = float(np.sum((A @ x - b) ** 2))
    den = float(np.sum((A @ x_ref - b) ** 2))
    if den == 0.0:
        return 0.0 if num == 0.0 else math.inf
    return abs(math.sqrt(num / den) - 1.0)


def metric_er1_gls(W, V, d, x, y):
    """er-1 = ||W x + V y - d|| / (||W||_F ||x|| + ||V||_F ||y|| + ||d||)"""
    return _safe_ratio(np.linalg.norm(W @ x + V @ y - d),
                       np.linalg.norm(W) * np.linalg.norm(x) + np.linalg.norm(V) * np.linalg.norm(y)
                       + np.linalg.norm(d))


def metric_er2_gls(y, y_ref):
    """er-2 = | ||y|| / ||y_ref|| - 1 |"""
    den = np.linalg.norm(y_ref)
    if den == 0.0:
        return 0.0 if np.linalg.norm(y) == 0.0 else math.inf
    return abs(np.linalg.norm(y) / den - 1.0)


# ------------------------------------------------------------------ reports
@dataclass
class GeneratorSpec:
    """Describes where a problem came from (generator_spec, inc/generate.hpp)."""
    kind: str  # "lse" | "gls"
    m: int
    n: int
    p: int
    cond: float = 1.0
    seed: int = 0
    distribution: str = "geometric"


@dataclass
class ExperimentReport:
    spec: GeneratorSpec
    method: str = "direct"
    metric1: float = 0.0
    metric2: float = 0.0
    iterations: int = 0
    inner_iterations: int = 0
    status: str = "converged"
    timing: dict = field(default_factory=lambda: {k: 0.0 for k in (
        "factorization", "init", "residual", "correction", "gmres", "other")})

    def to_json(self) -> dict:
        """report_to_json (io.hpp:77-96): same keys, same order."""
        s = self.spec
        return {"kind": s.kind, "m": s.m, "n": s.n, "p": s.p, "cond": s.cond, "seed": s.seed,
                "distribution": s.distribution, "method": self.method, "metric1": self.metric1,
                "metric2": self.metric2, "iterations": self.iterations,
                "inner_iterations": self.inner_iterations, "status": self.status,
                "timings": {k: self.timing[k] for k in (
                    "factorization", "init", "residual", "correction", "gmres", "other")}}

    def to_csv_row(self) -> str:
        """report_to_csv_row (io.hpp:108-125)."""
        s, t = self.spec, self.timing
        f = shortest_double
        return ",".join([s.kind, str(s.m), str(s.n), str(s.p), f(s.cond), str(s.seed),
                         s.distribution, self.method, f(self.metric1), f(self.metric2),
                         str(self.iterations), str(self.inner_iterations), self.status,
                         f(t["factorization"]), f(t["init"]), f(t["residual"]),
                         f(t["correction"]), f(t["gmres"]), f(t["other"])])


def write_reports(reports, fmt: str, out) -> None:
    """write_reports (io.hpp:129-142): JSON array (indent 2) or CSV with header."""
    if fmt == "json":
        out.write(json.dumps([r.to_json() for r in reports], indent=2) + "\n")
    elif fmt == "csv":
        out.write(CSV_HEADER + "\n")
        for r in reports:
            out.write(r.to_csv_row() + "\n")
    else:
        raise ValueError("write_reports: format must be 'json' or 'csv'")


# --------------------------------------------------------------- experiment
def run_experiment(problem, spec: GeneratorSpec, method: str,
                   cfg: api.RefinementConfig | None = None) -> ExperimentReport:
    """run_experiment (experiment.hpp:80-160) for a given LseProblem / GlsProblem."""
    if method not in METHODS:
        raise ValueError(f"run_experiment: unknown method '{method}'")
    cfg = cfg or api.RefinementConfig()
    rep = ExperimentReport(spec=spec, method=method)
    t0 = time.perf_counter()
    lse = isinstance(problem, api.LseProblem)
    try:
        tf = time.perf_counter()
        ref = api.lse_direct(problem) if lse else api.gls_direct(problem)
        t_ref = time.perf_counter() - tf
        if method == "direct":
            st = ref
            rep.timing["factorization"] = t_ref  # factor + solve, device-synchronous
        elif method == "ir":
            res = api.mplse(problem, cfg) if lse else api.mpgls(problem, cfg)
            st = res.state
            rep.status = res.trace.status
            rep.iterations = res.trace.iterations
            rep.timing.update({k: float(res.trace.timing.get(k, 0.0)) for k in rep.timing})
        else:
            gm = api.gmres_refine_lse if lse else api.gmres_refine_gls
            res = gm(problem, cfg, precond="left" if method == "gmres-left" else "bd_split")
            st = res.state
            rep.status = res.trace.status
            rep.iterations = res.trace.iterations
            rep.inner_iterations = res.trace.inner_iterations
            rep.timing.update({k: float(res.trace.timing.get(k, 0.0)) for k in rep.timing})
        if lse:
            A, B, b, d = (np.asarray(t) for t in (problem.A, problem.B, problem.b, problem.d))
            rep.metric1 = metric_err1_lse(A, B, b, d, np.asarray(st.x))
            rep.metric2 = metric_err2_lse(A, b, np.asarray(st.x), np.asarray(ref.x))
        else:
            W, V, d = (np.asarray(t) for t in (problem.W, problem.V, problem.d))
            rep.metric1 = metric_er1_gls(W, V, d, np.asarray(st.x), np.asarray(st.y))
            rep.metric2 = metric_er2_gls(np.asarray(st.y), np.asarray(ref.y))
    except MixedlsError:
        # experiment.hpp:155-160: failures are reported, not thrown
        rep.status = "diverged"
        rep.metric1 = rep.metric2 = math.inf
    rep.timing["other"] += max(0.0, time.perf_counter() - t0 - sum(rep.timing.values()))
    return rep
