"""Experiment harness and on-disk formats (inc/io.hpp,
inc/metrics.hpp, inc/experiment.hpp).  CPU tests: number format against the
C++ standard library's std::to_chars (compiled here), Matrix Market round
trips and errors, the report schema; GPU test: run_experiment on config C1."""
import io
import json
import math
import os
import shutil
import subprocess
import tempfile

import numpy as np
import pytest

from paper_2406_16499_b200 import harness as H

VALUES = [0.1, 100000.0, 123456.0, 1e-5, 0.001, 1.5, 1e16, 2.5e-7, 1234.5, 1e22, -0.0, 0.0,
          5e-324, 1.7976931348623157e308, 123.0, 1000.0, 10000.0, -3.25, 1e-300, 6.02214076e23,
          0.30000000000000004, 2.0 ** -1074, 9007199254740993.0, 1e21, 1e-7, 12345678.9]


def test_shortest_double_matches_to_chars():
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("no C++ compiler")
    rng = np.random.default_rng(0)
    vals = VALUES + list(rng.standard_normal(200) * 10.0 ** rng.integers(-30, 30, 200))
    src = r"""
#include <charconv>
#include <cstdio>
#include <cstdlib>
int main(int argc, char** argv) {
  double v;
  while (std::scanf("%la", &v) == 1) {
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof(buf), v);
    *r.ptr = 0;
    std::puts(buf);
  }
}
"""
    with tempfile.TemporaryDirectory() as td:
        cpp, exe = os.path.join(td, "t.cpp"), os.path.join(td, "t")
        open(cpp, "w").write(src)
        subprocess.run([gxx, "-std=c++17", "-O1", cpp, "-o", exe], check=True)
        out = subprocess.run([exe], input="\n".join(float(v).hex() for v in vals),
                             capture_output=True, text=True, check=True).stdout.split()
    assert [H.shortest_double(v) for v in vals] == out


def test_matrix_market_round_trip():
    rng = np.random.default_rng(1)
    M = rng.standard_normal((7, 3)) * 10.0 ** rng.integers(-20, 20, (7, 3))
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "m.mtx")
        H.write_matrix_market(M, path)
        lines = open(path).read().split("\n")
        assert lines[0] == "%%MatrixMarket matrix array real general"
        assert lines[1] == "7 3"
        assert lines[2] == H.shortest_double(M[0, 0]) and lines[3] == H.shortest_double(M[1, 0])
        assert np.array_equal(H.read_matrix_market(path), M)  # column-major, exact


def test_matrix_market_comments_and_errors():
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "a.mtx")
        open(p, "w").write("%%MatrixMarket matrix array real general\n% c1\n%c2\n2 2\n1\n2\n3\n4\n")
        assert np.array_equal(H.read_matrix_market(p), np.array([[1.0, 3.0], [2.0, 4.0]]))
        open(p, "w").write("%%MatrixMarket matrix coordinate real general\n2 2\n")
        with pytest.raises(H.ParseError) as e:
            H.read_matrix_market(p)
        assert e.value.line == 1
        open(p, "w").write("%%MatrixMarket matrix array real general\n2 x\n")
        with pytest.raises(H.ParseError) as e:
            H.read_matrix_market(p)
        assert e.value.line == 2
        open(p, "w").write("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n")
        with pytest.raises(H.ParseError):
            H.read_matrix_market(p)
        open(p, "w").write("")
        with pytest.raises(H.ParseError) as e:
            H.read_matrix_market(p)
        assert e.value.line == 1


def test_report_schema():
    spec = H.GeneratorSpec("lse", 200, 100, 50, 1e3, 1)
    r = H.ExperimentReport(spec, "ir", 1.5e-17, 0.0, 3, 0, "converged")
    j = r.to_json()
    assert list(j) == ["kind", "m", "n", "p", "cond", "seed", "distribution", "method", "metric1",
                       "metric2", "iterations", "inner_iterations", "status", "timings"]
    assert list(j["timings"]) == ["factorization", "init", "residual", "correction", "gmres",
                                  "other"]
    buf = io.StringIO()
    H.write_reports([r, r], "csv", buf)
    rows = buf.getvalue().strip().split("\n")
    assert rows[0] == H.CSV_HEADER and len(rows) == 3
    assert rows[1].startswith("lse,200,100,50,1000,1,geometric,ir,1.5e-17,0,3,0,converged,")
    buf = io.StringIO()
    H.write_reports([r], "json", buf)
    assert json.loads(buf.getvalue())[0]["status"] == "converged"


def test_csv_header_matches_reference():
    path = "/root/reference/proj/include/mixedls/io.hpp"
    if not os.path.exists(path):
        pytest.skip("reference sources not present")
    src = open(path).read()
    i = src.index("report_csv_header =")
    parts = src[i:src.index(";", i)].split('"')[1::2]
    assert "".join(parts) == H.CSV_HEADER


def test_metrics_definitions():
    rng = np.random.default_rng(2)
    A, B = rng.standard_normal((6, 4)), rng.standard_normal((2, 4))
    b, d, x = rng.standard_normal(6), rng.standard_normal(2), rng.standard_normal(4)
    e1 = np.linalg.norm(B @ x - d) / (np.linalg.norm(B) * np.linalg.norm(x) + np.linalg.norm(d))
    assert math.isclose(H.metric_err1_lse(A, B, b, d, x), e1, rel_tol=1e-14)
    assert H.metric_err2_lse(A, b, x, x) == 0.0
    assert H.metric_er2_gls(np.zeros(3), np.zeros(3)) == 0.0
    assert H.metric_er2_gls(np.ones(3), np.zeros(3)) == math.inf


@pytest.mark.gpu
def test_run_experiment_c1(gpu):
    from paper_2406_16499_b200 import generate as G

    A, B, b, d = G.lse_problem(200, 100, 50, 1e3, 1e2, 1)
    spec = H.GeneratorSpec("lse", 200, 100, 50, 1e3, 1)
    pb = gpu.LseProblem(A, B, b, d)
    cfg = gpu.RefinementConfig(maxit=10, precisions=gpu.PrecisionConfig("low", "working"))
    rd = H.run_experiment(pb, spec, "direct")
    ri = H.run_experiment(pb, spec, "ir", cfg)
    rg = H.run_experiment(pb, spec, "gmres-bd", cfg)
    assert rd.status == "converged" and rd.metric1 < 1e-14 and rd.metric2 == 0.0
    assert ri.status == "converged" and 1 <= ri.iterations <= 10
    assert ri.metric1 < 1e-13 and ri.metric2 < 1e-10
    assert rg.status == "converged" and rg.inner_iterations >= 1 and rg.metric2 < 1e-10
    rgl = H.run_experiment(pb, spec, "gmres-left", cfg)
    assert rgl.status == "converged" and rgl.inner_iterations >= 1
    W, V, dg = G.gls_problem(200, 100, 150, 1e4, 1e2, 2)
    rgls = H.run_experiment(gpu.GlsProblem(W, V, dg), H.GeneratorSpec("gls", 100, 200, 150, 1e4, 2),
                            "ir", gpu.RefinementConfig(maxit=10))
    assert rgls.status == "converged" and rgls.metric1 < 1e-13 and rgls.metric2 < 1e-10
    rgg = H.run_experiment(gpu.GlsProblem(W, V, dg), H.GeneratorSpec("gls", 100, 200, 150, 1e4, 2),
                           "gmres-bd", gpu.RefinementConfig(maxit=10))
    assert rgg.status == "converged" and rgg.inner_iterations >= 1 and rgg.metric2 < 1e-10
