"""The reference user's own program (tests/dropin_demo.cpp, built against the
unmodified reference headers + include/mixedls_b200.hpp) solving the same
problems on the CPU reference and on the B200 through the shim."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "oracle", "_ref", "b200_dropin_demo")


@pytest.mark.gpu
def test_reference_program_through_shim(gpu):
    if not os.path.exists(DEMO):
        pytest.skip("drop-in demo not built (needs /root/reference at build time)")
    out = subprocess.run([DEMO], capture_output=True, text=True, timeout=120).stdout
    lse = re.search(r"LSE ref_iters (\d+) gpu_iters (\d+) ref_status (\w+) gpu_status (\w+) relx (\S+)", out)
    gls = re.search(r"GLS ref_iters (\d+) gpu_iters (\d+) ref_status (\w+) gpu_status (\w+) relx (\S+) rely (\S+)", out)
    assert lse and gls, out
    assert abs(int(lse[1]) - int(lse[2])) <= 1 and lse[3] == lse[4] == "converged"
    assert float(lse[5]) <= 40 * 351 * 2.0 ** -53 * 1e3 * 10
    assert abs(int(gls[1]) - int(gls[2])) <= 1 and gls[3] == gls[4] == "converged"
    assert float(gls[5]) <= 1e-9 and float(gls[6]) <= 1e-9
    assert "EXC dimension_error" in out
    dr = re.search(r"DIRECT relx (\S+) relr (\S+)", out)
    assert dr and float(dr[1]) <= 1e-9 and float(dr[2]) <= 1e-9, out
    gm = re.findall(r"GMRES-(LSE|GLS) (\d) ref_iters (\d+) gpu_iters (\d+) ref_status (\w+) gpu_status (\w+) relx (\S+)", out)
    assert len(gm) == 4, out
    for kind, _, ri, gi, rs, gs, rx in gm:
        assert rs == gs == "converged" and abs(int(ri) - int(gi)) <= 1, (kind, ri, gi, rs, gs)
        assert float(rx) <= 1e-9, (kind, rx)


def test_dropin_demo_exception_path_without_gpu():
    """Off the GPU the shim still validates with the reference's own checks."""
    import torch

    if not os.path.exists(DEMO) or torch.cuda.is_available():
        pytest.skip("needs the built demo and no GPU")
    r = subprocess.run([DEMO], capture_output=True, text=True, timeout=120)
    # the first GPU call raises mixedls::error (no device) -> non-zero exit
    assert r.returncode != 0


HARN_GPU = os.path.join(ROOT, "oracle", "_ref", "b200_harness")
HARN_REF = os.path.join(ROOT, "oracle", "_ref", "ref_harness")
# m + n + p + 1 of the desk-scale sweep shapes (inc/experiment.hpp:220-260):
# LSE (2048, 256, 8), GLS (1024, 32, 1152)
DESK_N = {"lse": 2048 + 256 + 8 + 1, "gls": 1024 + 32 + 1152 + 1}
CELL = re.compile(r"CELL (\d+) kind (\w+) cond (\S+) method (\S+) status (\w+) iters (\d+) inner (\d+) m1 (\S+) m2 (\S+)")


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["lse", "gls"])
def test_reference_run_sweep_routed_to_b200(gpu, kind):
    """The reference's own run_experiment / run_sweep (unmodified
    inc/experiment.hpp, desk-scale paper_sweep_cells) with its IR and GMRES-IR
    calls routed to the B200 library (tests/harness_b200.cpp), against the same
    sweep on the plain reference: same status per cell, outer passes within 1,
    err-1 / err-2 (er-1 / er-2) of converged cells within 10x."""
    if not (os.path.exists(HARN_GPU) and os.path.exists(HARN_REF)):
        pytest.skip("harness not built (needs /root/reference at build time)")
    env = dict(os.environ, MIXEDLS_THREADS="1")  # one GPU: cells in order
    g = subprocess.run([HARN_GPU, kind], capture_output=True, text=True, timeout=600, env=env)
    r = subprocess.run([HARN_REF, kind], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, MIXEDLS_THREADS=str(os.cpu_count() or 1)))
    assert g.returncode == 0 and r.returncode == 0, (g.stderr, r.stderr)
    gc, rc = CELL.findall(g.stdout), CELL.findall(r.stdout)
    assert len(gc) == len(rc) > 0, (g.stdout, r.stdout)
    bad = []
    for a, b in zip(gc, rc):
        if a[:4] != b[:4]:
            bad.append(("cell mismatch", a, b))
            continue
        st_g, st_r, it_g, it_r = a[4], b[4], int(a[5]), int(b[5])
        if a[3] == "ir" and float(a[2]) * 2.0 ** -24 >= 0.1:
            # kappa * u_f >~ 1 (cond >= 1e7 with binary32 factors): classical IR
            # is outside its convergence theory and the pass count is rounding
            # noise (the reference takes 38 passes at seed 7, proj/test_output.txt:
            # 38, and 40+ at this seed).  Required: no worse than the reference.
            if st_g not in (st_r, "converged"):
                bad.append(("boundary status", a, b))
            elif st_g == "converged" and st_r == "converged" and it_g > it_r + 1:
                bad.append(("boundary passes", a, b))
            elif not float(a[7]) <= max(10 * float(b[7]), 1e-12):
                bad.append(("boundary metric", a, b))
            continue
        if st_g != st_r or abs(it_g - it_r) > 1:
            bad.append((a, b))
            continue
        if st_g == "converged":
            # m1 (err-1 / er-1, a backward-type error): within 10x of the
            # reference.  m2 (err-2 / er-2) is the forward error against the
            # binary64 direct solution: the parity bar of north_star,
            # c * N * u_r * kappa (tests/helpers.py), or within 10x -- a run that
            # stops one pass earlier (both below tol) legitimately ends with a
            # forward error many times the other run's at kappa >= 1e5
            cond = float(a[2])
            fwd_bound = 40 * DESK_N[kind] * 2.0 ** -53 * cond
            if not float(a[7]) <= max(10 * float(b[7]), 1e-12):
                bad.append(("metric", 7, a, b))
            if not float(a[8]) <= max(10 * float(b[8]), fwd_bound, 1e-12):
                bad.append(("metric", 8, a, b))
    assert not bad, bad
