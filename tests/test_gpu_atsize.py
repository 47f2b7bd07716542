"""Parity at the BASELINE configurations' full sizes (SURVEY.md §8 legend):

* C3 -- LSE 8192x4096/1024, kappa_A in {1e2, 1e4, 1e6}, kappa_B 1e2, (s,s,d,d),
  against the unmodified reference (oracle/_ref; mplse, inc/lse.hpp:303-429).
  The three reference solves (~2 min each on one core) run concurrently in
  threads (ctypes releases the GIL) while the GPU solves.
* C5 -- complex GLS n=4096, m=2048, p=3072, kappa_W 1e6, kappa_V 1e3 against
  the complex restatement (oracle port; the reference is real-only).
* C4 -- all 65,536 problems of the batch against oracle/_ref on every host
  thread: status, passes +-1, forward error <= 40 (m+n+p+1) u kappa_i.

Bar (tests/helpers.py): forward error <= 40 N u kappa, passes
within 1, final backward error within 2x of the oracle's, same status.
"""
import os
import threading

import numpy as np
import pytest

from paper_2406_16499_b200 import generate as G
from tests.helpers import U53, check_parity, fwd_bound, gls_backward, lse_backward, rel

pytestmark = pytest.mark.gpu


def _cfg(P, c):
    return P.RefinementConfig(maxit=c["maxit"], precisions=P.PrecisionConfig(c["prec"][0], c["prec"][1]))


def _run_threads(jobs):
    out = {}

    def work(key, fn):
        try:
            out[key] = fn()
        except Exception as exc:  # noqa: BLE001
            out[key] = exc

    ths = [threading.Thread(target=work, args=kv) for kv in jobs.items()]
    for t in ths:
        t.start()
    return ths, out


def test_c3_kappa_sweep_vs_reference(gpu, ref):
    P = gpu
    c = G.CONFIGS["C3"]
    m, n, p = c["m"], c["n"], c["p"]
    probs = {k: G.lse_problem(m, n, p, k, c["kappa_B"], c["seed"]) for k in c["kappa_sweep"]}
    ths, refs = _run_threads({k: (lambda pr=pr: ref.mplse(*pr, maxit=c["maxit"], prec=("s", "s", "d")))
                              for k, pr in probs.items()})
    gpu_res = {k: P.mplse(P.LseProblem(*pr), _cfg(P, c)) for k, pr in probs.items()}
    for t in ths:
        t.join()
    fails = []
    for k, (A, B, b, d) in probs.items():
        res, rr = gpu_res[k], refs[k]
        assert not isinstance(rr, Exception), rr
        st = res.state
        msgs = check_parity(f"C3 kappa {k:.0e}", rel(st.x, rr.x), fwd_bound(m, n, p, k),
                            res.trace.iterations, rr.iterations,
                            lse_backward(A, B, b, d, st.x, st.r, st.v),
                            lse_backward(A, B, b, d, rr.x, rr.r, rr.v), res.trace.status, rr.status)
        if res.trace.status != rr.status:
            msgs.append(f"C3 kappa {k:.0e}: status {res.trace.status} vs {rr.status}")
        # the per-phase trace is split like the reference's (refine.hpp:45-52)
        tm = res.trace.timing
        corrections = res.trace.iterations - (1 if res.trace.status == "converged" else 0)
        if corrections > 0 and not tm["correction"] > 0:
            msgs.append(f"C3 kappa {k:.0e}: correction phase not timed ({tm})")
        if not tm["residual"] > 0 or tm["gmres"] != 0:
            msgs.append(f"C3 kappa {k:.0e}: bad phase split ({tm})")
        fails += msgs
    assert not fails, fails


def test_c5_complex_gls_vs_port(gpu, port):
    P = gpu
    c = G.CONFIGS["C5"]
    n, m, p = c["n"], c["m"], c["p"]
    W, V, d = G.gls_problem(n, m, p, c["kappa_A"], c["kappa_B"], c["seed"], cplx=True)
    ths, refs = _run_threads({"c5": lambda: port.mpgls(W, V, d, maxit=c["maxit"], prec=("s", "s", "d"),
                                                       cplx=True)})
    res = P.mpgls(P.GlsProblem(W, V, d), _cfg(P, c))
    for t in ths:
        t.join()
    rr = refs["c5"]
    assert not isinstance(rr, Exception), rr
    st = res.state
    fwd = max(rel(st.x, rr.x), rel(st.y, rr.r))
    msgs = check_parity("C5", fwd, fwd_bound(n, m, p, c["kappa_A"]), res.trace.iterations,
                        rr.iterations, gls_backward(W, V, d, st.x, st.y, st.z),
                        gls_backward(W, V, d, rr.x, rr.r, rr.v), res.trace.status, rr.status)
    assert res.trace.status == rr.status
    assert not msgs, msgs


def test_c4_full_batch_vs_reference(gpu, ref):
    """Every one of the 65,536 C4 problems (the bench's batch, same seeds)."""
    import torch

    P = gpu
    c = G.CONFIGS["C4"]
    bt, m, n, p = c["batch"], c["m"], c["n"], c["p"]
    A, B, b, d, kA = G.lse_batch_torch(bt, m, n, p, seed=c["seed"], device="cuda")
    out = P.mplse_batched(A, B, b, d, P.RefinementConfig())
    torch.cuda.synchronize()
    x = out.x.cpu().numpy()
    it = out.iterations.cpu().numpy()
    st = out.status.cpu().numpy()
    assert not out.errcode.cpu().numpy().any()
    An, Bn = A.cpu().numpy(), B.cpu().numpy()
    del A, B
    torch.cuda.empty_cache()
    xr, rr, vr, st_r, it_r, err_r = ref.mplse_batch(An, Bn, b.cpu().numpy(), d.cpu().numpy(), maxit=40,
                                                    prec=("s", "s", "d"),
                                                    nthreads=len(os.sched_getaffinity(0)))
    assert not err_r.any()
    fwd = np.linalg.norm(x - xr, axis=1) / np.linalg.norm(xr, axis=1)
    bound = 40.0 * (m + n + p + 1) * U53 * kA.cpu().numpy()
    bad = np.flatnonzero(~(fwd <= bound))
    assert bad.size == 0, (bad[:10], (fwd / bound)[bad[:10]])
    assert np.abs(it.astype(np.int64) - it_r).max() <= 1
    assert np.array_equal(st, st_r)


def test_c3_gmres_ir_kappa_1e6_vs_reference(gpu, ref):
    """GMRES-IR with the block-diagonal split preconditioner (gmres_refine_lse,
    inc/krylov.hpp:545-689) at the C3 shape and kappa_A 1e6 -- where it is the
    rescue for classical IR -- against the unmodified
    reference: same status, outer passes within 1, forward error bound."""
    P = gpu
    c = G.CONFIGS["C3"]
    m, n, p = c["m"], c["n"], c["p"]
    A, B, b, d = G.lse_problem(m, n, p, 1e6, c["kappa_B"], c["seed"])
    ths, refs = _run_threads({"g": lambda: ref.gmres_lse(A, B, b, d, maxit=c["maxit"], prec=("s", "s", "d"),
                                                         precond="bd_split")})
    res = P.gmres_refine_lse(P.LseProblem(A, B, b, d), P.RefinementConfig(maxit=c["maxit"]),
                             precond="bd_split")
    for t in ths:
        t.join()
    rr = refs["g"]
    assert not isinstance(rr, Exception), rr
    assert res.trace.status == rr.status == "converged"
    assert abs(res.trace.iterations - rr.iterations) <= 1, (res.trace.iterations, rr.iterations)
    assert rel(res.state.x, rr.x) <= fwd_bound(m, n, p, 1e6)
    assert res.trace.timing["gmres"] > 0 and res.trace.timing["correction"] == 0
