#!/usr/bin/env python
"""Benchmark of the B200 classical-IR hot path (BASELINE.json metric).

Default workload (N=1): BASELINE config 4 -- 65,536 independent LSE problems
(A 256x128, B 32x128, kappa(A) = 10^U(1,5), kappa(B) = 10) at
(u_f, u_s, u, u_r) = (s, s, d, d), tol 1e-13, maxit 40 (reference defaults),
solved by ONE launch of the fused tile solver (one CTA per problem).  With
--gpus N (torchrun, one process per GPU) every rank solves its own 65,536
problems (weak scaling; independent problems, no collective on the data path).

A step = one pass of the hot path over the rank's whole batch with inputs
already resident in HBM (19.3 GB of fp64 A/B per GPU >> 126 MB L2, so no L2
flush is needed).  `e2e` re-times the same work through the C ABI with pinned
HOST buffers (H2D of inputs and D2H of x, r, v, status, iterations inside the
timed region).  `--impl reference` times the reference's own CPU
implementation (oracle/_ref, the unmodified reference headers) on all host
cores over a bounded sample of the same workload.

Other configs for ad-hoc runs: --config C1|C2 (single problems, latency).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "refined LSE/GLS solves/sec; GRQ/GQR GFLOP/s and residual GB/s vs B200 peak"
M, N, P = 256, 128, 32


def grq_flops(m, n, p):
    # GRQ(m,n,p) = (2p^2 n - 2/3 p^3) + (4mnp - 2mp^2) + (2mn^2 - 2/3 n^3)
    return (2 * p * p * n - 2 / 3 * p ** 3) + (4 * m * n * p - 2 * m * p * p) + (2 * m * n * n - 2 / 3 * n ** 3)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4", choices=["C4", "C1", "C2"])
    ap.add_argument("--batch", type=int, default=65536, help="problems per GPU (C4)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-large", action="store_true", help="skip the C3 large-path record")
    return ap.parse_args()


# ---------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()

    def summary(self):
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [num(r[1]) for r in rows if num(r[1])]
        load = [s for s in sm if s and s > 500] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": num(rows[0][2]), "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
def cpu_reference(A, B, b, d, seconds, maxit=40, prec=("s", "s", "d")):
    """Time the reference's CPU path (oracle/_ref = unmodified reference headers,
    else the bitwise-identical port) on a bounded sample with all host threads.
    A (S, m, n) ... host arrays.  Returns (solves/s, cores, kind, sample)."""
    from oracle.oracle import Oracle, available

    kind = "reference" if available("ref") else "port"
    orc = Oracle("ref" if kind == "reference" else "port")
    threads = len(os.sched_getaffinity(0)) if kind == "reference" else 1
    S = A.shape[0]
    # calibrate on a small slice, then size the sample for ~`seconds`
    k0 = min(S, max(8, 4 * threads))
    t0 = time.perf_counter()
    orc.mplse_batch(A[:k0], B[:k0], b[:k0], d[:k0], maxit=maxit, prec=prec, nthreads=threads)
    rate0 = k0 / max(time.perf_counter() - t0, 1e-6)
    k = int(min(S, max(k0, rate0 * seconds)))
    t0 = time.perf_counter()
    orc.mplse_batch(A[:k], B[:k], b[:k], d[:k], maxit=maxit, prec=prec, nthreads=threads)
    dt = time.perf_counter() - t0
    return k / dt, threads, kind, k, dt


def measured_traffic(batch):
    """DRAM bytes (read + write) per launch of the tile solver from the committed
    `ncu --set full` capture (profiles/c4_ncu_summary.json), scaled to `batch`
    problems; None when no capture is committed."""
    path = os.path.join(ROOT, "profiles", "c4_ncu_summary.json")
    try:
        with open(path) as fh:
            s = json.load(fh)
        return s["dram_bytes_per_problem"] * batch
    except (OSError, KeyError, ValueError):
        return None


def emit(obj):
    print(json.dumps(obj), flush=True)


def config_c4(batch, world):
    return {"workload": (f"C4 batched LSE: {batch} problems per GPU, A 256x128, B 32x128, "
                         "kappa(A)=10^U(1,5), kappa(B)=10, (u_f,u_s,u,u_r)=(s,s,d,d), "
                         "tol=1e-13, maxit=40"),
            "batch_per_gpu": batch, "m": M, "n": N, "p": P,
            "l2": "inputs 19.3 GB fp64 per GPU >> 126 MB L2; no flush needed",
            "parallelism": f"dp{world} (independent problems, no collective)"}


# ---------------------------------------------------------------------------
def run_reference(args, rank, world):
    import numpy as np

    if rank != 0:
        return
    from paper_2406_16499_b200 import generate as G

    # bounded sample of the C4 workload, generated on the host (same generator,
    # CPU RNG stream)
    S = 4096
    A, B, b, d, _ = G.lse_batch_torch(S, M, N, P, seed=1000, device="cpu")
    A, B, b, d = A.numpy(), B.numpy(), b.numpy(), d.numpy()
    vals = []
    info = None
    for step in range(args.warmup + args.steps):
        v, cores, kind, k, dt = cpu_reference(A, B, b, d, seconds=args.cpu_seconds / 2)
        if step >= args.warmup:
            vals.append(v)
            info = (cores, kind, k, dt)
    value = statistics.median(vals)
    cores, kind, k, dt = info
    emit({"impl": "reference", "metric": METRIC, "value": value, "unit": "solves/s",
          "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
          "ms_per_step": 1e3 * dt, "higher_is_better": True, "scaling": "weak",
          "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
          "config": config_c4(args.batch, world),
          "cpu_baseline": {"value": value, "unit": "solves/s", "cores": cores, "kind": kind,
                           "sample": f"{k} of the C4 problems per step (mplse per problem, "
                                     f"std::thread pool over {cores} host threads)"},
          "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0,
                  "d2h_bytes_per_step": 0}})


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_2406_16499_b200 as PK
    from paper_2406_16499_b200 import _capi
    from paper_2406_16499_b200 import generate as G

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    batch = args.batch
    A, B, b, d, kA = G.lse_batch_torch(batch, M, N, P, seed=1000 + rank, device=dev)
    torch.cuda.synchronize()
    cfg = PK.RefinementConfig()  # reference defaults: tol 1e-13, maxit 40, (s,s,d,d)

    def step():
        return PK.mplse_batched(A, B, b, d, cfg, stream=stream)

    for _ in range(args.warmup):
        out = step()
    torch.cuda.synchronize()
    lib = _capi.lib
    fp32_peak = lib.mlsb_fp32_fma_peak_tflops
    fp32_peak.restype = C.c_double
    fp64_peak = lib.mlsb_fp64_fma_peak_tflops
    fp64_peak.restype = C.c_double
    peak32 = fp32_peak(-1, None)
    peak64 = fp64_peak(-1, None)

    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local_rank) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            out = step()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    value = world * batch * args.steps / (ms_max * 1e-3)
    clocks = clk.summary()

    iters = out.iterations.cpu().numpy()
    status = out.status.cpu().numpy()
    err = out.errcode.cpu().numpy()
    elem = (M * N + P * N) * 8
    # fp64 sweeps per problem: max-abs scan, scaled cast, A^T r (solve_v), one residual per pass
    sweeps = 3 + iters.astype(np.float64)
    alg_bytes = float(sweeps.sum()) * elem + batch * 8 * (2 * (M + P) + 2 * N)
    alg_flops = batch * grq_flops(M, N, P)
    kern_s = ms_step * 1e-3
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    result = {
        "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64",
        "data": "synthetic (seeded Haar-SVD generator, BASELINE C4 spec)",
        "config": config_c4(batch, world),
        "roofline": {"bound": "hbm", "achieved": alg_bytes / kern_s / 1e9,
                     "peak": hbm, "unit": "GB/s", "frac": alg_bytes / kern_s / 1e9 / hbm,
                     "traffic": measured_traffic(batch),
                     "kernel": "lse_reg_kernel<float>",
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)"},
        "roofline_fp32": {"bound": "fp32_simt", "achieved": alg_flops / kern_s / 1e12,
                          "peak": peak32, "unit": "TFLOP/s",
                          "frac": alg_flops / kern_s / 1e12 / peak32 if peak32 > 0 else None,
                          "algorithmic_flops_per_launch": alg_flops,
                          "peak_source": "mlsb_fp32_fma_peak_tflops microbenchmark on this GPU",
                          "fp64_fma_peak_tflops": peak64},
        "gpu_launches": args.steps,  # one fused tile-solver launch per step
        "clocks": clocks,
        "solves": {"iterations_mean": float(iters.mean()), "iterations_max": int(iters.max()),
                   "converged": int((status == 0).sum()), "max_iterations": int((status == 1).sum()),
                   "diverged": int((status == 2).sum()), "errors": int((err != 0).sum())},
    }

    # ---- e2e: the public C ABI with pinned host buffers ----------------------
    if not args.no_e2e:
        # with several ranks on one host the pinned copies are bounded (16,384
        # problems = 4.9 GB per rank) so that 8 ranks fit in host memory
        eb = batch if world == 1 else min(batch, 16384)
        Ae, Be = A[:eb], B[:eb]
        hA = torch.empty_strided(Ae.shape, Ae.stride(), dtype=A.dtype, pin_memory=True)
        hA.copy_(Ae)
        hB = torch.empty_strided(Be.shape, Be.stride(), dtype=B.dtype, pin_memory=True)
        hB.copy_(Be)
        del Ae, Be
        hb = b[:eb].cpu().pin_memory()
        hd = d[:eb].cpu().pin_memory()
        ox = torch.empty((eb, N), dtype=torch.float64, pin_memory=True)
        orr = torch.empty((eb, M), dtype=torch.float64, pin_memory=True)
        ov = torch.empty((eb, P), dtype=torch.float64, pin_memory=True)
        ost = torch.empty(eb, dtype=torch.int32, pin_memory=True)
        oit = torch.empty(eb, dtype=torch.int64, pin_memory=True)
        oerr = torch.empty(eb, dtype=torch.int32, pin_memory=True)
        ccfg = cfg.to_c()
        ex = _capi.Exec(_capi.MLSB_HOST, -1, C.c_void_p(stream.cuda_stream))
        vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731

        def e2e_step():
            rc = lib.mlsb_mplse_batched(eb, vp(hA), M, hA.stride(0), vp(hB), P, hB.stride(0),
                                        vp(hb), M, vp(hd), P, M, N, P, C.byref(ccfg), vp(ox),
                                        vp(orr), vp(ov), vp(ost), vp(oit), vp(oerr), None, None,
                                        C.byref(ex))
            _capi.raise_for(rc)

        e2e_step()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ke = max(1, min(args.steps, 3))
        for _ in range(ke):
            e2e_step()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        dt = float(tt.item())
        h2d = (hA.numel() + hB.numel() + hb.numel() + hd.numel()) * 8
        d2h = (ox.numel() + orr.numel() + ov.numel()) * 8 + eb * (4 + 8 + 4)
        result["e2e"] = {"value": world * eb * ke / dt, "unit": "solves/s",
                         "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                         "steps": ke, "problems_per_rank": eb,
                         "api": "mlsb_mplse_batched (C ABI), pinned host buffers"}

    # ---- CPU baseline: the reference on this host, bounded sample, rank 0, N=1
    # (the full batch when it fits in ~cpu_seconds)
    if rank == 0 and world == 1 and not args.no_cpu:
        if args.no_e2e:
            S = min(batch, 16384)
            An, Bn = A[:S].cpu().numpy(), B[:S].cpu().numpy()
            bn, dn = b[:S].cpu().numpy(), d[:S].cpu().numpy()
        else:  # the pinned host copies (same problems, no second 19 GB copy)
            An, Bn, bn, dn = hA.numpy(), hB.numpy(), hb.numpy(), hd.numpy()
        v, cores, kind, k, dt = cpu_reference(An, Bn, bn, dn, args.cpu_seconds)
        result["cpu_baseline"] = {"value": v, "unit": "solves/s", "cores": cores, "kind": kind,
                                  "sample": f"first {k} of the same {batch} C4 problems "
                                            f"({dt:.1f} s, std::thread pool over {cores} threads)"}
        del An, Bn
    if not args.no_e2e:
        del hA, hB
    # ---- the large-problem path on this GPU (BASELINE config 3, one solve) and
    # its trailing-update GEMM at the C3 shape, for the record (rank 0, N = 1)
    if rank == 0 and world == 1 and not args.no_large:
        del A, B
        torch.cuda.empty_cache()
        result["large_path"] = large_path_record(peak32)
    if rank == 0:
        emit(result)


def large_path_record(peak32):
    """C3 (LSE 8192x4096/1024, kappa_A 1e4) through the public API, device phase
    times from the trace, plus the binary32 WY GEMM C -= V W2 (8192 x 3968,
    K = 128) timed with CUDA events."""
    import numpy as np
    import torch

    import paper_2406_16499_b200 as PK
    from paper_2406_16499_b200 import _capi
    from paper_2406_16499_b200 import generate as G

    c = G.CONFIGS["C3"]
    t0 = time.perf_counter()
    A3, B3, b3, d3 = G.lse_problem(c["m"], c["n"], c["p"], c["kappa_A"], c["kappa_B"], c["seed"])
    gen_s = time.perf_counter() - t0
    cfg3 = PK.RefinementConfig(maxit=c["maxit"])
    PK.mplse(PK.LseProblem(A3, B3, b3, d3), cfg3)  # warm-up (allocator, module load)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = PK.mplse(PK.LseProblem(A3, B3, b3, d3), cfg3)
    wall = time.perf_counter() - t0
    ph = {k: float(v) for k, v in res.trace.timing.items()}
    dev_s = sum(ph.values())
    out = {"workload": "C3 LSE 8192x4096/1024, kappa_A 1e4, (s,s,d,d), one solve via mplse (host arrays)",
           "status": res.trace.status, "iterations": res.trace.iterations,
           "device_ms": dev_s * 1e3, "wall_ms_incl_host_staging": wall * 1e3,
           "phases_ms": {k: v * 1e3 for k, v in ph.items()}, "input_generation_s": gen_s,
           "grq_tflops": grq_flops(c["m"], c["n"], c["p"]) / ph["factorization"] / 1e12}
    # the trailing-update GEMM at the C3 QR-stage shape
    lib = _capi.lib
    lib.mlsb_wy_gemm_f32.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, C.c_void_p,
                                     C.c_int64, C.c_void_p, C.c_int64, C.c_float, C.c_void_p, C.c_int64,
                                     C.c_void_p, C.c_size_t, C.c_void_p]
    Mm, Nn, Kk = 8192, 3968, 128
    dev = torch.device("cuda")
    Va = torch.randn(Kk, Mm, device=dev)
    Wb = torch.randn(Nn, Kk, device=dev)
    Cc = torch.randn(Nn, Mm, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    call = lambda: lib.mlsb_wy_gemm_f32(0, 0, Mm, Nn, Kk, -1.0, Va.data_ptr(), Mm, Wb.data_ptr(), Kk, 1.0,  # noqa: E731
                                        Cc.data_ptr(), Mm, None, 0, st)
    for _ in range(3):
        call()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20):
        call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    tf = 2.0 * Mm * Nn * Kk / ms / 1e9
    out["trailing_update_gemm"] = {"shape": "C -= V W2, 8192 x 3968, K = 128 (binary32 SIMT FFMA)",
                                   "ms": ms, "tflops": tf, "peak_tflops": peak32,
                                   "frac": tf / peak32 if peak32 > 0 else None}
    return out


def run_single(args):
    """Latency of one C1 / C2 solve through the public API (host buffers)."""
    import numpy as np
    import torch

    import paper_2406_16499_b200 as PK
    from paper_2406_16499_b200 import generate as G

    c = G.CONFIGS[args.config]
    cfg = PK.RefinementConfig(maxit=c["maxit"], precisions=PK.PrecisionConfig(c["prec"][0], c["prec"][1], "working", c["prec"][2]))
    if c["kind"] == "lse":
        A, B, b, d = G.lse_problem(c["m"], c["n"], c["p"], c["kappa_A"], c["kappa_B"], c["seed"])
        call = lambda: PK.mplse(PK.LseProblem(A, B, b, d), cfg)  # noqa: E731
    else:
        W, V, d = G.gls_problem(c["n"], c["m"], c["p"], c["kappa_A"], c["kappa_B"], c["seed"])
        call = lambda: PK.mpgls(PK.GlsProblem(W, V, d), cfg)  # noqa: E731
    for _ in range(args.warmup):
        res = call()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        res = call()
        ts.append(time.perf_counter() - t0)
    med = statistics.median(ts)
    emit({"metric": METRIC, "value": 1.0 / med, "unit": "solves/s", "n_gpus": 1,
          "steps": args.steps, "warmup": args.warmup, "ms_per_step": med * 1e3,
          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64",
          "data": "synthetic", "config": {"workload": args.config, **{k: v for k, v in c.items() if k != "prec"}},
          "iterations": res.trace.iterations, "status": res.trace.status,
          "device_phase_seconds": res.trace.timing})


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch

        if args.impl == "ours":
            torch.cuda.set_device(local_rank)
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            torch.distributed.init_process_group("gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.config != "C4":
        if rank == 0:
            run_single(args)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch

        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
