#!/usr/bin/env python
"""Benchmark of the B200 classical-IR hot path (BASELINE.json metric).

Headline workload (the JSON line's `value`): BASELINE config 4 -- one batch of
65,536 independent LSE problems (A 256x128, B 32x128, kappa(A) = 10^U(1,5),
kappa(B) = 10) at (u_f, u_s, u, u_r) = (s, s, d, d), tol 1e-13, maxit 40
(reference defaults), solved by ONE launch of the fused tile solver (one CTA
per problem).  With --gpus N (torchrun, one process per GPU) the SAME 65,536
problems are partitioned into N contiguous shards (dist.shard_plan; each rank
generates only its shard with the per-block seed rule of generate.py), each
rank solves its shard with no collective, and one NCCL gather brings x, r, v,
status and passes to rank 0 inside every timed step (strong scaling, SURVEY
§8(e), the reference's run_sweep partition of one cell list,
inc/experiment.hpp:191-217).

A step = one pass of the hot path over the batch with inputs already resident
in HBM (19.3 GB of fp64 A/B >> 126 MB L2, so no L2 flush is needed).  `e2e`
re-times the same work through the C ABI (mlsb_mplse_batched) with pinned HOST
buffers (H2D of the inputs and D2H of x, r, v, status, passes inside the timed
region).

At N = 1, rank 0 adds, after the timed region:
  * cpu_baseline: the unmodified reference (oracle/_ref) on all host threads
    over ALL 65,536 problems, whose results are then compared problem by
    problem with the GPU's (`parity.c4`);
  * `records`: C1, C2, C3 (kappa_A 1e2 / 1e4 / 1e6) and C5 solved on this GPU
    through the public API, each with device phase times, the reference timed
    on ONE host core (trace.timing phases; C5: the complex port, labelled --
    the reference is real-only) and a parity verdict against it;
  * the binary32 WY trailing-update GEMM at the C3 shape against the FP32 peak.

`--impl reference` times the reference's own CPU implementation (oracle/_ref)
on all host cores over the FIRST problems of the same batch (regenerated
bitwise-identically with the same per-block seed rule); that process never
loads the product library.
"""
from __future__ import annotations

import argparse
import ctypes as C
import importlib.util
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "refined LSE/GLS solves/sec; GRQ/GQR GFLOP/s and residual GB/s vs B200 peak"
M, N, P = 256, 128, 32
U53 = 2.0 ** -53
PRODUCT_SO = "libmixedls_b200"


def load_generate():
    """paper_2406_16499_b200/generate.py loaded by file path: numpy/torch only,
    without importing the package (whose __init__ loads the product library)."""
    path = os.path.join(ROOT, "paper_2406_16499_b200", "generate.py")
    spec = importlib.util.spec_from_file_location("mlsb_generate_standalone", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def product_loaded() -> bool:
    try:
        with open("/proc/self/maps") as fh:
            return PRODUCT_SO in fh.read()
    except OSError:
        return False


def grq_flops(m, n, p):
    # GRQ(m,n,p) = (2p^2 n - 2/3 p^3) + (4mnp - 2mp^2) + (2mn^2 - 2/3 n^3)
    return (2 * p * p * n - 2 / 3 * p ** 3) + (4 * m * n * p - 2 * m * p * p) + (2 * m * n * n - 2 / 3 * n ** 3)


def gqr_flops(n, m, p):
    # GQR(n,m,p; n >= p) = (2nm^2 - 2/3 m^3) + (4npm - 2pm^2) + (2np^2 - 2/3 p^3)
    return (2 * n * m * m - 2 / 3 * m ** 3) + (4 * n * p * m - 2 * p * m * m) + (2 * n * p * p - 2 / 3 * p ** 3)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=65536, help="C4 problems in the whole job")
    ap.add_argument("--ref-sample", type=int, default=4096,
                    help="--impl reference: problems per step (the first ones of the batch)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip cpu_baseline + C4 parity")
    ap.add_argument("--no-records", action="store_true", help="skip the C1/C2/C3/C5 records")
    ap.add_argument("--c3-kappas", default="1e2,1e4,1e6")
    ap.add_argument("--no-c5", action="store_true")
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


def emit(obj):
    print(json.dumps(obj), flush=True)


def config_c4(batch, world):
    return {"workload": (f"C4 batched LSE: {batch} problems in the job, A 256x128, B 32x128, "
                         "kappa(A)=10^U(1,5), kappa(B)=10, (u_f,u_s,u,u_r)=(s,s,d,d), "
                         "tol=1e-13, maxit=40"),
            "batch": batch, "batch_per_gpu": -(-batch // world), "m": M, "n": N, "p": P,
            "l2": "inputs 19.3 GB fp64 >> 126 MB L2 at N=1; no flush needed",
            "parallelism": (f"dp{world}: contiguous shards of one batch, no collective on the "
                            "data path, one NCCL gather of the results to rank 0 per step"
                            if world > 1 else "dp1")}


def peaks_file():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            return json.load(fh)
    return {}


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


# ---------------------------------------------------------------------------
def run_reference(args, rank, world):
    """The reference's CPU path (oracle/_ref: the unmodified reference headers
    behind a C shim, std::thread pool over all host threads) on the first
    `ref_sample` problems of the SAME batch the GPU arm solves."""
    if rank != 0:
        return
    import numpy as np
    import torch

    G = load_generate()
    S = min(args.ref_sample, args.batch)
    gdev = "cuda" if torch.cuda.is_available() else "cpu"
    A, B, b, d, _ = G.lse_batch_torch(S, M, N, P, seed=1000, device=gdev)
    A, B, b, d = (t.cpu().numpy() for t in (A, B, b, d))
    if gdev == "cuda":
        torch.cuda.synchronize()
    from oracle.oracle import Oracle, available

    kind = "reference" if available("ref") else "port"
    orc = Oracle("ref" if kind == "reference" else "port")
    cores = len(os.sched_getaffinity(0)) if kind == "reference" else 1
    assert not product_loaded(), "the reference arm must not load the product library"
    vals, dts = [], []
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        orc.mplse_batch(A, B, b, d, maxit=40, prec=("s", "s", "d"), nthreads=cores)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            vals.append(S / dt)
            dts.append(dt)
    value = statistics.median(vals)
    emit({"impl": "reference", "metric": METRIC, "value": value, "unit": "solves/s",
          "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
          "ms_per_step": 1e3 * statistics.median(dts), "higher_is_better": True,
          "scaling": "strong", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
          "config": config_c4(args.batch, world),
          "product_library_loaded": product_loaded(),
          "cpu_baseline": {"value": value, "unit": "solves/s", "cores": cores, "kind": kind,
                           "sample": (f"the first {S} of the {args.batch} C4 problems per step "
                                      + ("(bitwise the GPU arm's inputs: same per-block seeds, "
                                         "generated on cuda); " if gdev == "cuda" else
                                         "(same per-block seeds, generated on the CPU: not "
                                         "bitwise the GPU arm's inputs); ") +
                                      f"mplse per problem on a std::thread pool over {cores} "
                                      "host threads")},
          "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0,
                  "d2h_bytes_per_step": 0}})


# ---------------------------------------------------------------------------
def c4_backward(A, B, b, d, x, r, v, chunk=4096):
    """Stop-test max ratio (inc/lse.hpp:281-290) of every problem, fp64 on the
    device (the checker's arithmetic, not the product's)."""
    import torch

    out = []
    for s0 in range(0, A.shape[0], chunk):
        sl = slice(s0, s0 + chunk)
        a, bb, xx, rr, vv = A[sl], B[sl], x[sl], r[sl], v[sl]
        f1 = b[sl] - rr - torch.bmm(a, xx[:, :, None])[:, :, 0]
        f2 = d[sl] - torch.bmm(bb, xx[:, :, None])[:, :, 0]
        f3 = torch.bmm(bb.transpose(1, 2), vv[:, :, None])[:, :, 0] - \
            torch.bmm(a.transpose(1, 2), rr[:, :, None])[:, :, 0]
        nA = torch.linalg.matrix_norm(a)
        nB = torch.linalg.matrix_norm(bb)
        nr, nv, nx = rr.norm(dim=1), vv.norm(dim=1), xx.norm(dim=1)

        def ratio(num, den):
            q = num / den
            return torch.where(den > 0, q, torch.where(num == 0, torch.zeros_like(q),
                                                         torch.full_like(q, float("inf"))))

        out.append(torch.stack([ratio(f1.norm(dim=1), b[sl].norm(dim=1) + nr + nA * nx),
                                ratio(f2.norm(dim=1), d[sl].norm(dim=1) + nB * nx),
                                ratio(f3.norm(dim=1), nA * nr + nB * nv)]).amax(0))
    return torch.cat(out)


def c4_parity(A, B, b, d, kA, out, ref):
    """Problem-by-problem comparison of the GPU batch with the reference's
    (SURVEY §8(d) bar: forward error <= 40 (m+n+p+1) u kappa_i, passes +-1,
    same status, backward error within 2x of the reference's)."""
    import numpy as np
    import torch

    dev = A.device
    xr, rr, vr, st_r, it_r, err_r = ref
    xg = out.x
    xr_t = torch.from_numpy(xr).to(dev)
    fwd = (xg - xr_t).norm(dim=1) / xr_t.norm(dim=1)
    bound = 40.0 * (M + N + P + 1) * U53 * kA
    be_g = c4_backward(A, B, b, d, out.x, out.r, out.v)
    be_r = c4_backward(A, B, b, d, xr_t, torch.from_numpy(rr).to(dev), torch.from_numpy(vr).to(dev))
    it_g = out.iterations.cpu().numpy()
    st_g = out.status.cpu().numpy()
    both_conv = torch.from_numpy((st_g == 0) & (st_r == 0)).to(dev)
    floor = torch.where(both_conv, torch.full_like(be_r, max(10 * U53, 2e-13)),
                        torch.full_like(be_r, 10 * U53))
    be_bad = be_g > torch.maximum(2.0 * be_r, floor)
    fwd_bad = ~(fwd <= bound)
    idiff = np.abs(it_g.astype(np.int64) - it_r.astype(np.int64))
    fr = (fwd / bound).cpu().numpy()
    ok = (int(idiff.max()) <= 1 and int((st_g != st_r).sum()) == 0 and int(fwd_bad.sum().item()) == 0
          and int(be_bad.sum().item()) == 0)
    return {"ok": ok, "c4_checked": int(A.shape[0]), "against": "oracle/_ref (unmodified reference)",
            "max_iter_diff": int(idiff.max()), "iter_diff_hist": {str(k): int((idiff == k).sum())
                                                                  for k in range(int(idiff.max()) + 1)},
            "mean_passes_gpu": float(it_g.mean()), "mean_passes_ref": float(it_r.mean()),
            "status_mismatches": int((st_g != st_r).sum()),
            "ref_errors": int((err_r != 0).sum()),
            "fwd_violations": int(fwd_bad.sum().item()),
            "max_fwd_over_bound": float(fr.max()),
            "backward_violations": int(be_bad.sum().item()),
            "max_backward_gpu": float(be_g.max().item()), "max_backward_ref": float(be_r.max().item())}


# MLSB_BENCH_DIST=gloo: the N > 1 code path on ONE GPU (all ranks on cuda:0,
# collectives through host copies) -- a functional check of the sharded
# bench where this sandbox has a single GPU; never used for a measurement
DIST_BACKEND = os.environ.get("MLSB_BENCH_DIST", "nccl")


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2406_16499_b200 as PK
    from paper_2406_16499_b200 import _capi
    from paper_2406_16499_b200 import generate as G
    from paper_2406_16499_b200.dist import shard_plan

    dev = torch.device("cuda", local_rank if DIST_BACKEND == "nccl" else 0)
    if DIST_BACKEND != "nccl":
        local_rank = 0
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    total = args.batch
    sh = shard_plan(total, world, rank)
    counts = [shard_plan(total, world, r).count for r in range(world)]
    A, B, b, d, kA = G.lse_batch_torch(sh.count, M, N, P, seed=1000, device=dev, start=sh.start)
    torch.cuda.synchronize()
    cfg = PK.RefinementConfig()  # reference defaults: tol 1e-13, maxit 40, (s,s,d,d)
    width = max(counts)

    # final gather buffers (rank 0): x, r, v, status, passes of the whole batch
    def gather(out):
        if world == 1:
            return out
        parts = []
        for t in (out.x, out.r, out.v, out.status.to(torch.float64)[:, None],
                  out.iterations.to(torch.float64)[:, None]):
            parts.append(t)
        flat = torch.cat(parts, dim=1)
        if flat.shape[0] < width:
            flat = torch.cat([flat, flat.new_zeros((width - flat.shape[0], flat.shape[1]))])
        if DIST_BACKEND != "nccl":
            flat = flat.cpu()
        bufs = [torch.empty_like(flat) for _ in range(world)] if rank == 0 else None
        dist.gather(flat, bufs, dst=0)
        if rank == 0:
            return torch.cat([bb[:c] for bb, c in zip(bufs, counts)])
        return None

    def step():
        out = PK.mplse_batched(A, B, b, d, cfg, stream=stream)
        g = gather(out)
        return out, g

    for _ in range(args.warmup):
        out, gathered = step()
    torch.cuda.synchronize()
    lib = _capi.lib
    lib.mlsb_fp32_fma_peak_tflops.restype = C.c_double
    lib.mlsb_fp64_fma_peak_tflops.restype = C.c_double
    peak32 = lib.mlsb_fp32_fma_peak_tflops(-1, None)
    peak64 = lib.mlsb_fp64_fma_peak_tflops(-1, None)

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local_rank) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            out, gathered = step()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev if DIST_BACKEND == "nccl" else "cpu")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    value = total * args.steps / (ms_max * 1e-3)
    clocks = clk.summary()

    # the gather alone (device time, max over ranks)
    gather_ms = 0.0
    if world > 1:
        g0, g1 = torch.cuda.Event(True), torch.cuda.Event(True)
        dist.barrier()
        g0.record(stream)
        gather(out)
        g1.record(stream)
        torch.cuda.synchronize()
        tg = torch.tensor([g0.elapsed_time(g1)], dtype=torch.float64,
                          device=dev if DIST_BACKEND == "nccl" else "cpu")
        dist.all_reduce(tg, op=dist.ReduceOp.MAX)
        gather_ms = float(tg.item())

    iters = out.iterations.cpu().numpy()
    status = out.status.cpu().numpy()
    err = out.errcode.cpu().numpy()
    solves = {"iterations_mean": float(iters.mean()), "iterations_max": int(iters.max()),
              "converged": int((status == 0).sum()), "max_iterations": int((status == 1).sum()),
              "diverged": int((status == 2).sum()), "errors": int((err != 0).sum())}
    if world > 1:
        st = torch.tensor([solves["converged"], solves["max_iterations"], solves["diverged"],
                           solves["errors"], int(iters.sum())], dtype=torch.float64,
                          device=dev if DIST_BACKEND == "nccl" else "cpu")
        dist.all_reduce(st)
        solves = {"iterations_mean": float(st[4]) / total, "converged": int(st[0]),
                  "max_iterations": int(st[1]), "diverged": int(st[2]), "errors": int(st[3])}
        if rank == 0:
            solves["gathered_rows_on_rank0"] = int(gathered.shape[0])
    elem = (M * N + P * N) * 8
    # fp64 sweeps per problem: max-abs scan, scaled cast, A^T r (solve_v), one residual per pass
    sweeps = 3 + iters.astype(np.float64)
    alg_bytes = float(sweeps.sum()) * elem + sh.count * 8 * (2 * (M + P) + 2 * N)
    alg_flops = sh.count * grq_flops(M, N, P)
    kern_s = ms_step * 1e-3
    hbm = peaks_file().get("hbm_gbs", 6553.3)
    result = {
        "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32+f64",
        "data": "synthetic (seeded Haar-SVD generator, BASELINE C4 spec, per-block seeds)",
        "config": config_c4(total, world),
        # the kernel is latency-bound (per-CTA reflector chain): its FP32 FMA
        # fraction on the GRQ flops is the bound reported; HBM alongside
        "roofline": {"bound": "fp32", "achieved": alg_flops / kern_s / 1e12, "peak": peak32,
                     "unit": "TFLOP/s", "frac": alg_flops / kern_s / 1e12 / peak32 if peak32 > 0 else None,
                     "traffic": measured_traffic(sh.count),
                     "traffic_source": "profiles/c4_ncu_summary.json (ncu --set full, dram bytes/problem)",
                     "kernel": "lse_reg_kernel<float,256,128,32>",
                     "algorithmic_flops_per_launch": alg_flops,
                     "peak_source": "mlsb_fp32_fma_peak_tflops: register-only FFMA microbenchmark on this GPU"},
        "roofline_hbm": {"bound": "hbm", "achieved": alg_bytes / kern_s / 1e9, "peak": hbm,
                         "unit": "GB/s", "frac": alg_bytes / kern_s / 1e9 / hbm,
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)"},
        "fp64_fma_peak_tflops": peak64,
        "gpu_launches": args.steps,  # one fused tile-solver launch per step (the gather is NCCL)
        "clocks": clocks,
        "solves": solves,
    }
    if world > 1:
        result["gather_ms"] = gather_ms

    # ---- e2e: the public C ABI with pinned host buffers (the rank's shard) ----
    hA = hB = hb = hd = None
    if not args.no_e2e:
        eb = sh.count
        hA = torch.empty_strided(A.shape, A.stride(), dtype=A.dtype, pin_memory=True)
        hA.copy_(A)
        hB = torch.empty_strided(B.shape, B.stride(), dtype=B.dtype, pin_memory=True)
        hB.copy_(B)
        hb = b.cpu().pin_memory()
        hd = d.cpu().pin_memory()
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
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ke = max(1, min(args.steps, 3))
        for _ in range(ke):
            e2e_step()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], dtype=torch.float64, device=dev if DIST_BACKEND == "nccl" else "cpu")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        h2d = (hA.numel() + hB.numel() + hb.numel() + hd.numel()) * 8
        d2h = (ox.numel() + orr.numel() + ov.numel()) * 8 + eb * (4 + 8 + 4)
        same = bool(torch.equal(ox, out.x.cpu()) and torch.equal(oit, out.iterations.cpu()))
        result["e2e"] = {"value": total * ke / dt, "unit": "solves/s",
                         "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
                         "steps": ke, "problems_per_rank": eb,
                         "bitwise_equal_to_device_run": same,
                         "api": "mlsb_mplse_batched (C ABI), pinned host buffers"}

    # ---- CPU baseline + C4 parity: the reference on this host, rank 0, N = 1
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle.oracle import Oracle, available

        if hA is not None:
            An, Bn, bn, dn = hA.numpy(), hB.numpy(), hb.numpy(), hd.numpy()
        else:
            An, Bn, bn, dn = (t.cpu().numpy() for t in (A, B, b, d))
        kind = "reference" if available("ref") else "port"
        orc = Oracle("ref" if kind == "reference" else "port")
        threads = len(os.sched_getaffinity(0))
        t0 = time.perf_counter()
        ref = orc.mplse_batch(An, Bn, bn, dn, maxit=40, prec=("s", "s", "d"), nthreads=threads)
        dt = time.perf_counter() - t0
        result["cpu_baseline"] = {"value": total / dt, "unit": "solves/s", "cores": threads,
                                  "kind": kind,
                                  "sample": f"all {total} C4 problems of the timed batch ({dt:.1f} s, "
                                            f"mplse per problem, std::thread pool over {threads} threads)"}
        result["parity"] = {"c4": c4_parity(A, B, b, d, kA, out, ref)}
        del An, Bn, ref
    del hA, hB
    if rank == 0 and world == 1 and not args.no_records:
        del A, B, b, d, out
        torch.cuda.empty_cache()
        recs, par = single_records(args, peak32)
        result["records"] = recs
        result.setdefault("parity", {}).update(par)
    if rank == 0:
        emit(result)


# ---------------------------------------------------------------------------
def _ref_single(orc, kind, args_, out, key):
    t0 = time.perf_counter()
    try:
        res = orc.mplse(*args_[0], **args_[1]) if kind == "lse" else orc.mpgls(*args_[0], **args_[1])
        out[key] = (res, time.perf_counter() - t0, None)
    except Exception as exc:  # noqa: BLE001 -- reported in the record
        out[key] = (None, time.perf_counter() - t0, repr(exc))


def _parity_single(kind, inputs, res, ref, kappa, dims, tol=1e-13):
    import numpy as np

    from tests.helpers import check_parity, fwd_bound, gls_backward, lse_backward, rel

    st = res.state
    if kind == "lse":
        A, B, b, d = inputs
        xg, rg, vg = (np.asarray(t) for t in (st.x, st.r, st.v))
        fwd = rel(xg, ref.x)
        be_g = lse_backward(A, B, b, d, xg, rg, vg)
        be_r = lse_backward(A, B, b, d, ref.x, ref.r, ref.v)
        extra = {}
    else:
        W, V, d = inputs
        xg, yg, zg = (np.asarray(t) for t in (st.x, st.y, st.z))
        fwd = rel(xg, ref.x)
        extra = {"fwd_y": rel(yg, ref.r)}
        be_g = gls_backward(W, V, d, xg, yg, zg)
        be_r = gls_backward(W, V, d, ref.x, ref.r, ref.v)
    bound = fwd_bound(*dims, kappa)
    msgs = check_parity("", fwd, bound, res.trace.iterations, ref.iterations, be_g, be_r,
                        res.trace.status, ref.status, tol)
    if kind != "lse" and not extra["fwd_y"] <= bound:
        msgs.append(f"forward error of y {extra['fwd_y']:.3e} > bound")
    if res.trace.status != ref.status:
        msgs.append(f"status gpu {res.trace.status} vs oracle {ref.status}")
    return {"ok": not msgs, "fwd": fwd, "fwd_bound": bound, **extra,
            "passes_gpu": res.trace.iterations, "passes_ref": ref.iterations,
            "status_gpu": res.trace.status, "status_ref": ref.status,
            "backward_gpu": be_g, "backward_ref": be_r, "violations": msgs}


def _gpu_single(PK, kind, inputs, cfg, reps):
    """Solve through the public API with host arrays; returns (result, median
    wall seconds incl. host staging, device phase seconds of the last run)."""
    import torch

    call = (lambda: PK.mplse(PK.LseProblem(*inputs), cfg)) if kind == "lse" else \
        (lambda: PK.mpgls(PK.GlsProblem(*inputs), cfg))
    res = call()  # warm-up (module load, allocator)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        res = call()
        ts.append(time.perf_counter() - t0)
    return res, statistics.median(ts), dict(res.trace.timing)


def single_records(args, peak32):
    """C1, C2, C3 (three kappas) and C5 on this GPU vs the reference on one host
    core; the oracle solves run in threads (ctypes releases the
    GIL) while the GPU works."""
    import numpy as np

    import paper_2406_16499_b200 as PK
    from oracle.oracle import Oracle, available
    from paper_2406_16499_b200 import generate as G

    kind_ref = "reference" if available("ref") else "port"
    ref = Oracle("ref" if kind_ref == "reference" else "port")
    port = Oracle("port")
    recs, par = {}, {}
    lvl = {"low": "s", "working": "d", "extended": "dd"}

    def cfg_of(c):
        return PK.RefinementConfig(maxit=c["maxit"], precisions=PK.PrecisionConfig(
            c["prec"][0], c["prec"][1], "working", c["prec"][2]))

    def oracle_kw(c):
        return dict(maxit=c["maxit"], prec=tuple(lvl[q] for q in c["prec"]))

    # ---- C1, C2: small single problems (latency), reference on 1 core, 5 reps
    for name in ("C1", "C2"):
        c = G.CONFIGS[name]
        if c["kind"] == "lse":
            inputs = G.lse_problem(c["m"], c["n"], c["p"], c["kappa_A"], c["kappa_B"], c["seed"])
            dims = (c["m"], c["n"], c["p"])
        else:
            inputs = G.gls_problem(c["n"], c["m"], c["p"], c["kappa_A"], c["kappa_B"], c["seed"])
            dims = (c["n"], c["m"], c["p"])
        k = "lse" if c["kind"] == "lse" else "gls"
        res, wall, ph = _gpu_single(PK, k, inputs, cfg_of(c), reps=20)
        cts = []
        for _ in range(5):
            t0 = time.perf_counter()
            rr = ref.mplse(*inputs, **oracle_kw(c)) if k == "lse" else ref.mpgls(*inputs, **oracle_kw(c))
            cts.append(time.perf_counter() - t0)
        dev_s = sum(ph.values())
        recs[name] = {"workload": f"{name} {c['kind'].upper()} {dims}, kappa {c['kappa_A']:.0e}/{c['kappa_B']:.0e}",
                      "status": res.trace.status, "iterations": res.trace.iterations,
                      "device_ms": dev_s * 1e3, "wall_ms_incl_host_staging": wall * 1e3,
                      "solves_per_s": 1.0 / wall, "phases_ms": {q: v * 1e3 for q, v in ph.items()},
                      "cpu_baseline": {"kind": kind_ref, "cores": 1,
                                       "ms": statistics.median(cts) * 1e3,
                                       "phases_ms": dict(zip(("factorization", "init", "residual",
                                                              "correction", "gmres", "other"),
                                                             (float(q) * 1e3 for q in rr.phases))),
                                       "iterations": rr.iterations},
                      "speedup_wall_vs_cpu": statistics.median(cts) / wall}
        par[name] = _parity_single(k, inputs, res, rr, c["kappa_A"], dims)

    # ---- C3 (kappa sweep) and C5: big single problems; oracles in threads
    c3 = G.CONFIGS["C3"]
    kappas = [float(x) for x in args.c3_kappas.split(",") if x]
    probs, threads, done = {}, [], {}
    for kap in kappas:
        t0 = time.perf_counter()
        probs[f"C3_k{kap:.0e}"] = (G.lse_problem(c3["m"], c3["n"], c3["p"], kap, c3["kappa_B"], c3["seed"]),
                                   kap, time.perf_counter() - t0)
    for key, (inp, kap, _) in probs.items():
        th = threading.Thread(target=_ref_single, args=(ref, "lse", (inp, oracle_kw(c3)), done, key))
        th.start()
        threads.append(th)
    c5 = G.CONFIGS["C5"]
    if not args.no_c5:
        t0 = time.perf_counter()
        inp5 = G.gls_problem(c5["n"], c5["m"], c5["p"], c5["kappa_A"], c5["kappa_B"], c5["seed"], cplx=True)
        gen5 = time.perf_counter() - t0
        kw5 = dict(oracle_kw(c5), cplx=True)
        th = threading.Thread(target=_ref_single, args=(port, "gls", (inp5, kw5), done, "C5"))
        th.start()
        threads.append(th)
    gpu = {}
    for key, (inp, kap, gen_s) in probs.items():
        gpu[key] = _gpu_single(PK, "lse", inp, cfg_of(c3), reps=3) + (gen_s,)
    if not args.no_c5:
        gpu["C5"] = _gpu_single(PK, "gls", inp5, cfg_of(c5), reps=3) + (gen5,)
    gemm = trailing_gemm_record(peak32)
    gmres = gmres_records(PK, probs, c3)
    for th in threads:
        th.join()

    m3, n3, p3 = c3["m"], c3["n"], c3["p"]
    for key, (inp, kap, _) in probs.items():
        res, wall, ph, gen_s = gpu[key]
        rr, cdt, cerr = done[key]
        passes = res.trace.iterations
        corr = max(passes - (1 if res.trace.status == "converged" else 0), 0)
        resid_bytes = 8.0 * (m3 * n3 + p3 * n3)
        rec = {"workload": f"C3 LSE {m3}x{n3}/{p3}, kappa_A {kap:.0e}, kappa_B 1e2, (s,s,d,d), maxit 40",
               "status": res.trace.status, "iterations": passes,
               "device_ms": sum(ph.values()) * 1e3, "wall_ms_incl_host_staging": wall * 1e3,
               "phases_ms": {q: v * 1e3 for q, v in ph.items()}, "input_generation_s": gen_s,
               "grq_tflops": grq_flops(m3, n3, p3) / ph["factorization"] / 1e12,
               "grq_frac_fp32": grq_flops(m3, n3, p3) / ph["factorization"] / 1e12 / peak32,
               "residual_gbs": passes * resid_bytes / ph["residual"] / 1e9 if ph["residual"] > 0 else None,
               "correction_gbs": (corr * 2 * 4.0 * (m3 * n3 + p3 * n3) / ph["correction"] / 1e9
                                  if ph["correction"] > 0 else None),
               "ms_per_correction": ph["correction"] * 1e3 / corr if corr else None}
        if rr is not None:
            rec["cpu_baseline"] = {"kind": kind_ref, "cores": 1, "s": cdt,
                                   "phases_s": dict(zip(("factorization", "init", "residual", "correction",
                                                         "gmres", "other"), (float(q) for q in rr.phases))),
                                   "iterations": rr.iterations,
                                   "note": f"{len(threads)} single-threaded oracle solves ran concurrently"}
            rec["speedup_wall_vs_cpu"] = cdt / wall
            par[key] = _parity_single("lse", inp, res, rr, kap, (m3, n3, p3))
        else:
            par[key] = {"ok": False, "oracle_error": cerr}
        recs[key] = rec
    if not args.no_c5:
        res, wall, ph, gen_s = gpu["C5"]
        rr, cdt, cerr = done["C5"]
        n5, mm5, p5 = c5["n"], c5["m"], c5["p"]
        rec = {"workload": f"C5 complex GLS n={n5}, m={mm5}, p={p5}, kappa_W 1e6, kappa_V 1e3, (c64,c64,c128,c128)",
               "status": res.trace.status, "iterations": res.trace.iterations,
               "device_ms": sum(ph.values()) * 1e3, "wall_ms_incl_host_staging": wall * 1e3,
               "phases_ms": {q: v * 1e3 for q, v in ph.items()}, "input_generation_s": gen_s,
               "gqr_tflops_real_equiv": 4 * gqr_flops(n5, mm5, p5) / ph["factorization"] / 1e12}
        if rr is not None:
            rec["cpu_baseline"] = {"kind": "port (complex restatement; the reference is real-only)",
                                   "cores": 1, "s": cdt, "iterations": rr.iterations,
                                   "informational": True}
            par["C5"] = _parity_single("gls", inp5, res, rr, c5["kappa_A"], (n5, mm5, p5))
            par["C5"]["against"] = "oracle port (complex; no reference path exists)"
        else:
            par["C5"] = {"ok": False, "oracle_error": cerr}
        recs["C5"] = rec
    recs["trailing_update_gemm"] = gemm
    recs["gmres_ir_c3"] = gmres
    return recs, par


def gmres_records(PK, probs, c3):
    """GMRES-IR (gmres_refine_lse, inc/krylov.hpp:545-689) at
    the C3 shape, both preconditioners, at kappa_A 1e4 and 1e6 (where
    classical IR approaches its limit): device phases, outer / inner
    iterations, wall time through the public API.  GPU only: the reference's
    GMRES-IR at this size is minutes of CPU time (its factorization alone is
    ~80 s); parity at size is tests/test_gpu_atsize.py."""
    import torch

    out = {}
    for key, (inp, kap, _) in probs.items():
        if kap not in (1e4, 1e6):
            continue
        for pc in ("bd_split", "left"):
            cfg = PK.RefinementConfig(maxit=c3["maxit"])
            PK.gmres_refine_lse(PK.LseProblem(*inp), cfg, precond=pc)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = PK.gmres_refine_lse(PK.LseProblem(*inp), cfg, precond=pc)
            wall = time.perf_counter() - t0
            ph = dict(r.trace.timing)
            out[f"{key}_{pc}"] = {"status": r.trace.status, "outer": r.trace.iterations,
                                  "inner": r.trace.inner_iterations, "device_ms": sum(ph.values()) * 1e3,
                                  "wall_ms": wall * 1e3, "phases_ms": {q: v * 1e3 for q, v in ph.items()},
                                  "ms_per_inner": (ph["gmres"] * 1e3 / r.trace.inner_iterations
                                                   if r.trace.inner_iterations else None)}
    return out


def trailing_gemm_record(peak32):
    """The binary32 WY GEMM C -= V W2 at the C3 QR-stage shape (8192 x 3968,
    K = 128), timed with CUDA events against the live FP32 peak."""
    import torch

    from paper_2406_16499_b200 import _capi

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
    return {"shape": "C -= V W2, 8192 x 3968, K = 128 (binary32 SIMT FFMA)",
            "ms": ms, "tflops": tf, "peak_tflops": peak32,
            "frac": tf / peak32 if peak32 > 0 else None}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch

        if args.impl == "ours" and DIST_BACKEND == "nccl":
            torch.cuda.set_device(local_rank)
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            torch.distributed.init_process_group("gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch

        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
