// C ABI of libmixedls_b200.so (include/mixedls_b200.h).  Validation mirrors
// the reference's exception behaviour (lse.hpp:27-34, gls.hpp:26-32,
// precision.hpp:63-70, refine.hpp:33-37); every solve runs on the GPU.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mixedls_b200.h"
#include "large_internal.h"
#include "mlsb_internal.h"

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(MLSB_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

double unit_roundoff(int32_t lvl) {
  switch (lvl) {
    case MLSB_LOW: return 0x1p-24;
    case MLSB_WORKING: return 0x1p-53;
    case MLSB_EXTENDED: return 0x1p-106;
  }
  return -1.0;
}

// refinement_config::validate + precision_config::validate
int check_config(const mlsb_config* c) {
  if (!c) return fail(MLSB_ERR_INVALID_INPUT, "config is null");
  if (!(c->tol > 0.0)) return fail(MLSB_ERR_INVALID_INPUT, "refinement_config: tol must be positive");
  if (c->maxit < 1) return fail(MLSB_ERR_INVALID_INPUT, "refinement_config: maxit must be >= 1");
  const double uf = unit_roundoff(c->u_f), us = unit_roundoff(c->u_s), u = unit_roundoff(c->u),
               ur = unit_roundoff(c->u_r);
  if (uf < 0 || us < 0 || u < 0 || ur < 0)
    return fail(MLSB_ERR_INVALID_INPUT, "precision_config: unknown precision level");
  if (c->u != MLSB_WORKING)
    return fail(MLSB_ERR_INVALID_INPUT, "precision_config: working precision must be binary64");
  if (uf < us || us < u || u < ur)
    return fail(MLSB_ERR_INVALID_INPUT, "precision_config: requires u_f >= u_s >= u >= u_r");
  return MLSB_OK;
}

struct DevScope {
  int prev = -1;
  bool ok = true;
  explicit DevScope(const mlsb_exec* ex) {
    if (ex && ex->device >= 0) {
      cudaGetDevice(&prev);
      ok = cudaSetDevice(ex->device) == cudaSuccess;
    }
  }
  ~DevScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// stream-ordered device scratch, released on scope exit
struct DevBuf {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  cudaError_t alloc(size_t bytes, cudaStream_t s) {
    st = s;
    if (bytes == 0) bytes = 16;
    return cudaMallocAsync(&p, bytes, s);
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// Host -> device copy of a large range at pinned-memory speed when the source
// is PAGEABLE (numpy / std::vector inputs of the single-problem and batched
// entry points): cudaMemcpyAsync from pageable memory measured 9 GB/s on the
// B200 box, pinned DMA 55 GB/s, one host memcpy thread 13 GB/s.  SH_T host
// threads each copy their chunks into their own pair of pinned staging slots
// and DMA them on their own stream (a slot is reused only after its previous
// DMA completed); the caller's stream waits for every staging stream at the
// end and the staging streams wait for the caller's stream at the start (the
// destination may come from cudaMallocAsync on it).  Pinned sources and small
// ranges take the plain asynchronous copy.  One staging at a time per process.
constexpr int SH_T = 8;
constexpr size_t SH_CH = size_t(8) << 20;
struct StagePool {
  std::mutex mu;
  int device = -1;
  void* slot[SH_T][2] = {};
  cudaEvent_t ev[SH_T][2] = {};
  cudaStream_t s[SH_T] = {};
  cudaEvent_t start = nullptr, done[SH_T] = {};
  bool ready = false;
};
StagePool g_stage;

cudaError_t stage_h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  cudaPointerAttributes at{};
  const bool pinned = cudaPointerGetAttributes(&at, src) == cudaSuccess &&
                      (at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeDevice ||
                       at.type == cudaMemoryTypeManaged);
  cudaGetLastError();  // a pageable pointer is not an error worth keeping
  if (pinned || bytes < 4 * SH_CH) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
  std::lock_guard<std::mutex> lock(g_stage.mu);
  int dev = 0;
  cudaGetDevice(&dev);
  cudaError_t e;
  if (!g_stage.ready || g_stage.device != dev) {
    if (g_stage.ready) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);  // one device only
    for (int t = 0; t < SH_T; ++t) {
      for (int k = 0; k < 2; ++k) {
        if ((e = cudaHostAlloc(&g_stage.slot[t][k], SH_CH, cudaHostAllocDefault))) return e;
        if ((e = cudaEventCreateWithFlags(&g_stage.ev[t][k], cudaEventDisableTiming))) return e;
      }
      if ((e = cudaStreamCreateWithFlags(&g_stage.s[t], cudaStreamNonBlocking))) return e;
      if ((e = cudaEventCreateWithFlags(&g_stage.done[t], cudaEventDisableTiming))) return e;
    }
    if ((e = cudaEventCreateWithFlags(&g_stage.start, cudaEventDisableTiming))) return e;
    g_stage.device = dev;
    g_stage.ready = true;
  }
  if ((e = cudaEventRecord(g_stage.start, st))) return e;
  for (int t = 0; t < SH_T; ++t)
    if ((e = cudaStreamWaitEvent(g_stage.s[t], g_stage.start, 0))) return e;
  const size_t nch = (bytes + SH_CH - 1) / SH_CH;
  std::vector<cudaError_t> err(SH_T, cudaSuccess);
  auto work = [&](int t) {
    cudaSetDevice(dev);
    for (size_t c = size_t(t), r = 0; c < nch; c += SH_T, ++r) {
      const int k = int(r & 1);
      const size_t off = c * SH_CH, len = std::min(SH_CH, bytes - off);
      cudaError_t e2;
      if ((e2 = cudaEventSynchronize(g_stage.ev[t][k]))) { err[t] = e2; return; }
      memcpy(g_stage.slot[t][k], static_cast<const char*>(src) + off, len);
      if ((e2 = cudaMemcpyAsync(static_cast<char*>(dst) + off, g_stage.slot[t][k], len, cudaMemcpyHostToDevice,
                                g_stage.s[t])) ||
          (e2 = cudaEventRecord(g_stage.ev[t][k], g_stage.s[t]))) {
        err[t] = e2;
        return;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < SH_T; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  for (int t = 0; t < SH_T; ++t) {
    if (err[t]) return err[t];
    if ((e = cudaEventRecord(g_stage.done[t], g_stage.s[t])) || (e = cudaStreamWaitEvent(st, g_stage.done[t], 0)))
      return e;
  }
  return cudaSuccess;
}

int64_t* iterations_ptr_guard(int64_t* p, int64_t i) { return p ? p + i : nullptr; }

int check_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(MLSB_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  // keep stream-ordered scratch cached across calls (default threshold 0 would
  // hand it back to the driver at every synchronize)
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  return MLSB_OK;
}

struct Shape {
  int kind;
  int64_t m, n, p;
  // element counts of the two matrices (rows, cols) and of the outputs
  int64_t ra, ca, rb, cb;
  int64_t nx, nr, nv;  // x, r|y, v|z lengths
  int64_t nb, nd;      // rhs lengths (LSE b, d; GLS 0, d)
};

Shape lse_shape(int64_t m, int64_t n, int64_t p) {
  return Shape{mlsb::KIND_LSE, m, n, p, m, n, p, n, n, m, p, m, p};
}
Shape gls_shape(int64_t n, int64_t m, int64_t p) {
  return Shape{mlsb::KIND_GLS, m, n, p, n, m, n, p, m, p, n, 0, n};
}

// Which engine solves this shape: the one-CTA tile kernels (batched, small),
// or the whole-GPU large path (blocked GRQ/GQR + host-driven IR).
bool route_large(const Shape& s, const mlsb_config* cfg, bool cplx) {
  if (cplx) return true;
  if (getenv("MLSB_FORCE_LARGE")) return true;
  const size_t lim = mlsb::device_smem_limit();
  if (s.kind == mlsb::KIND_LSE && mlsb::lse_reg_supported(s.m, s.n, s.p, cfg->u_f, cfg->u_s, cfg->u_r, lim))
    return false;
  const int64_t R = s.kind == mlsb::KIND_LSE ? s.m + s.p : s.n;
  const int64_t C = s.kind == mlsb::KIND_LSE ? s.n : s.m + s.p;
  const bool large_ok = true;  // any real precision combination (u_f = working: binary64 panels/GEMMs)
  const size_t need_g = mlsb::tile_smem_bytes(s.kind, s.m, s.n, s.p, cfg->u_f, cfg->u_s, cfg->u_r, true);
  if (need_g > lim) return large_ok;
  return large_ok && R * C > 384 * 384;
}

// One problem through the large path.  Inputs/outputs follow the exec's pointer
// kind; `esz` = 8 (real) or 16 (complex interleaved).
int solve_large(const Shape& s, int esz, const void* A, int64_t lda, const void* B, int64_t ldb,
                const void* b, const void* d, const mlsb_config* cfg, void* o1, void* o2, void* o3,
                mlsb_trace* trace, int64_t* singular_index, const mlsb_exec* ex, bool cplx,
                int32_t* status_out = nullptr, int64_t* iters_out = nullptr,
                int32_t* err_out = nullptr, double* hist_out = nullptr, int gmres = 0,
                double alpha_scale = 1.0) {
  const bool dev = ex && ex->pointer_kind == MLSB_DEVICE;
  cudaStream_t st = ex ? static_cast<cudaStream_t>(ex->stream) : nullptr;
  cudaError_t e;
  DevBuf bA, bB, bb, bd, bx, br, bv;
  mlsb::lg::LargeProblem P{};
  P.kind = s.kind;
  P.m = s.m;
  P.n = s.n;
  P.p = s.p;
  P.tol = cfg->tol;
  P.maxit = cfg->maxit;
  P.u_f = cfg->u_f;
  P.u_s = cfg->u_s;
  P.u_r = cfg->u_r;
  P.cplx = cplx;
  P.gmres = gmres;
  P.alpha_scale = alpha_scale;
  if (dev) {
    P.A = A;
    P.lda = lda;
    P.B = B;
    P.ldb = ldb;
    P.b = b;
    P.d = d;
    P.x = o1;
    P.r = o2;
    P.v = o3;
  } else {
    const size_t nA = size_t(lda) * (s.ca - 1) + s.ra, nB = size_t(ldb) * (s.cb - 1) + s.rb;
    if ((e = bA.alloc(esz * nA, st)) || (e = bB.alloc(esz * nB, st)) ||
        (e = bd.alloc(esz * s.nd, st)) || (e = bx.alloc(esz * s.nx, st)) ||
        (e = br.alloc(esz * s.nr, st)) || (e = bv.alloc(esz * s.nv, st)))
      return cuda_fail(e, "cudaMallocAsync");
    if ((e = stage_h2d(bA.p, A, esz * nA, st)) || (e = stage_h2d(bB.p, B, esz * nB, st)) ||
        (e = cudaMemcpyAsync(bd.p, d, esz * s.nd, cudaMemcpyHostToDevice, st)))
      return cuda_fail(e, "cudaMemcpyAsync(H2D)");
    if (s.nb > 0) {
      if ((e = bb.alloc(esz * s.nb, st)) ||
          (e = cudaMemcpyAsync(bb.p, b, esz * s.nb, cudaMemcpyHostToDevice, st)))
        return cuda_fail(e, "copy b");
    }
    P.A = bA.p;
    P.lda = lda;
    P.B = bB.p;
    P.ldb = ldb;
    P.b = bb.p;
    P.d = bd.p;
    P.x = bx.p;
    P.r = br.p;
    P.v = bv.p;
  }
  mlsb::lg::LargeOut out;
  int rc = mlsb::lg::large_solve(P, st, &out);
  if (rc) return fail(rc, rc == MLSB_ERR_UNSUPPORTED ? "precision combination not supported by the large-problem path"
                                                   : std::string("large path: ") + cudaGetErrorString(cudaGetLastError()));
  if (status_out) *status_out = out.status;
  if (iters_out) *iters_out = out.iters;
  if (err_out) *err_out = out.err;
  if (hist_out) memcpy(hist_out, out.hist.data(), sizeof(double) * out.hist.size());
  if (out.err == MLSB_ERR_SINGULAR) {
    if (singular_index) *singular_index = out.sing;
    if (!err_out)
      return fail(MLSB_ERR_SINGULAR, "singular_triangular: zero pivot (diagonal index " +
                                         std::to_string(out.sing) + ")");
    return MLSB_OK;
  }
  if (out.err == MLSB_ERR_INVALID_INPUT) {
    if (!err_out) return fail(MLSB_ERR_INVALID_INPUT, "rhs scaling overflowed (extreme norm imbalance)");
    return MLSB_OK;
  }
  if (!dev) {
    if ((o1 && (e = cudaMemcpyAsync(o1, P.x, esz * s.nx, cudaMemcpyDeviceToHost, st))) ||
        (o2 && (e = cudaMemcpyAsync(o2, P.r, esz * s.nr, cudaMemcpyDeviceToHost, st))) ||
        (o3 && (e = cudaMemcpyAsync(o3, P.v, esz * s.nv, cudaMemcpyDeviceToHost, st))))
      return cuda_fail(e, "cudaMemcpyAsync(D2H)");
  }
  if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "cudaStreamSynchronize");
  if (trace) {
    trace->status = out.status;
    trace->iterations = out.iters;
    trace->inner_iterations = out.inner;
    for (int k = 0; k < 6; ++k) trace->phase_seconds[k] = out.phases[k];
    if (trace->residual_history)
      memcpy(trace->residual_history, out.hist.data(), sizeof(double) * out.hist.size());
  }
  return MLSB_OK;
}

int run(const Shape& s, int64_t batch, const double* A, int64_t lda, int64_t sA, const double* B,
        int64_t ldb, int64_t sB, const double* b, int64_t sb, const double* d, int64_t sd,
        const mlsb_config* cfg, double* x, double* r, double* v, int32_t* status, int64_t* iters,
        int32_t* errcode, int64_t* sing, double* hist, double* phases_out, bool force_sync,
        const mlsb_exec* ex);

// Host-buffer batches: chunks of problems flow through NSLOT device slots on
// NSLOT streams, so the host->device copy of chunk k+1 (the bound: 295 KB per
// C4 problem over PCIe) overlaps the solve of chunk k and the copy-back of
// chunk k-1.  Each chunk is a device-mode launch of the same solver.
constexpr int64_t kChunk = 4096;
constexpr int NSLOT = 3;
int run_pipelined(const Shape& s, int64_t batch, const double* A, int64_t lda, int64_t sA,
                  const double* B, int64_t ldb, int64_t sB, const double* b, int64_t sb,
                  const double* d, int64_t sd, const mlsb_config* cfg, double* x, double* r,
                  double* v, int32_t* status, int64_t* iters, int32_t* errcode, int64_t* sing,
                  double* hist, const mlsb_exec* ex) {
  cudaStream_t user = ex ? static_cast<cudaStream_t>(ex->stream) : nullptr;
  const int64_t spanA = (kChunk - 1) * sA + lda * (s.ca - 1) + s.ra;
  const int64_t spanB = (kChunk - 1) * sB + ldb * (s.cb - 1) + s.rb;
  const int64_t spanb = s.nb > 0 ? (kChunk - 1) * sb + s.nb : 0;
  const int64_t spand = (kChunk - 1) * sd + s.nd;
  const int64_t nh = hist ? cfg->maxit * 3 : 0;
  struct Slot {
    cudaStream_t st = nullptr;
    DevBuf A, B, b, d, x, r, v, status, iters, err, sing, hist;
  } slot[NSLOT];
  cudaError_t e = cudaSuccess;
  cudaEvent_t start;
  if ((e = cudaEventCreateWithFlags(&start, cudaEventDisableTiming))) return cuda_fail(e, "event");
  cudaEventRecord(start, user);  // chunks start after the caller's prior work
  int rc = MLSB_OK;
  for (int k = 0; k < NSLOT && !e; ++k) {
    Slot& S = slot[k];
    if ((e = cudaStreamCreateWithFlags(&S.st, cudaStreamNonBlocking))) break;
    cudaStreamWaitEvent(S.st, start, 0);
    if ((e = S.A.alloc(8 * spanA, S.st)) || (e = S.B.alloc(8 * spanB, S.st)) ||
        (e = S.b.alloc(8 * (spanb + 1), S.st)) || (e = S.d.alloc(8 * spand, S.st)) ||
        (e = S.x.alloc(8 * kChunk * s.nx, S.st)) || (e = S.r.alloc(8 * kChunk * s.nr, S.st)) ||
        (e = S.v.alloc(8 * kChunk * s.nv, S.st)) || (e = S.status.alloc(4 * kChunk, S.st)) ||
        (e = S.iters.alloc(8 * kChunk, S.st)) || (e = S.err.alloc(4 * kChunk, S.st)) ||
        (e = S.sing.alloc(8 * kChunk, S.st)) || (e = S.hist.alloc(8 * kChunk * (nh + 1), S.st)))
      break;
  }
  for (int64_t c0 = 0, k = 0; c0 < batch && !e && rc == MLSB_OK; c0 += kChunk, ++k) {
    Slot& S = slot[k % NSLOT];
    const int64_t nb = std::min<int64_t>(kChunk, batch - c0);
    const int64_t nA = (nb - 1) * sA + lda * (s.ca - 1) + s.ra;
    const int64_t nB = (nb - 1) * sB + ldb * (s.cb - 1) + s.rb;
    const int64_t nd = (nb - 1) * sd + s.nd;
    if ((e = cudaMemcpyAsync(S.A.p, A + c0 * sA, 8 * nA, cudaMemcpyHostToDevice, S.st)) ||
        (e = cudaMemcpyAsync(S.B.p, B + c0 * sB, 8 * nB, cudaMemcpyHostToDevice, S.st)) ||
        (e = cudaMemcpyAsync(S.d.p, d + c0 * sd, 8 * nd, cudaMemcpyHostToDevice, S.st)))
      break;
    if (s.nb > 0 && (e = cudaMemcpyAsync(S.b.p, b + c0 * sb, 8 * ((nb - 1) * sb + s.nb),
                                         cudaMemcpyHostToDevice, S.st)))
      break;
    const mlsb_exec dex{MLSB_DEVICE, ex ? ex->device : -1, S.st};
    rc = run(s, nb, S.A.as<double>(), lda, sA, S.B.as<double>(), ldb, sB,
             s.nb > 0 ? S.b.as<double>() : nullptr, sb, S.d.as<double>(), sd, cfg, S.x.as<double>(),
             S.r.as<double>(), S.v.as<double>(), S.status.as<int32_t>(), S.iters.as<int64_t>(),
             S.err.as<int32_t>(), S.sing.as<int64_t>(), hist ? S.hist.as<double>() : nullptr,
             nullptr, false, &dex);
    if (rc) break;
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
      return dst ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, S.st) : cudaSuccess;
    };
    if ((e = d2h(x ? x + c0 * s.nx : nullptr, S.x.p, 8 * nb * s.nx)) ||
        (e = d2h(r ? r + c0 * s.nr : nullptr, S.r.p, 8 * nb * s.nr)) ||
        (e = d2h(v ? v + c0 * s.nv : nullptr, S.v.p, 8 * nb * s.nv)) ||
        (e = d2h(status ? status + c0 : nullptr, S.status.p, 4 * nb)) ||
        (e = d2h(iters ? iters + c0 : nullptr, S.iters.p, 8 * nb)) ||
        (e = d2h(errcode ? errcode + c0 : nullptr, S.err.p, 4 * nb)) ||
        (e = d2h(sing ? sing + c0 : nullptr, S.sing.p, 8 * nb)) ||
        (e = d2h(hist ? hist + c0 * nh : nullptr, S.hist.p, 8 * nb * nh)))
      break;
  }
  cudaError_t es = cudaSuccess;
  for (int k = 0; k < NSLOT; ++k)
    if (slot[k].st) {
      const cudaError_t ek = cudaStreamSynchronize(slot[k].st);
      if (ek && !es) es = ek;
    }
  for (int k = NSLOT - 1; k >= 0; --k) {  // buffers are freed (stream-ordered) before the streams
    Slot& S = slot[k];
    for (DevBuf* bf : {&S.A, &S.B, &S.b, &S.d, &S.x, &S.r, &S.v, &S.status, &S.iters, &S.err,
                       &S.sing, &S.hist})
      if (bf->p) {
        cudaFreeAsync(bf->p, S.st);
        bf->p = nullptr;
      }
    if (S.st) {
      cudaStreamSynchronize(S.st);
      cudaStreamDestroy(S.st);
    }
  }
  cudaEventDestroy(start);
  if (rc) return rc;
  if (e) return cuda_fail(e, "pipelined batch");
  if (es) return cuda_fail(es, "pipelined batch: cudaStreamSynchronize");
  return MLSB_OK;
}

// Run `batch` problems.  Host mode: copy in, solve, copy out, synchronize
// (large host batches go through run_pipelined).  Device mode: launch only
// (asynchronous on the stream).
int run(const Shape& s, int64_t batch, const double* A, int64_t lda, int64_t sA, const double* B,
        int64_t ldb, int64_t sB, const double* b, int64_t sb, const double* d, int64_t sd,
        const mlsb_config* cfg, double* x, double* r, double* v, int32_t* status, int64_t* iters,
        int32_t* errcode, int64_t* sing, double* hist, double* phases_out, bool force_sync,
        const mlsb_exec* ex) {
  const bool dev = ex && ex->pointer_kind == MLSB_DEVICE;
  cudaStream_t st = ex ? static_cast<cudaStream_t>(ex->stream) : nullptr;
  const size_t lim = mlsb::device_smem_limit();
  if (lim == 0) return fail(MLSB_ERR_CUDA, "cannot query the CUDA device");
  if (route_large(s, cfg, false) && !phases_out) {
    // independent large problems: one whole-GPU solve each
    for (int64_t i = 0; i < batch; ++i) {
      int32_t st_i = 1, er_i = 0;
      int64_t it_i = 0, sg_i = -1;
      std::vector<double> h(hist ? size_t(cfg->maxit) * 3 : 0);
      int rc = solve_large(s, 8, A + i * sA, lda, B + i * sB, ldb, s.nb ? b + i * sb : nullptr,
                           d + i * sd, cfg, x + i * s.nx, r + i * s.nr, v + i * s.nv, nullptr, &sg_i,
                           ex, false, &st_i, &it_i, &er_i, hist ? h.data() : nullptr);
      if (rc) return rc;
      auto put = [&](void* dst, const void* src, size_t bytes) {
        if (!dst) return;
        if (dev) cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
        else memcpy(dst, src, bytes);
      };
      put(status ? status + i : nullptr, &st_i, 4);
      put(iterations_ptr_guard(iters, i), &it_i, 8);
      put(errcode ? errcode + i : nullptr, &er_i, 4);
      put(sing ? sing + i : nullptr, &sg_i, 8);
      if (hist) put(hist + i * cfg->maxit * 3, h.data(), sizeof(double) * h.size());
    }
    if (dev) cudaStreamSynchronize(st);
    return MLSB_OK;
  }
  if (!dev && !phases_out && batch >= 2 * kChunk && !getenv("MLSB_DEBUG_STAMPS"))
    return run_pipelined(s, batch, A, lda, sA, B, ldb, sB, b, sb, d, sd, cfg, x, r, v, status, iters,
                         errcode, sing, hist, ex);
  const bool use_reg = s.kind == mlsb::KIND_LSE &&
                       mlsb::lse_reg_supported(s.m, s.n, s.p, cfg->u_f, cfg->u_s, cfg->u_r, lim);
  // factors in shared memory when they fit, else in an L2-resident global workspace
  bool m_global = false;
  size_t need = mlsb::tile_smem_bytes(s.kind, s.m, s.n, s.p, cfg->u_f, cfg->u_s, cfg->u_r, false);
  if (!use_reg && need > lim) {
    m_global = true;
    need = mlsb::tile_smem_bytes(s.kind, s.m, s.n, s.p, cfg->u_f, cfg->u_s, cfg->u_r, true);
  }
  if (!use_reg && need > lim)
    return fail(MLSB_ERR_UNSUPPORTED,
                "problem too large for the one-CTA tile solver (" + std::to_string(need) +
                    " B shared memory > " + std::to_string(lim) + " B)");

  mlsb::TileArgs a{};
  a.kind = s.kind;
  a.m = s.m;
  a.n = s.n;
  a.p = s.p;
  a.batch = batch;
  a.tol = cfg->tol;
  a.maxit = cfg->maxit;
  a.u_f = cfg->u_f;
  a.u_s = cfg->u_s;
  a.u_r = cfg->u_r;
  a.lda = lda;
  a.ldb = ldb;
  cudaError_t e;
  DevBuf bA, bB, bb, bd, bx, br, bv, bst, bit, berr, bsing, bhist, bph;
  // -- inputs --
  if (dev) {
    a.A = A;
    a.sA = sA;
    a.B = B;
    a.sB = sB;
    a.b = b;
    a.sb = sb;
    a.d = d;
    a.sd = sd;
  } else {
    auto span = [&](int64_t ld, int64_t rows, int64_t cols, int64_t stride) {
      return (batch - 1) * stride + ld * (cols - 1) + rows;
    };
    const int64_t nA = span(lda, s.ra, s.ca, sA), nB = span(ldb, s.rb, s.cb, sB);
    if ((e = bA.alloc(sizeof(double) * nA, st)) || (e = bB.alloc(sizeof(double) * nB, st)))
      return cuda_fail(e, "cudaMallocAsync");
    if ((e = stage_h2d(bA.p, A, sizeof(double) * nA, st)) || (e = stage_h2d(bB.p, B, sizeof(double) * nB, st)))
      return cuda_fail(e, "cudaMemcpyAsync(H2D)");
    a.A = bA.as<double>();
    a.sA = sA;
    a.B = bB.as<double>();
    a.sB = sB;
    if (s.nb > 0) {
      const int64_t nbb = (batch - 1) * sb + s.nb;
      if ((e = bb.alloc(sizeof(double) * nbb, st)) ||
          (e = cudaMemcpyAsync(bb.p, b, sizeof(double) * nbb, cudaMemcpyHostToDevice, st)))
        return cuda_fail(e, "copy b");
      a.b = bb.as<double>();
      a.sb = sb;
    }
    const int64_t ndd = (batch - 1) * sd + s.nd;
    if ((e = bd.alloc(sizeof(double) * ndd, st)) ||
        (e = cudaMemcpyAsync(bd.p, d, sizeof(double) * ndd, cudaMemcpyHostToDevice, st)))
      return cuda_fail(e, "copy d");
    a.d = bd.as<double>();
    a.sd = sd;
  }
  // -- outputs --
  if (dev) {
    a.x = x;
    a.r = r;
    a.v = v;
    a.status = status;
    a.iters = iters;
    a.sing = sing;
    a.hist = hist;
  } else {
    if ((e = bx.alloc(sizeof(double) * batch * s.nx, st)) ||
        (e = br.alloc(sizeof(double) * batch * s.nr, st)) ||
        (e = bv.alloc(sizeof(double) * batch * s.nv, st)) ||
        (e = bst.alloc(sizeof(int32_t) * batch, st)) ||
        (e = bit.alloc(sizeof(int64_t) * batch, st)) ||
        (e = bsing.alloc(sizeof(int64_t) * batch, st)))
      return cuda_fail(e, "cudaMallocAsync");
    a.x = bx.as<double>();
    a.r = br.as<double>();
    a.v = bv.as<double>();
    a.status = bst.as<int32_t>();
    a.iters = bit.as<int64_t>();
    a.sing = bsing.as<int64_t>();
    if (hist) {
      if ((e = bhist.alloc(sizeof(double) * batch * cfg->maxit * 3, st)))
        return cuda_fail(e, "cudaMallocAsync");
      a.hist = bhist.as<double>();
    }
  }
  if (dev && errcode) {
    a.err = errcode;
  } else {
    if ((e = berr.alloc(sizeof(int32_t) * batch, st))) return cuda_fail(e, "cudaMallocAsync");
    a.err = berr.as<int32_t>();
  }
  if (phases_out) {
    if ((e = bph.alloc(sizeof(double) * batch * 6, st))) return cuda_fail(e, "cudaMallocAsync");
    a.phases = bph.as<double>();
  }
  DevBuf bstamps;
  const bool dbg = getenv("MLSB_DEBUG_STAMPS") != nullptr;
  void* probe = nullptr;
  if (dbg) {
    if ((e = bstamps.alloc(64 * 8, st))) return cuda_fail(e, "cudaMallocAsync(stamps)");
    cudaMemsetAsync(bstamps.p, 0, 64 * 8, st);
    a.stamps = bstamps.as<unsigned long long>();
    probe = mlsb::probe_buffer();
  }
  DevBuf bgws;
  if (m_global) {
    const size_t per = mlsb::tile_gws_bytes(s.kind, s.m, s.n, s.p, cfg->u_f);
    if ((e = bgws.alloc(per * size_t(batch), st))) return cuda_fail(e, "cudaMallocAsync(workspace)");
    a.gws = bgws.p;
  }
  // defined outputs for every problem: history rows past a problem's pass count
  // read 0, and a problem the kernel rejects (errcode != 0) reports 0 passes
  // and status -1 instead of stale memory
  if (a.hist && (e = cudaMemsetAsync(a.hist, 0, sizeof(double) * batch * cfg->maxit * 3, st)))
    return cuda_fail(e, "cudaMemsetAsync(history)");
  if ((a.iters && (e = cudaMemsetAsync(a.iters, 0, sizeof(int64_t) * batch, st))) ||
      (a.status && (e = cudaMemsetAsync(a.status, 0xff, sizeof(int32_t) * batch, st))))
    return cuda_fail(e, "cudaMemsetAsync(status)");
  if ((e = use_reg ? mlsb::launch_lse_reg(a, st) : mlsb::launch_tile_solver(a, st)))
    return cuda_fail(e, "tile solver launch");

  if (!dev) {
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
      return dst ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st) : cudaSuccess;
    };
    if ((e = d2h(x, a.x, sizeof(double) * batch * s.nx)) ||
        (e = d2h(r, a.r, sizeof(double) * batch * s.nr)) ||
        (e = d2h(v, a.v, sizeof(double) * batch * s.nv)) ||
        (e = d2h(status, a.status, sizeof(int32_t) * batch)) ||
        (e = d2h(iters, a.iters, sizeof(int64_t) * batch)) ||
        (e = d2h(errcode, a.err, sizeof(int32_t) * batch)) ||
        (e = d2h(sing, a.sing, sizeof(int64_t) * batch)) ||
        (e = d2h(hist, a.hist, sizeof(double) * batch * cfg->maxit * 3)))
      return cuda_fail(e, "cudaMemcpyAsync(D2H)");
  }
  if (phases_out) {
    if ((e = cudaMemcpyAsync(phases_out, a.phases, sizeof(double) * 6,
                             cudaMemcpyDeviceToHost, st)))
      return cuda_fail(e, "copy phases");
  }
  if (!dev || force_sync || dbg) {
    if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "cudaStreamSynchronize");
  }
  if (dbg) {
    unsigned long long h[64];
    cudaMemcpy(h, a.stamps, sizeof(h), cudaMemcpyDeviceToHost);
    fprintf(stderr, "MLSB_STAMPS(us from start):");
    for (int i = 1; i < 32; ++i)
      if (h[i]) fprintf(stderr, " [%d] %.1f", i, (h[i] - h[0]) * 1e-3);
    fprintf(stderr, "\n");
    if (void* pp = probe) {
      unsigned long long pr[128];
      cudaMemcpy(pr, pp, sizeof(pr), cudaMemcpyDeviceToHost);
      fprintf(stderr, "MLSB_PROBE raw (cycles from slot 0):");
      for (int i = 0; i < 40; ++i)
        if (pr[i]) fprintf(stderr, " [%d] %lld", i, (long long)(pr[i] - pr[0]));
      fprintf(stderr, "\n");
      fprintf(stderr, "MLSB_PROBE per QR step j1 (owner warp): sum/upd/gen/pub cycles after previous publish\n");
      for (int i = 1; i < 32; ++i)
        if (pr[i] && pr[96 + i - 1])
          fprintf(stderr, "  j1=%d w%d: %lld %lld %lld %lld\n", 33 + i, (33 + i) & 15,
                  (long long)(pr[i] - pr[96 + i - 1]), (long long)(pr[32 + i] - pr[96 + i - 1]),
                  (long long)(pr[64 + i] - pr[96 + i - 1]), (long long)(pr[96 + i] - pr[96 + i - 1]));
      fprintf(stderr, "\n");
    }

  }
  return MLSB_OK;
}

// single-problem driver shared by mplse / mpgls
int solve_single(const Shape& s, const double* A, int64_t lda, const double* B, int64_t ldb,
                 const double* b, const double* d, const mlsb_config* cfg, double* o1, double* o2,
                 double* o3, mlsb_trace* trace, int64_t* singular_index, const mlsb_exec* ex) {
  if (int rc = check_device()) return rc;
  DevScope scope(ex);
  if (!scope.ok) return fail(MLSB_ERR_CUDA, "cudaSetDevice failed");
  if (route_large(s, cfg, false))
    return solve_large(s, 8, A, lda, B, ldb, b, d, cfg, o1, o2, o3, trace, singular_index, ex, false);
  const bool dev = ex && ex->pointer_kind == MLSB_DEVICE;
  cudaStream_t st = ex ? static_cast<cudaStream_t>(ex->stream) : nullptr;
  int32_t status = 1, errc = 0;
  int64_t iters = 0, sing = -1;
  double phases[6] = {0, 0, 0, 0, 0, 0};
  std::vector<double> hist_h(trace && trace->residual_history ? size_t(cfg->maxit) * 3 : 0);
  int rc;
  if (dev) {
    // device arrays for the outputs, small bookkeeping through a device scratch
    DevBuf bk;
    cudaError_t e = bk.alloc(64 + (hist_h.empty() ? 0 : hist_h.size() * 8), st);
    if (e) return cuda_fail(e, "cudaMallocAsync");
    char* base = bk.as<char>();
    int32_t* d_st = reinterpret_cast<int32_t*>(base);
    int32_t* d_err = reinterpret_cast<int32_t*>(base + 8);
    int64_t* d_it = reinterpret_cast<int64_t*>(base + 16);
    int64_t* d_sing = reinterpret_cast<int64_t*>(base + 24);
    double* d_hist = hist_h.empty() ? nullptr : reinterpret_cast<double*>(base + 64);
    rc = run(s, 1, A, lda, 0, B, ldb, 0, b, 0, d, 0, cfg, o1, o2, o3, d_st, d_it, d_err, d_sing,
             d_hist, phases, true, ex);
    if (rc) return rc;
    if ((e = cudaMemcpyAsync(&status, d_st, 4, cudaMemcpyDeviceToHost, st)) ||
        (e = cudaMemcpyAsync(&errc, d_err, 4, cudaMemcpyDeviceToHost, st)) ||
        (e = cudaMemcpyAsync(&iters, d_it, 8, cudaMemcpyDeviceToHost, st)) ||
        (e = cudaMemcpyAsync(&sing, d_sing, 8, cudaMemcpyDeviceToHost, st)))
      return cuda_fail(e, "copy trace");
    if (!hist_h.empty() &&
        (e = cudaMemcpyAsync(hist_h.data(), d_hist, hist_h.size() * 8, cudaMemcpyDeviceToHost, st)))
      return cuda_fail(e, "copy history");
    if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "cudaStreamSynchronize");
  } else {
    // outputs are only written back on success: stage them
    std::vector<double> t1(s.nx), t2(s.nr), t3(s.nv);
    rc = run(s, 1, A, lda, 0, B, ldb, 0, b, 0, d, 0, cfg, t1.data(), t2.data(), t3.data(), &status,
             &iters, &errc, &sing, hist_h.empty() ? nullptr : hist_h.data(), phases, true, ex);
    if (rc) return rc;
    if (errc == 0) {
      if (o1) memcpy(o1, t1.data(), t1.size() * 8);
      if (o2) memcpy(o2, t2.data(), t2.size() * 8);
      if (o3) memcpy(o3, t3.data(), t3.size() * 8);
    }
  }
  if (errc == 3) {
    if (singular_index) *singular_index = sing;
    return fail(MLSB_ERR_SINGULAR, "singular_triangular: zero pivot (diagonal index " +
                                       std::to_string(sing) + ")");
  }
  if (errc == 2)
    return fail(MLSB_ERR_INVALID_INPUT, "rhs scaling overflowed (extreme norm imbalance)");
  if (errc != 0) return fail(MLSB_ERR_OTHER, "device error " + std::to_string(errc));
  if (trace) {
    trace->status = status;
    trace->iterations = iters;
    trace->inner_iterations = 0;
    for (int k = 0; k < 6; ++k) trace->phase_seconds[k] = phases[k];
    if (trace->residual_history)
      memcpy(trace->residual_history, hist_h.data(), sizeof(double) * 3 * size_t(iters));
  }
  return MLSB_OK;
}

}  // namespace

extern "C" {

mlsb_config mlsb_default_config(void) {
  mlsb_config c;
  c.tol = 1e-13;
  c.maxit = 40;
  c.u_f = MLSB_LOW;
  c.u_s = MLSB_LOW;
  c.u = MLSB_WORKING;
  c.u_r = MLSB_WORKING;
  return c;
}

const char* mlsb_last_error(void) { return g_last_error.c_str(); }

int mlsb_version(void) { return 1; }

int mlsb_mplse(const double* A, int64_t lda, const double* B, int64_t ldb, const double* b,
               const double* d, int64_t m, int64_t n, int64_t p, const mlsb_config* cfg,
               double* x, double* r, double* v, mlsb_trace* trace, int64_t* singular_index,
               const mlsb_exec* exec) {
  // lse_problem::validate (lse.hpp:27-34), then refinement_config::validate
  if (m <= 0 || n <= 0 || p <= 0) return fail(MLSB_ERR_DIMENSION, "lse_problem: empty matrix");
  if (p > n || n > m + p)
    return fail(MLSB_ERR_DIMENSION, "lse_problem: requires p <= n <= m + p");
  if (lda < m || ldb < p) return fail(MLSB_ERR_DIMENSION, "lse_problem: leading dimension too small");
  if (!A || !B || !b || !d) return fail(MLSB_ERR_DIMENSION, "lse_problem: null input");
  if (int rc = check_config(cfg)) return rc;
  return solve_single(lse_shape(m, n, p), A, lda, B, ldb, b, d, cfg, x, r, v, trace,
                      singular_index, exec);
}

int mlsb_mpgls(const double* W, int64_t ldw, const double* V, int64_t ldv, const double* d,
               int64_t n, int64_t m, int64_t p, const mlsb_config* cfg, double* x, double* y,
               double* z, mlsb_trace* trace, int64_t* singular_index, const mlsb_exec* exec) {
  // gls_problem::validate (gls.hpp:26-32)
  if (n <= 0 || m <= 0 || p <= 0) return fail(MLSB_ERR_DIMENSION, "gls_problem: empty matrix");
  if (m > n || n > m + p) return fail(MLSB_ERR_DIMENSION, "gls_problem: requires m <= n <= m + p");
  if (ldw < n || ldv < n) return fail(MLSB_ERR_DIMENSION, "gls_problem: leading dimension too small");
  if (!W || !V || !d) return fail(MLSB_ERR_DIMENSION, "gls_problem: null input");
  if (int rc = check_config(cfg)) return rc;
  return solve_single(gls_shape(n, m, p), W, ldw, V, ldv, nullptr, d, cfg, x, y, z, trace,
                      singular_index, exec);
}

// binary64 direct solvers: the initial solve of the refinement at
// u_f = u_s = u = u_r = working with zero refinement passes.
static mlsb_config direct_config() {
  mlsb_config c = mlsb_default_config();
  c.u_f = c.u_s = c.u = c.u_r = MLSB_WORKING;
  c.maxit = 0;
  return c;
}

int mlsb_lse_direct(const double* A, int64_t lda, const double* B, int64_t ldb, const double* b,
                    const double* d, int64_t m, int64_t n, int64_t p, double* x, double* r,
                    double* v, int64_t* singular_index, const mlsb_exec* exec) {
  if (m <= 0 || n <= 0 || p <= 0) return fail(MLSB_ERR_DIMENSION, "lse_problem: empty matrix");
  if (p > n || n > m + p)
    return fail(MLSB_ERR_DIMENSION, "lse_problem: requires p <= n <= m + p");
  if (lda < m || ldb < p) return fail(MLSB_ERR_DIMENSION, "lse_problem: leading dimension too small");
  if (!A || !B || !b || !d) return fail(MLSB_ERR_DIMENSION, "lse_problem: null input");
  const mlsb_config c = direct_config();
  return solve_single(lse_shape(m, n, p), A, lda, B, ldb, b, d, &c, x, r, v, nullptr,
                      singular_index, exec);
}

int mlsb_gls_direct(const double* W, int64_t ldw, const double* V, int64_t ldv, const double* d,
                    int64_t n, int64_t m, int64_t p, double* x, double* y, double* z,
                    int64_t* singular_index, const mlsb_exec* exec) {
  if (n <= 0 || m <= 0 || p <= 0) return fail(MLSB_ERR_DIMENSION, "gls_problem: empty matrix");
  if (m > n || n > m + p) return fail(MLSB_ERR_DIMENSION, "gls_problem: requires m <= n <= m + p");
  if (ldw < n || ldv < n) return fail(MLSB_ERR_DIMENSION, "gls_problem: leading dimension too small");
  if (!W || !V || !d) return fail(MLSB_ERR_DIMENSION, "gls_problem: null input");
  const mlsb_config c = direct_config();
  return solve_single(gls_shape(n, m, p), W, ldw, V, ldv, nullptr, d, &c, x, y, z, nullptr,
                      singular_index, exec);
}

int mlsb_gmres_lse(const double* A, int64_t lda, const double* B, int64_t ldb, const double* b,
                   const double* d, int64_t m, int64_t n, int64_t p, const mlsb_config* cfg,
                   int precond, double alpha_scale, double* x, double* r, double* v,
                   mlsb_trace* trace, int64_t* singular_index, const mlsb_exec* exec) {
  // gmres_refine_lse (krylov.hpp:545): same validation as mplse
  if (m <= 0 || n <= 0 || p <= 0) return fail(MLSB_ERR_DIMENSION, "lse_problem: empty matrix");
  if (p > n || n > m + p)
    return fail(MLSB_ERR_DIMENSION, "lse_problem: requires p <= n <= m + p");
  if (lda < m || ldb < p) return fail(MLSB_ERR_DIMENSION, "lse_problem: leading dimension too small");
  if (!A || !B || !b || !d) return fail(MLSB_ERR_DIMENSION, "lse_problem: null input");
  if (int rc = check_config(cfg)) return rc;
  if (precond != MLSB_PRECOND_LEFT && precond != MLSB_PRECOND_BD_SPLIT)
    return fail(MLSB_ERR_INVALID_INPUT, "gmres: unknown preconditioner");
  if (!(alpha_scale > 0.0)) return fail(MLSB_ERR_INVALID_INPUT, "gmres: alpha_scale must be positive");
  if (cfg->u_f != MLSB_LOW) return fail(MLSB_ERR_UNSUPPORTED, "gmres: built for u_f = low");
  if (int rc = check_device()) return rc;
  DevScope scope(exec);
  if (!scope.ok) return fail(MLSB_ERR_CUDA, "cudaSetDevice failed");
  return solve_large(lse_shape(m, n, p), 8, A, lda, B, ldb, b, d, cfg, x, r, v, trace,
                     singular_index, exec, false, nullptr, nullptr, nullptr, nullptr,
                     precond == MLSB_PRECOND_LEFT ? 1 : 2, alpha_scale);
}

int mlsb_gmres_gls(const double* W, int64_t ldw, const double* V, int64_t ldv, const double* d,
                   int64_t n, int64_t m, int64_t p, const mlsb_config* cfg, int precond,
                   double alpha_scale, double* x, double* y, double* z, mlsb_trace* trace,
                   int64_t* singular_index, const mlsb_exec* exec) {
  // gmres_refine_gls (krylov.hpp:673): same validation as mpgls
  if (n <= 0 || m <= 0 || p <= 0) return fail(MLSB_ERR_DIMENSION, "gls_problem: empty matrix");
  if (m > n || n > m + p) return fail(MLSB_ERR_DIMENSION, "gls_problem: requires m <= n <= m + p");
  if (ldw < n || ldv < n) return fail(MLSB_ERR_DIMENSION, "gls_problem: leading dimension too small");
  if (!W || !V || !d) return fail(MLSB_ERR_DIMENSION, "gls_problem: null input");
  if (int rc = check_config(cfg)) return rc;
  if (precond != MLSB_PRECOND_LEFT && precond != MLSB_PRECOND_BD_SPLIT)
    return fail(MLSB_ERR_INVALID_INPUT, "gmres: unknown preconditioner");
  if (!(alpha_scale > 0.0)) return fail(MLSB_ERR_INVALID_INPUT, "gmres: alpha_scale must be positive");
  if (cfg->u_f != MLSB_LOW) return fail(MLSB_ERR_UNSUPPORTED, "gmres: built for u_f = low");
  if (int rc = check_device()) return rc;
  DevScope scope(exec);
  if (!scope.ok) return fail(MLSB_ERR_CUDA, "cudaSetDevice failed");
  return solve_large(gls_shape(n, m, p), 8, W, ldw, V, ldv, nullptr, d, cfg, x, y, z, trace,
                     singular_index, exec, false, nullptr, nullptr, nullptr, nullptr,
                     precond == MLSB_PRECOND_LEFT ? 1 : 2, alpha_scale);
}

int mlsb_mplse_z(const double* A, int64_t lda, const double* B, int64_t ldb, const double* b,
                 const double* d, int64_t m, int64_t n, int64_t p, const mlsb_config* cfg,
                 double* x, double* r, double* v, mlsb_trace* trace, int64_t* singular_index,
                 const mlsb_exec* exec) {
  if (m <= 0 || n <= 0 || p <= 0) return fail(MLSB_ERR_DIMENSION, "lse_problem: empty matrix");
  if (p > n || n > m + p)
    return fail(MLSB_ERR_DIMENSION, "lse_problem: requires p <= n <= m + p");
  if (lda < m || ldb < p) return fail(MLSB_ERR_DIMENSION, "lse_problem: leading dimension too small");
  if (!A || !B || !b || !d) return fail(MLSB_ERR_DIMENSION, "lse_problem: null input");
  if (int rc = check_config(cfg)) return rc;
  if (int rc = check_device()) return rc;
  DevScope scope(exec);
  if (!scope.ok) return fail(MLSB_ERR_CUDA, "cudaSetDevice failed");
  return solve_large(lse_shape(m, n, p), 16, A, lda, B, ldb, b, d, cfg, x, r, v, trace,
                     singular_index, exec, true);
}

int mlsb_mpgls_z(const double* W, int64_t ldw, const double* V, int64_t ldv, const double* d,
                 int64_t n, int64_t m, int64_t p, const mlsb_config* cfg, double* x, double* y,
                 double* z, mlsb_trace* trace, int64_t* singular_index, const mlsb_exec* exec) {
  if (n <= 0 || m <= 0 || p <= 0) return fail(MLSB_ERR_DIMENSION, "gls_problem: empty matrix");
  if (m > n || n > m + p) return fail(MLSB_ERR_DIMENSION, "gls_problem: requires m <= n <= m + p");
  if (ldw < n || ldv < n) return fail(MLSB_ERR_DIMENSION, "gls_problem: leading dimension too small");
  if (!W || !V || !d) return fail(MLSB_ERR_DIMENSION, "gls_problem: null input");
  if (int rc = check_config(cfg)) return rc;
  if (int rc = check_device()) return rc;
  DevScope scope(exec);
  if (!scope.ok) return fail(MLSB_ERR_CUDA, "cudaSetDevice failed");
  return solve_large(gls_shape(n, m, p), 16, W, ldw, V, ldv, nullptr, d, cfg, x, y, z, trace,
                     singular_index, exec, true);
}

int mlsb_mplse_batched(int64_t batch, const double* A, int64_t lda, int64_t strideA,
                       const double* B, int64_t ldb, int64_t strideB, const double* b,
                       int64_t strideb, const double* d, int64_t strided, int64_t m, int64_t n,
                       int64_t p, const mlsb_config* cfg, double* x, double* r, double* v,
                       int32_t* status, int64_t* iterations, int32_t* errcode,
                       int64_t* singular_index, double* history, const mlsb_exec* exec) {
  if (batch < 0) return fail(MLSB_ERR_DIMENSION, "batch must be >= 0");
  if (m <= 0 || n <= 0 || p <= 0) return fail(MLSB_ERR_DIMENSION, "lse_problem: empty matrix");
  if (p > n || n > m + p)
    return fail(MLSB_ERR_DIMENSION, "lse_problem: requires p <= n <= m + p");
  if (lda < m || ldb < p) return fail(MLSB_ERR_DIMENSION, "lse_problem: leading dimension too small");
  if (int rc = check_config(cfg)) return rc;
  if (batch == 0) return MLSB_OK;
  if (int rc = check_device()) return rc;
  DevScope scope(exec);
  if (!scope.ok) return fail(MLSB_ERR_CUDA, "cudaSetDevice failed");
  return run(lse_shape(m, n, p), batch, A, lda, strideA, B, ldb, strideB, b, strideb, d, strided,
             cfg, x, r, v, status, iterations, errcode, singular_index, history, nullptr, false,
             exec);
}

int mlsb_mpgls_batched(int64_t batch, const double* W, int64_t ldw, int64_t strideW,
                       const double* V, int64_t ldv, int64_t strideV, const double* d,
                       int64_t strided, int64_t n, int64_t m, int64_t p, const mlsb_config* cfg,
                       double* x, double* y, double* z, int32_t* status, int64_t* iterations,
                       int32_t* errcode, int64_t* singular_index, double* history,
                       const mlsb_exec* exec) {
  if (batch < 0) return fail(MLSB_ERR_DIMENSION, "batch must be >= 0");
  if (n <= 0 || m <= 0 || p <= 0) return fail(MLSB_ERR_DIMENSION, "gls_problem: empty matrix");
  if (m > n || n > m + p) return fail(MLSB_ERR_DIMENSION, "gls_problem: requires m <= n <= m + p");
  if (ldw < n || ldv < n) return fail(MLSB_ERR_DIMENSION, "gls_problem: leading dimension too small");
  if (int rc = check_config(cfg)) return rc;
  if (batch == 0) return MLSB_OK;
  if (int rc = check_device()) return rc;
  DevScope scope(exec);
  if (!scope.ok) return fail(MLSB_ERR_CUDA, "cudaSetDevice failed");
  return run(gls_shape(n, m, p), batch, W, ldw, strideW, V, ldv, strideV, nullptr, 0, d, strided,
             cfg, x, y, z, status, iterations, errcode, singular_index, history, nullptr, false,
             exec);
}

}  // extern "C"
