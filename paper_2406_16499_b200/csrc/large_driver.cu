// Large-problem path: ONE LSE/GLS problem on the whole GPU (BASELINE configs
// 3 and 5).  Host-driven (C++) orchestration of device kernels:
//
//   pre-scaling + cast         k_maxabs / k_cast          (lse.hpp:314-338, gls.hpp:287-306)
//   blocked GRQ / GQR at u_f   panel_factor (cluster) + compact-WY GEMMs
//                              (factor.hpp:34-75, householder.hpp:173-222)
//   initial solve at u_f       WY applies, blocked TRSV    (lse.hpp:346-366, gls.hpp:313-326)
//   IR loop                    tiled fp64 dual-GEMV residual, stop test on device,
//                              one 64-byte D2H per pass, cascade at u_s
//                              (lse.hpp:377-421, gls.hpp:336-380)
//
// Factors stay in HBM: the stacked fp32 (complex64) matrix M with T / R and
// the packed reflectors, plus dense per-panel reflector blocks V_b and their
// T_b for the blocked applies.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <type_traits>
#include <vector>

#include "large_common.cuh"
#include "large_internal.h"
#include "large_kernels.cuh"
#include "large_cascade.cuh"
#include "../../include/mixedls_b200.h"
#include "mlsb_internal.h"

namespace mlsb {
namespace lg {

// ----------------------------------------------------------- glue kernels
template <class WT>
__global__ void k_rhs_scale(const WT* src, int n, double c, WT* dst, int* bad) {
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) {
    WT v = src[i];
    WT o;
    if constexpr (tr<WT>::cplx) o = WT{v.x / c, v.y / c};
    else o = v / c;
    dst[i] = o;
    if (bad && !finite_(o)) atomicOr(bad, 1);
  }
}
template <class A, class B>
__global__ void k_convert(const A* src, int n, B* dst) {
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) dst[i] = widen_to<B>(src[i]);
}
template <class T>
__global__ void k_fill(T* x, int n, T v) {
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) x[i] = v;
}
template <class T>
__global__ void k_copy(const T* x, int n, T* y) {
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) y[i] = x[i];
}
// y = a - b (elementwise), n entries
template <class T>
__global__ void k_sub(const T* a, const T* b, int n, T* y) {
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) y[i] = a[i] - b[i];
}
// y = a - (b + c)
template <class T>
__global__ void k_sub2(const T* a, const T* b, const T* c, int n, T* y) {
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) y[i] = a[i] - (b[i] + c[i]);
}
// y = a + (b - c)
template <class T>
__global__ void k_addsub(const T* a, const T* b, const T* c, int n, T* y) {
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) y[i] = a[i] + (b[i] - c[i]);
}
// y = a - b - c  (left to right)
template <class T>
__global__ void k_subsub(const T* a, const T* b, const T* c, int n, T* y) {
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) y[i] = a[i] - b[i] - c[i];
}
template <class T>
__global__ void k_neg(T* x, int n) {
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) x[i] = -x[i];
}
// r_f = b_f - A_f x_f, A_f = fl(A * inv) in the factor precision (lse.hpp:353-355):
// column tiles of GNC (thread per row, loads in batches of 16 from a running
// pointer) write partials that k_rowgemv_red sums in tile order
template <class FT, class WT>
__global__ void __launch_bounds__(KT) k_rowgemv_cast(const WT* A, int64_t lda, int rows, int cols, double inv,
                                                     const FT* x, FT* part) {
  const int i = blockIdx.x * KT + threadIdx.x, j0 = blockIdx.y * GNC, jn = min(GNC, cols - j0);
  if (i >= rows) return;
  FT acc = zero<FT>();
  const WT* p = A + i + int64_t(j0) * lda;
  for (int jb = 0; jb < jn; jb += 16) {
    WT t[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) t[u] = jb + u < jn ? p[int64_t(u) * lda] : zero<WT>();
#pragma unroll
    for (int u = 0; u < 16; ++u)
      if (jb + u < jn) mac(acc, narrow<FT>(scale<WT>(inv, t[u])), x[j0 + jb + u]);
    p += int64_t(16) * lda;
  }
  part[int64_t(blockIdx.y) * rows + i] = acc;
}
template <class FT>
__global__ void k_rowgemv_red(const FT* part, int rows, int ntiles, const FT* bf, FT* rf) {
  for (int i = blockIdx.x * KT + threadIdx.x; i < rows; i += gridDim.x * KT) {
    FT s = zero<FT>();
    for (int t = 0; t < ntiles; ++t) s = s + part[int64_t(t) * rows + i];
    rf[i] = bf[i] - s;
  }
}
// max |x| over n entries (bits, NaN skipped)
template <class T>
__global__ void k_vmax(const T* x, int n, unsigned long long* bits) {
  __shared__ double red[KT / 32];
  double mx = 0.0;
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) {
    const double t = mag(widen_to<typename tr<T>::wide>(x[i]));
    mx = (mx < t) ? t : mx;
  }
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m2 = 0.0;
    for (int w = 0; w < KT / 32; ++w) m2 = fmax(m2, red[w]);
    atomic_max_nonneg(bits, m2);
  }
}
__device__ __forceinline__ double bits_or_one(const unsigned long long* bits) {
  const double s = __longlong_as_double((long long)*bits);
  return s == 0.0 ? 1.0 : s;
}
// out = narrow<CT>(x / s), s = max read from bits (or 1 when bits is null)
template <class WT, class CT>
__global__ void k_demote(const WT* x, int n, const unsigned long long* bits, CT* out) {
  const double s = bits ? bits_or_one(bits) : 1.0;
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) {
    const WT v = x[i];
    WT q;
    if constexpr (tr<WT>::cplx) q = WT{v.x / s, v.y / s};
    else q = v / s;
    out[i] = widen_to<CT>(q);
  }
}
// y += s * widen(c)  (promote_with_scale + update, refine.hpp:117-119); flag non-finite
template <class WT, class CT>
__global__ void k_promote_add(WT* y, int n, const CT* c, const unsigned long long* bits, bool neg,
                              int* bad) {
  const double s = bits ? bits_or_one(bits) : 1.0;
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) {
    WT cv = widen_to<WT>(c[i]);
    if (neg) cv = -cv;
    const WT v = y[i] + scale<WT>(s, cv);
    y[i] = v;
    if (!finite_(v)) atomicOr(bad, 1);
  }
}
// y = s * widen(c)
template <class WT, class CT>
__global__ void k_promote(WT* y, int n, const CT* c, const unsigned long long* bits) {
  const double s = bits ? bits_or_one(bits) : 1.0;
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) y[i] = scale<WT>(s, widen_to<WT>(c[i]));
}
template <class WT>
__global__ void k_scale_out(const WT* x, int n, double f, WT* out) {
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) out[i] = scale<WT>(f, x[i]);
}

// ------------------------------------------------------- stop test kernel
struct StopIn {
  // vector segments whose squared norms are needed (up to 6), and which
  // segments enter the demotion scale sigma
  const void* seg[6];
  int len[6];
  int sigma_mask;  // bit s: segment s is a residual block
};
struct StopOut {
  double nrm[6];
  double sigma;
  int bad;
  int pad;
};
template <class WT>
__global__ void __launch_bounds__(1024) k_stop(StopIn in, StopOut* out, unsigned long long* sbits,
                                                const int* badflag) {
  __shared__ double red[32][8];
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  for (int s = 0; s < 6; ++s) {
    const WT* x = static_cast<const WT*>(in.seg[s]);
    if (!x) continue;
    for (int i = tid; i < in.len[s]; i += 1024) {
      const WT v = x[i];
      acc[s] += abs2d(v);
      if ((in.sigma_mask >> s) & 1) {
        const double t = mag(v);
        acc[6] = (acc[6] < t) ? t : acc[6];
      }
    }
  }
  for (int k = 0; k < 7; ++k)
    for (int o = 16; o; o >>= 1) {
      const double t = __shfl_xor_sync(0xffffffffu, acc[k], o);
      acc[k] = k < 6 ? acc[k] + t : fmax(acc[k], t);
    }
  if (l == 0)
    for (int k = 0; k < 7; ++k) red[w][k] = acc[k];
  __syncthreads();
  if (tid == 0) {
    double t[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int ww = 0; ww < 32; ++ww)
      for (int k = 0; k < 7; ++k) t[k] = k < 6 ? t[k] + red[ww][k] : fmax(t[k], red[ww][k]);
    for (int k = 0; k < 6; ++k) out->nrm[k] = sqrt(t[k]);
    out->sigma = t[6];
    out->bad = badflag ? *badflag : 0;
    *sbits = (unsigned long long)__double_as_longlong(t[6]);
  }
}

// ------------------------------------------------------------- host helpers
static inline int nblk(int64_t n, int per = KT, int cap = 148 * 8) {
  return int(std::max<int64_t>(1, std::min<int64_t>(cap, (n + per - 1) / per)));
}

struct Arena {
  char* base = nullptr;
  size_t used = 0, cap = 0;
  cudaStream_t st = nullptr;
  // debug (MLSB_POISON=1): the arena starts as huge finite garbage instead of
  // whatever the pool held, so a read of a never-written entry shows up;
  // MLSB_POISON_ZERO=i zeroes the i-th take() again (bisection)
  int ntake = 0;
  cudaError_t init(size_t bytes, cudaStream_t s) {
    st = s;
    cap = bytes;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&base), bytes, s);
    if (!e && getenv("MLSB_POISON")) e = cudaMemsetAsync(base, 0x7F, bytes, s);
    return e;
  }
  template <class T> T* take(size_t n) {
    used = (used + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base + used);
    used += n * sizeof(T);
    if (used > cap) return nullptr;
    static const int zi = getenv("MLSB_POISON_ZERO") ? atoi(getenv("MLSB_POISON_ZERO")) : -1;
    if (ntake++ == zi && getenv("MLSB_POISON")) cudaMemsetAsync(p, 0, n * sizeof(T), st);
    return p;
  }
  ~Arena() {
    if (base) cudaFreeAsync(base, st);
  }
};

template <class FT>
struct Blk {
  const FT* V;
  int64_t ldv;
  int L, nbk;
  const FT* T;
  int voff;
  int ldt;
};
// F = P_0 P_1 ... P_last, P_b = I - V_b T_b V_b^H
template <class FT>
struct Fac {
  std::vector<Blk<FT>> b;
  std::vector<BlkD<FT>> hd;  // descriptors of the persistent apply (device copy in `dev`)
  BlkD<FT>* dev = nullptr;
  int nrows = 0;             // max(voff + L)
};

// Scratch of the persistent cascade kernels (large_cascade.cuh), set by solve()
// for its thread: step counters / flags and the per-step partials.
// Three lanes, so that three streams can run persistent kernels at once (the
// correction's independent applies and solves); `lane` selects the one the
// next apply_F / trsv call uses.
constexpr int CZ_LANES = 3;
struct CzScratch {
  static inline thread_local int* cnt = nullptr;    // per lane: [CZ_CNT] apply counters | [CZ_CNT] trsv flags
  static inline thread_local char* part = nullptr;  // per lane: partials of k_fac_apply
  static inline thread_local size_t part_bytes = 0; // per lane
  static inline thread_local int lane = 0;
  static int* lane_cnt() { return cnt ? cnt + size_t(lane) * 2 * 1024 : nullptr; }
  static void* lane_part() { return part ? part + size_t(lane) * part_bytes : nullptr; }
};
constexpr int CZ_CNT = 1024;
struct CzScratchGuard {
  CzScratchGuard(int* c, char* p, size_t n) {
    CzScratch::cnt = c;
    CzScratch::part = p;
    CzScratch::part_bytes = n;
    CzScratch::lane = 0;
  }
  ~CzScratchGuard() {
    CzScratch::cnt = nullptr;
    CzScratch::part = nullptr;
    CzScratch::part_bytes = 0;
    CzScratch::lane = 0;
  }
};
// A second stream (and two events) for independent halves of the GMRES
// preconditioners, set by solve() when the persistent kernels are in use.
struct CzAux {
  static inline thread_local cudaStream_t s = nullptr;
  static inline thread_local cudaEvent_t fork = nullptr, join = nullptr;
};
struct CzLane {  // RAII: apply_F / trsv calls in this scope use lane `l`
  int prev;
  explicit CzLane(int l) : prev(CzScratch::lane) { CzScratch::lane = l; }
  ~CzLane() { CzScratch::lane = prev; }
};
// MLSB_CASCADE_OLD=1: round-1 block-per-launch applies and TRSVs (A/B switch)
static bool cascade_on() {
  static const bool off = getenv("MLSB_CASCADE_OLD") != nullptr;
  return !off;
}
static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 1;
  }
  return n;
}

// device copy of a factor's block descriptors (after its stage is built)
template <class FT>
static cudaError_t fac_upload(Fac<FT>& F, BlkD<FT>* dst, cudaStream_t st) {
  F.hd.clear();
  F.nrows = 0;
  for (const Blk<FT>& b : F.b) {
    F.hd.push_back(BlkD<FT>{b.V, b.T, b.ldv, b.L, b.nbk, b.voff, b.ldt});
    F.nrows = std::max(F.nrows, b.voff + b.L);
  }
  if (F.hd.empty() || int(F.hd.size()) > CZ_MAXB || !dst) return cudaSuccess;
  F.dev = dst;
  return cudaMemcpyAsync(dst, F.hd.data(), sizeof(BlkD<FT>) * F.hd.size(), cudaMemcpyHostToDevice, st);
}

// the whole factor in one cooperative launch; false if it does not apply
template <class FT, class CT>
static bool apply_F_persistent(const Fac<FT>& F, bool herm, CT* x, cudaStream_t st) {
  if (!cascade_on() || !F.dev || !CzScratch::cnt) return false;
  constexpr int RB = 32 * (16 / sizeof(FT) > 0 ? 16 / sizeof(FT) : 1);
  const int nb = int(F.hd.size());
  const int G = (F.nrows + RB - 1) / RB;
  if (nb == 0 || G > sm_count() ||
      size_t(nb) * G * 128 * sizeof(CT) > CzScratch::part_bytes || nb > CZ_CNT)
    return false;
  int* cnt = CzScratch::lane_cnt();
  if (cudaMemsetAsync(cnt, 0, sizeof(int) * nb, st) != cudaSuccess) return false;
  const BlkD<FT>* blks = F.dev;
  int hm = herm ? 1 : 0, nr = F.nrows;
  CT* part = static_cast<CT*>(CzScratch::lane_part());
  const size_t sm = sizeof(FT) * 128 * (128 + 16 / sizeof(FT));  // staged T_b
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_fac_apply<FT, CT, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)) ||
        cudaFuncSetAttribute(k_fac_apply<FT, CT, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)) ||
        cudaFuncSetAttribute(k_fac_apply<FT, CT, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)) ||
        cudaFuncSetAttribute(k_fac_apply<FT, CT, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)))
      return false;
    attr = true;
  }
  (void)hm;
  // 16-byte loads when every block's columns start 16-byte aligned at every
  // CTA's first row (voff, ldv and the base multiples of the vector width)
  bool al = true;
  for (const BlkD<FT>& b : F.hd)
    al = al && (reinterpret_cast<uintptr_t>(b.V) % 16 == 0) && (b.ldv * sizeof(FT)) % 16 == 0 &&
         (size_t(b.voff) * sizeof(FT)) % 16 == 0;
  void* args[] = {(void*)&blks, (void*)&nb, (void*)&x, (void*)&nr, (void*)&part, (void*)&cnt};
  void* fn = herm ? (al ? reinterpret_cast<void*>(k_fac_apply<FT, CT, true, true>)
                        : reinterpret_cast<void*>(k_fac_apply<FT, CT, true, false>))
                  : (al ? reinterpret_cast<void*>(k_fac_apply<FT, CT, false, true>)
                        : reinterpret_cast<void*>(k_fac_apply<FT, CT, false, false>));
  return cudaLaunchCooperativeKernel(fn, dim3(G), dim3(CZ_NT), args, sm, st) == cudaSuccess;
}

// ypart: WYB * 256 partials of the dot kernel
template <class FT, class CT>
static void apply_F(const Fac<FT>& F, bool herm, CT* x, CT* ypart, cudaStream_t st) {
  if (apply_F_persistent<FT, CT>(F, herm, x, st)) return;
  const int nb = int(F.b.size());
  for (int s = 0; s < nb; ++s) {
    const Blk<FT>& b = F.b[herm ? s : nb - 1 - s];
    const int dch = (b.L + WYD - 1) / WYD, dpc = WYD * ((dch + 255) / 256);  // <= 256 partials
    const int nd = (b.L + dpc - 1) / dpc;
    const int uch = (b.L + WYR - 1) / WYR, upc = WYR * ((uch + 147) / 148);  // <= 148 update CTAs
    const int nu = (b.L + upc - 1) / upc;
    k_wy_dot<FT, CT><<<nd, KT, 0, st>>>(b.V, b.ldv, b.L, b.nbk, x + b.voff, dpc, ypart);
    k_wy_upd<FT, CT><<<nu, KT, 0, st>>>(b.V, b.ldv, b.L, b.nbk, ypart, nd, b.T, b.ldt, herm, upc, x + b.voff);
  }
}

// upper-triangular solve with U = M[r0:r0+k, c0:c0+k]; herm: U^H x = b.
// Diagonal blocks of TRB = 128 (one CTA each), off-diagonal GEMV updates.
template <class FT, class CT>
static bool trsv_persistent(const FT* M, int64_t ld, int64_t r0, int64_t c0, int k, bool herm, CT* x,
                            cudaStream_t st) {
  if (!cascade_on() || !CzScratch::cnt || k <= 0) return false;
  const int K = (k + CZT - 1) / CZT;
  if (K > sm_count() || K > CZ_CNT) return false;
  const size_t sm = sizeof(FT) * CZT * (CZT + 4) + sizeof(CT) * CZT * 6;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_trsv_chain<FT, CT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)) ||
        cudaFuncSetAttribute(k_trsv_chain<FT, CT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)))
      return false;
    attr = true;
  }
  int* flags = CzScratch::lane_cnt() + CZ_CNT;
  if (cudaMemsetAsync(flags, 0, sizeof(int) * K, st) != cudaSuccess) return false;
  void* args[] = {(void*)&M, (void*)&ld, (void*)&r0, (void*)&c0, (void*)&k, (void*)&x, (void*)&flags};
  void* fn = herm ? reinterpret_cast<void*>(k_trsv_chain<FT, CT, true>)
                  : reinterpret_cast<void*>(k_trsv_chain<FT, CT, false>);
  return cudaLaunchCooperativeKernel(fn, dim3(K), dim3(CZ_NT), args, sm, st) == cudaSuccess;
}

template <class FT, class CT>
static void trsv(const FT* M, int64_t ld, int64_t r0, int64_t c0, int k, bool herm, CT* x,
                 cudaStream_t st) {
  if (trsv_persistent<FT, CT>(M, ld, r0, c0, k, herm, x, st)) return;
  const size_t sm = sizeof(FT) * TRB * (TRB + 1) + sizeof(CT) * TRB;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_trsv_diag128<FT, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    attr = true;
  }
  if (!herm) {
    for (int i1 = k; i1 > 0; i1 -= TRB) {
      const int i0 = std::max(0, i1 - TRB), bs = i1 - i0;
      k_trsv_diag128<FT, CT><<<1, TRB, sm, st>>>(M, ld, r0, c0, i0, bs, false, x);
      if (i0 > 0) k_trsv_off<FT, CT><<<nblk(i0, 64), KT, 0, st>>>(M, ld, r0, c0, i0, bs, k, false, x);
    }
  } else {
    for (int i0 = 0; i0 < k; i0 += TRB) {
      const int bs = std::min(TRB, k - i0);
      k_trsv_diag128<FT, CT><<<1, TRB, sm, st>>>(M, ld, r0, c0, i0, bs, true, x);
      if (i0 + bs < k)
        k_trsv_off<FT, CT><<<nblk(k - i0 - bs, KT / 32), KT, 0, st>>>(M, ld, r0, c0, i0, bs, k, true, x);
    }
  }
}

// column-tiled partials need rows * ceil(cols / GNC) scratch entries; solve()
// provides the scratch for its thread (without it: one tile, y written directly)
template <class CT>
struct GemvScratch {
  static inline thread_local CT* p = nullptr;
  static inline thread_local size_t n = 0;
};
template <class FT, class CT>
static void gemv_n(const FT* M, int64_t ld, int r0, int rows, int c0, int cols, Mask mk, const CT* x,
                   CT* y, cudaStream_t st) {
  if (rows <= 0) return;
  const int nt = std::max(1, (cols + GNC - 1) / GNC);
  CT* part = GemvScratch<CT>::p;
  if (!part || size_t(rows) * nt > GemvScratch<CT>::n) {
    k_gemv_n<FT, CT><<<dim3((rows + KT - 1) / KT, 1), KT, 0, st>>>(M, ld, r0, rows, c0, cols, std::max(cols, 1),
                                                                   mk, x, y);
    return;
  }
  k_gemv_n<FT, CT><<<dim3((rows + KT - 1) / KT, nt), KT, 0, st>>>(M, ld, r0, rows, c0, cols, GNC, mk, x, part);
  k_gemv_n_red<CT><<<nblk(rows), KT, 0, st>>>(part, rows, nt, y);
}
template <class CT>
struct GemvScratchGuard {
  GemvScratchGuard(CT* p, size_t n) {
    GemvScratch<CT>::p = p;
    GemvScratch<CT>::n = n;
  }
  ~GemvScratchGuard() {
    GemvScratch<CT>::p = nullptr;
    GemvScratch<CT>::n = 0;
  }
};

template <class FT, class CT>
static void gemv_h(const FT* M, int64_t ld, int r0, int rows, int c0, int cols, Mask mk, const CT* x,
                   CT* y, cudaStream_t st) {
  if (cols <= 0) return;
  k_gemv_h<FT, CT><<<nblk(cols, KT / 32), KT, 0, st>>>(M, ld, r0, rows, c0, cols, mk, x, y);
}

template <class FT>
static cudaError_t gemm(bool ha, bool hb, int Mr, int N, int K, double alpha, const FT* A,
                        int64_t lda, const FT* B, int64_t ldb, double beta, FT* C, int64_t ldc,
                        FT* work, size_t wn, cudaStream_t st) {
  if constexpr (tr<FT>::cplx)
    return gemm_c64(ha, hb, Mr, N, K, cf{float(alpha), 0.f}, A, lda, B, ldb, cf{float(beta), 0.f}, C,
                    ldc, work, wn, st);
  else if constexpr (std::is_same<FT, double>::value)
    return gemm_f64(ha, hb, Mr, N, K, alpha, A, lda, B, ldb, beta, C, ldc, work, wn, st);
  else
    return gemm_f32(ha, hb, Mr, N, K, float(alpha), A, lda, B, ldb, float(beta), C, ldc, work, wn, st);
}

// ----------------------------------------------- blocked GRQ / GQR at u_f
// Two-level blocking.  Panels of NB = 32 reflectors are factored by one
// cluster each (panel_factor); NBO / NB consecutive panels form an outer
// block whose own columns (rows, for RQ) are brought up to date by rank-NB
// updates, and whose merged compact-WY form (V: L x NBO, T: NBO x NBO,
// k_tmerge) then updates the whole trailing matrix in ONE rank-NBO product --
// three GEMMs with K = NBO or K = L instead of K = NB, the arithmetic
// intensity the FP32 FFMA roofline needs.
//
// Look-ahead: after outer block B, the columns (rows) of block B+1 are
// updated first; block B+1 is then factored (panels, inner updates, T merge)
// on the high-priority stream `s2` while the remaining trailing update of
// block B (the big GEMMs) runs on `st` over the other SMs.
struct WsBuf {
  void* W;
  void* W2;
  void* work;
  size_t wn;
};
struct Streams {
  cudaStream_t st, s2;
  cudaEvent_t ev_upd, ev_pan;
  WsBuf ws[2];   // [0] for st, [1] for s2 (inner updates and Gram products)
  void* G;       // NBO x NBO Gram matrix of the block factored on s2
};

// resident-CTA cap of a trailing update that runs beside a look-ahead block
// factorization: 148 + 100 CTAs of the 2-per-SM GEMM tile leave one slot free
// on 48 SMs for the panel cluster and the small inner-update GEMMs
static int trail_cap() {
  static const int v = getenv("MLSB_TRAIL_CAP") ? atoi(getenv("MLSB_TRAIL_CAP")) : 148 + 100;
  return v;
}
#define kTrailCap trail_cap()

// Skinny compact-WY products of the inner updates (one panel's nbk <= 32
// reflectors onto the <= 96 later columns / rows of its outer block).  As
// three library-shaped GEMMs these cost a split-K GEMM + its reduction + a
// one-tile T GEMM, each a mostly-idle launch on the look-ahead critical path;
// here they are two kernels:
//   k_skinny_part: P_g[k][n] = sum over CTA g's row chunks of op(V[r][k]) X(r, n)
//     QR: X(r, n) = C2[r + n ld], op = conj  (P = V^H C2, nbk x nc)
//     RQ: X(r, n) = Ma[n + r ld], op = id    (P = (Ma V)^T, nbk x nr)
//   k_skinny_tmul: W = sum_g P_g in CTA order, then
//     QR: W2 = T^H W (nbk x nc, ld nbk);  RQ: W2 = W^T T (nr x nbk, ld nr)
// Neither needs co-residency: they run beside the capped trailing GEMM.
constexpr int SK_RC = 64, SK_NT = 256, SK_NMAX = 96, SK_GMAX = 96, SK_VLD = 36;
template <class FT, bool RQ>
__global__ void __launch_bounds__(SK_NT) k_skinny_part(const FT* __restrict__ X, int64_t ld,
                                                       const FT* __restrict__ V, int64_t ldv, int L, int nbk,
                                                       int nc, FT* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char sk_sm[];
  FT* Vs = reinterpret_cast<FT*>(sk_sm);  // [SK_RC][SK_VLD], V row-major
  FT* Xs = Vs + SK_RC * SK_VLD;           // [nc][SK_RC + 1]
  const int t = threadIdx.x, kq = t & 7, ng = t >> 3;
  FT acc[3][4];
#pragma unroll
  for (int j = 0; j < 3; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[j][q] = zero<FT>();
  const int nchunk = (L + SK_RC - 1) / SK_RC;
  for (int ch = blockIdx.x; ch < nchunk; ch += gridDim.x) {
    const int r0 = ch * SK_RC, rows = min(SK_RC, L - r0);
    __syncthreads();
    for (int i = t; i < SK_RC * 32; i += SK_NT) {
      const int r = i % SK_RC, k = i / SK_RC;
      Vs[r * SK_VLD + k] = (r < rows && k < nbk) ? V[r0 + r + k * ldv] : zero<FT>();
    }
    if (!RQ) {
      for (int i = t; i < SK_RC * nc; i += SK_NT) {
        const int r = i % SK_RC, n = i / SK_RC;
        Xs[n * (SK_RC + 1) + r] = r < rows ? X[r0 + r + n * ld] : zero<FT>();
      }
    } else {
      for (int i = t; i < SK_RC * nc; i += SK_NT) {
        const int n = i % nc, r = i / nc;
        Xs[n * (SK_RC + 1) + r] = r < rows ? X[n + (r0 + r) * ld] : zero<FT>();
      }
    }
    __syncthreads();
#pragma unroll 4
    for (int r = 0; r < SK_RC; ++r) {
      FT v[4];
      if constexpr (sizeof(FT) == 4) {
        const float4 q4 = *reinterpret_cast<const float4*>(Vs + r * SK_VLD + 4 * kq);
        v[0] = q4.x, v[1] = q4.y, v[2] = q4.z, v[3] = q4.w;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = Vs[r * SK_VLD + 4 * kq + q];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (!RQ) v[q] = conj_(v[q]);
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int n = ng + 32 * j;
        if (n < nc) {
          const FT x = Xs[n * (SK_RC + 1) + r];
#pragma unroll
          for (int q = 0; q < 4; ++q) mac(acc[j][q], v[q], x);
        }
      }
    }
  }
  FT* P = part + size_t(blockIdx.x) * 32 * nc;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const int n = ng + 32 * j;
    if (n < nc)
#pragma unroll
      for (int q = 0; q < 4; ++q) P[4 * kq + q + 32 * n] = acc[j][q];
  }
}

template <class FT, bool RQ>
__global__ void __launch_bounds__(128) k_skinny_tmul(const FT* __restrict__ part, int G, int nbk, int nc,
                                                     const FT* __restrict__ T, int ldt, FT* __restrict__ W2) {
  __shared__ FT ws[4][32];
  const int w = threadIdx.x >> 5, k = threadIdx.x & 31, n = blockIdx.x * 4 + w;
  if (n >= nc) return;  // whole warp
  const FT* p = part + k + 32 * n;
  const size_t gs = size_t(32) * nc;
  FT s = zero<FT>();
  int g = 0;
  for (; g + 8 <= G; g += 8) {
    FT b[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) b[i] = p[(g + i) * gs];
#pragma unroll
    for (int i = 0; i < 8; ++i) s = s + b[i];
  }
  for (; g < G; ++g) s = s + p[g * gs];
  ws[w][k] = s;
  __syncwarp();
  if (k >= nbk) return;
  FT o = zero<FT>();
  for (int kk = 0; kk <= k; ++kk) {
    const FT tv = T[kk + int64_t(ldt) * k];
    mac(o, RQ ? tv : conj_(tv), ws[w][kk]);
  }
  if (!RQ) W2[k + int64_t(nbk) * n] = o;
  else W2[n + int64_t(nc) * k] = o;
}

static bool skinny_on() {
  static const bool v = getenv("MLSB_SKINNY_OLD") == nullptr;
  return v;
}
template <class FT>
static bool skinny_fits(int L, int nbk, int nc, const WsBuf& w) {
  const int G = std::min((L + SK_RC - 1) / SK_RC, SK_GMAX);
  return skinny_on() && nbk <= 32 && nc > 0 && nc <= SK_NMAX && L > 0 && size_t(G) * 32 * nc <= w.wn;
}
// W2 of an inner update (skinny_fits must hold)
template <class FT, bool RQ>
static cudaError_t skinny_w2(const FT* X, int64_t ld, const FT* V, int64_t ldv, int L, int nbk, int nc,
                             const FT* Tb, int ldt, FT* W2, const WsBuf& w, cudaStream_t st) {
  constexpr size_t smax = (SK_RC * SK_VLD + SK_NMAX * (SK_RC + 1)) * sizeof(FT);
  static const cudaError_t attr =
      cudaFuncSetAttribute(k_skinny_part<FT, RQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smax));
  if (attr) return attr;
  const int G = std::min((L + SK_RC - 1) / SK_RC, SK_GMAX);
  const size_t sm = (SK_RC * SK_VLD + size_t(nc) * (SK_RC + 1)) * sizeof(FT);
  FT* part = static_cast<FT*>(w.work);
  k_skinny_part<FT, RQ><<<G, SK_NT, sm, st>>>(X, ld, V, ldv, L, nbk, nc, part);
  k_skinny_tmul<FT, RQ><<<(nc + 3) / 4, 128, 0, st>>>(part, G, nbk, nc, Tb, ldt, W2);
  return cudaGetLastError();
}

// C2 := P^H C2 = C2 - V T^H (V^H C2) for C2 = M[j0:j0+L, c0:c0+nc]
template <class FT>
static cudaError_t qr_update(FT* M, int64_t ld, int j0, int L, int nbk, int c0, int nc, const FT* V,
                             int64_t ldv, const FT* Tb, int ldt, const WsBuf& w, cudaStream_t st) {
  if (nc <= 0) return cudaSuccess;
  cudaError_t e;
  FT* W = static_cast<FT*>(w.W);
  FT* W2 = static_cast<FT*>(w.W2);
  FT* work = static_cast<FT*>(w.work);
  FT* C2 = M + j0 + int64_t(c0) * ld;
  if (skinny_fits<FT>(L, nbk, nc, w)) {
    if ((e = skinny_w2<FT, false>(C2, ld, V, ldv, L, nbk, nc, Tb, ldt, W2, w, st))) return e;
    return gemm<FT>(false, false, L, nc, nbk, -1.0, V, ldv, W2, nbk, 1.0, C2, ld, nullptr, 0, st);
  }
  if ((e = gemm<FT>(true, false, nbk, nc, L, 1.0, V, ldv, C2, ld, 0.0, W, nbk, work, w.wn, st))) return e;
  if ((e = gemm<FT>(true, false, nbk, nc, nbk, 1.0, Tb, ldt, W, nbk, 0.0, W2, nbk, nullptr, 0, st))) return e;
  return gemm<FT>(false, false, L, nc, nbk, -1.0, V, ldv, W2, nbk, 1.0, C2, ld, nullptr, 0, st);
}

// rows [r0, r0+nr) of M[:, cb : cb+L] := (...) P = (...) - ((...) V) T V^H
template <class FT>
static cudaError_t rq_update(FT* M, int64_t ld, int r0, int nr, int cb, int L, int nbk, const FT* V,
                             int64_t ldv, const FT* Tb, int ldt, const WsBuf& w, cudaStream_t st) {
  if (nr <= 0) return cudaSuccess;
  cudaError_t e;
  FT* W = static_cast<FT*>(w.W);
  FT* W2 = static_cast<FT*>(w.W2);
  FT* work = static_cast<FT*>(w.work);
  FT* Ma = M + r0 + int64_t(cb) * ld;
  if (skinny_fits<FT>(L, nbk, nr, w)) {
    if ((e = skinny_w2<FT, true>(Ma, ld, V, ldv, L, nbk, nr, Tb, ldt, W2, w, st))) return e;
    return gemm<FT>(false, true, nr, L, nbk, -1.0, W2, nr, V, ldv, 1.0, Ma, ld, nullptr, 0, st);
  }
  if ((e = gemm<FT>(false, false, nr, nbk, L, 1.0, Ma, ld, V, ldv, 0.0, W, nr, work, w.wn, st))) return e;
  if ((e = gemm<FT>(false, false, nr, nbk, nbk, 1.0, W, nr, Tb, ldt, 0.0, W2, nr, nullptr, 0, st))) return e;
  return gemm<FT>(false, true, nr, L, nbk, -1.0, W2, nr, V, ldv, 1.0, Ma, ld, nullptr, 0, st);
}

// merged T of an outer block (nbo reflectors, V: L x nbo at ld L) into Tout
template <class FT>
static cudaError_t block_t(int L, int nbo, const FT* V, const FT* Tp, FT* Tout, const Streams& S,
                          cudaStream_t st) {
  FT* G = static_cast<FT*>(S.G);
  const WsBuf& w = S.ws[1];
  cudaError_t e;
  if ((e = gemm<FT>(true, false, nbo, nbo, L, 1.0, V, L, V, L, 0.0, G, nbo, static_cast<FT*>(w.work), w.wn,
                    st)))
    return e;
  if constexpr (tr<FT>::cplx) return tmerge_c64(nbo, G, nbo, Tp, Tout, NBO, st);
  else if constexpr (std::is_same<FT, double>::value) return tmerge_f64(nbo, G, nbo, Tp, Tout, NBO, st);
  else return tmerge_f32(nbo, G, nbo, Tp, Tout, NBO, st);
}

// QR of M[0:rows, 0:k] (columns), trailing columns up to cend.
// V of outer block B: (rows - B NBO) x NBO dense at ld rows - B NBO (zeros
// above each panel's unit diagonal); panel j's T at Tbuf + j NB NB.
template <class FT>
static cudaError_t qr_stage(FT* M, int64_t ld, int rows, int k, int cend, FT* Vbuf, FT* Tbuf,
                            FT* TBig, FT* taus, Fac<FT>& F, const Streams& S) {
  cudaError_t e;
  const int nob = (k + NBO - 1) / NBO;
  if (nob == 0) return cudaSuccess;
  std::vector<size_t> voff(nob + 1, 0);
  for (int B = 0; B < nob; ++B) voff[B + 1] = voff[B] + size_t(rows - B * NBO) * NBO;
  if ((e = cudaMemsetAsync(Vbuf, 0, voff[nob] * sizeof(FT), S.st))) return e;
  auto TBof = [&](int B) { return TBig + size_t(B) * NBO * NBO; };  // kept for the cascade
  // panels, inner updates and the T merge of block B, on stream s
  // MLSB_FACT_PROF=1: split of the block factorizations (panels | inner updates | T merge)
  static const bool bprof = getenv("MLSB_FACT_PROF") != nullptr;
  std::vector<cudaEvent_t> be;
  auto bmark = [&](cudaStream_t s2) {
    if (!bprof) return;
    cudaEvent_t x;
    cudaEventCreate(&x);
    cudaEventRecord(x, s2);
    be.push_back(x);
  };
  auto factor_block = [&](int B, cudaStream_t s, const WsBuf& w) -> cudaError_t {
    const int j0 = B * NBO, nbo = std::min(NBO, k - j0), L0 = rows - j0;
    FT* Vb = Vbuf + voff[B];
    cudaError_t e2;
    for (int c = j0; c < j0 + nbo; c += NB) {
      const int nbk = std::min(NB, j0 + nbo - c), o = c - j0;
      FT* Vp = Vb + o + int64_t(o) * L0;
      FT* Tp = Tbuf + size_t(c / NB) * NB * NB;
      bmark(s);
      if ((e2 = panel_factor<FT>(M, ld, c, c, rows - c, nbk, false, taus + c, Vp, L0, Tp, 0, s))) return e2;
      bmark(s);
      if ((e2 = qr_update<FT>(M, ld, c, rows - c, nbk, c + nbk, j0 + nbo - c - nbk, Vp, L0, Tp, NB, w, s)))
        return e2;
    }
    bmark(s);
    if (nbo > NB && (e2 = block_t<FT>(L0, nbo, Vb, Tbuf + size_t(j0 / NB) * NB * NB, TBof(B), S, s))) return e2;
    bmark(s);
    return cudaSuccess;
  };
  if ((e = factor_block(0, S.st, S.ws[0]))) return e;
  // MLSB_FACT_PROF=1: per-block event split of the look-ahead pipeline (stderr)
  static const bool fprof = getenv("MLSB_FACT_PROF") != nullptr;
  std::vector<cudaEvent_t> fe;
  auto fmark = [&](cudaStream_t s) {
    if (!fprof) return;
    cudaEvent_t x;
    cudaEventCreate(&x);
    cudaEventRecord(x, s);
    fe.push_back(x);
  };
  for (int B = 0; B < nob; ++B) {
    const int j0 = B * NBO, nbo = std::min(NBO, k - j0), L0 = rows - j0;
    const FT* Vb = Vbuf + voff[B];
    const FT* Tb = nbo > NB ? TBof(B) : Tbuf + size_t(j0 / NB) * NB * NB;
    const int ldt = nbo > NB ? NBO : NB;
    if (B > 0) cudaStreamWaitEvent(S.st, S.ev_pan, 0);  // block B was factored on s2
    F.b.push_back(Blk<FT>{Vb, L0, L0, nbo, Tb, j0, ldt});
    const int c1 = j0 + nbo;
    if (B + 1 < nob) {
      const int nbn = std::min(NBO, k - c1);
      fmark(S.st);
      if ((e = qr_update<FT>(M, ld, j0, L0, nbo, c1, nbn, Vb, L0, Tb, ldt, S.ws[0], S.st))) return e;
      cudaEventRecord(S.ev_upd, S.st);
      fmark(S.st);
      cudaStreamWaitEvent(S.s2, S.ev_upd, 0);
      if ((e = factor_block(B + 1, S.s2, S.ws[1]))) return e;
      cudaEventRecord(S.ev_pan, S.s2);
      fmark(S.s2);
      set_gemm_cta_cap(kTrailCap);  // leave SM slots to the look-ahead stream
      e = qr_update<FT>(M, ld, j0, L0, nbo, c1 + nbn, cend - c1 - nbn, Vb, L0, Tb, ldt, S.ws[0], S.st);
      set_gemm_cta_cap(0);
      if (e) return e;
      fmark(S.st);
    } else {
      if ((e = qr_update<FT>(M, ld, j0, L0, nbo, c1, cend - c1, Vb, L0, Tb, ldt, S.ws[0], S.st))) return e;
    }
  }
  if (fprof && !fe.empty()) {
    cudaEventSynchronize(fe.back());
    double tn = 0, tf = 0, tt = 0;
    for (size_t i = 0; i + 3 < fe.size(); i += 4) {
      float a = 0, b = 0, c = 0;
      cudaEventElapsedTime(&a, fe[i], fe[i + 1]);
      cudaEventElapsedTime(&b, fe[i + 1], fe[i + 2]);
      cudaEventElapsedTime(&c, fe[i + 1], fe[i + 3]);
      tn += a, tf += b, tt += c;
    }
    float wall = 0;
    cudaEventElapsedTime(&wall, fe.front(), fe.back());
    fprintf(stderr, "[fact] qr_stage rows %d k %d: next-cols updates %.3f ms, block factorizations %.3f ms, "
                    "trailing updates %.3f ms, wall %.3f ms\n", rows, k, tn, tf, tt, wall);
    // per block: 4 x (panel, inner update) then T merge = 10 marks
    double tp = 0, ti = 0, tm = 0;
    for (size_t i = 0; i + 9 < be.size(); i += 10) {
      for (int q = 0; q < 4; ++q) {
        float a2 = 0, b2 = 0;
        cudaEventElapsedTime(&a2, be[i + 2 * q], be[i + 2 * q + 1]);
        cudaEventElapsedTime(&b2, be[i + 2 * q + 1], be[i + 2 * q + 2]);
        tp += a2, ti += b2;
      }
      float c2 = 0;
      cudaEventElapsedTime(&c2, be[i + 8], be[i + 9]);
      tm += c2;
    }
    fprintf(stderr, "[fact]   blocks: panels %.3f ms, inner updates %.3f ms, Gram + T merge %.3f ms\n", tp, ti, tm);
    for (auto x : be) cudaEventDestroy(x);
    for (auto x : fe) cudaEventDestroy(x);
  }
  return cudaSuccess;
}

// RQ of the block rows [rb, rb+rr) x columns [cb, cb+cc) (rows bottom-up), applied
// from the right to every row above; panels of NB rows from the bottom, NBO / NB
// panels per outer block.
template <class FT>
static cudaError_t rq_stage(FT* M, int64_t ld, int rb, int rr, int cb, int cc, FT* Vbuf, FT* Tbuf,
                            FT* TBig, FT* taus, Fac<FT>& F, const Streams& S) {
  cudaError_t e;
  const int kk = std::min(rr, cc);
  const int np = (kk + NB - 1) / NB;
  if (np == 0) return cudaSuccess;
  constexpr int PPB = NBO / NB;  // panels per outer block
  const int nob = (np + PPB - 1) / PPB;
  // panel b: reflectors j in [r1 - nbk, r1), r1 = kk - b NB; row of j = rb + rr - kk + j,
  // pivot column = cb + cc - kk + j
  auto r1_of = [&](int b) { return kk - b * NB; };
  auto nbk_of = [&](int b) { return std::min(NB, r1_of(b)); };
  auto row_first = [&](int b) { return int64_t(rb + rr - kk + r1_of(b) - 1); };
  auto pcmax = [&](int b) { return int64_t(cb + cc - kk + r1_of(b) - 1); };
  auto L_of = [&](int b) { return int(pcmax(b) - cb + 1); };
  auto above_of = [&](int b) { return int(row_first(b) - (nbk_of(b) - 1)); };  // rows [0, above)
  auto pend = [&](int B) { return std::min(np, (B + 1) * PPB); };
  auto nbo_of = [&](int B) { return r1_of(B * PPB) - (pend(B) < np ? r1_of(pend(B)) : 0); };
  std::vector<size_t> voff(nob + 1, 0);
  for (int B = 0; B < nob; ++B) voff[B + 1] = voff[B] + size_t(L_of(B * PPB)) * NBO;
  if ((e = cudaMemsetAsync(Vbuf, 0, voff[nob] * sizeof(FT), S.st))) return e;
  auto TBof = [&](int B) { return TBig + size_t(B) * NBO * NBO; };  // kept for the cascade
  auto Vp_of = [&](int b) { return Vbuf + voff[b / PPB] + size_t(b % PPB) * NB * L_of((b / PPB) * PPB); };
  auto factor_block = [&](int B, cudaStream_t s, const WsBuf& w) -> cudaError_t {
    const int L0 = L_of(B * PPB), bend = pend(B);
    cudaError_t e2;
    for (int b = B * PPB; b < bend; ++b) {
      FT* Tp = Tbuf + size_t(b) * NB * NB;
      if ((e2 = panel_factor<FT>(M, ld, row_first(b), pcmax(b), L_of(b), nbk_of(b), true,
                                 taus + size_t(b) * NB, Vp_of(b), L0, Tp, cb, s)))
        return e2;
      const int nrem = above_of(b) - above_of(bend - 1);  // rows of the block's later panels
      if ((e2 = rq_update<FT>(M, ld, above_of(b) - nrem, nrem, cb, L_of(b), nbk_of(b), Vp_of(b), L0, Tp, NB,
                              w, s)))
        return e2;
    }
    const int nbo = nbo_of(B);
    if (nbo > NB) return block_t<FT>(L0, nbo, Vbuf + voff[B], Tbuf + size_t(B * PPB) * NB * NB, TBof(B), S, s);
    return cudaSuccess;
  };
  if ((e = factor_block(0, S.st, S.ws[0]))) return e;
  for (int B = 0; B < nob; ++B) {
    if (B > 0) cudaStreamWaitEvent(S.st, S.ev_pan, 0);
    const int L0 = L_of(B * PPB), nbo = nbo_of(B), bend = pend(B);
    const FT* Vb = Vbuf + voff[B];
    const FT* Tb = nbo > NB ? TBof(B) : Tbuf + size_t(B * PPB) * NB * NB;
    const int ldt = nbo > NB ? NBO : NB;
    F.b.push_back(Blk<FT>{Vb, L0, L0, nbo, Tb, 0, ldt});
    const int above = above_of(bend - 1);
    if (B + 1 < nob) {
      const int nbn = nbo_of(B + 1);
      if ((e = rq_update<FT>(M, ld, above - nbn, nbn, cb, L0, nbo, Vb, L0, Tb, ldt, S.ws[0], S.st))) return e;
      cudaEventRecord(S.ev_upd, S.st);
      cudaStreamWaitEvent(S.s2, S.ev_upd, 0);
      if ((e = factor_block(B + 1, S.s2, S.ws[1]))) return e;
      cudaEventRecord(S.ev_pan, S.s2);
      set_gemm_cta_cap(kTrailCap);
      e = rq_update<FT>(M, ld, 0, above - nbn, cb, L0, nbo, Vb, L0, Tb, ldt, S.ws[0], S.st);
      set_gemm_cta_cap(0);
      if (e) return e;
    } else {
      if ((e = rq_update<FT>(M, ld, 0, above, cb, L0, nbo, Vb, L0, Tb, ldt, S.ws[0], S.st))) return e;
    }
  }
  return cudaSuccess;
}

// ------------------------------------------------------------- GMRES-IR (LSE)
// gmres_refine_lse (krylov.hpp:545-689) on the large path's factors: the
// augmented operator is applied matrix-free to the scaled binary64 A, B (exact
// division, like the reference's scaled copy); the preconditioners work on the
// binary32 factors widened to binary64 (promote_factors is exact).
struct GmBuf {
  double* p = nullptr;
  cudaStream_t s = nullptr;
  ~GmBuf() {
    if (p) cudaFreeAsync(p, s);
  }
};

__global__ void k_add_div(const double* x, double s, int n, double* y) {  // y += x / s
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) y[i] += x[i] / s;
}
__global__ void k_finite_flag(const double* x, int n, int* flag) {
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT)
    if (!isfinite(x[i])) atomicOr(flag, 1);
}

// dst (rows x cols, ld rows) = src / s with exact division: the GMRES operator's
// scaled copy of A, B (the reference scales a copy, krylov.hpp:557-563), made
// once per solve so the operator streams it (k_resid_stream, multiply by 1.0)
// instead of dividing every entry on every application
__global__ void k_div_copy(const double* src, int64_t lds, int rows, int cols, double s, double* dst) {
  const int64_t total = int64_t(rows) * cols;
  for (int64_t e = int64_t(blockIdx.x) * KT + threadIdx.x; e < total; e += int64_t(gridDim.x) * KT) {
    const int64_t j = e / rows, i = e - j * rows;
    dst[e] = src[i + j * lds] / s;
  }
}

// out = [alpha u1 + A u3; B u3; A^T u1 + B^T u2]  (augmented_operator::apply, krylov.hpp:62-77)
// gA, gB: the exactly scaled copies (so sA = sB = 1 and the stream kernel's
// scaling multiplies by 1.0); otherwise the raw inputs with exact division
static void gm_op(int m, int n, int p, double alpha, const double* gA, const double* gB,
                  int64_t lda, int64_t ldb, double sA, double sB, const double* u, double* out,
                  double* rpart, double* cpart, cudaStream_t st) {
  const int R = m + p, C = n;
  const int ntr = (R + RTR - 1) / RTR, ntc = (C + RTC - 1) / RTC;
  dim3 g2(ntr, ntc);
  if (sA == 1.0 && sB == 1.0) {
    const Stack<double> S{gA, gB, lda, ldb, m, true, 1.0, 1.0};
    k_resid_stream<double><<<g2, KT, 0, st>>>(S, R, C, u + R, u, rpart, cpart);
  } else {
    const StackX SX{gA, gB, lda, ldb, m, true, sA, sB};
    k_resid_tile<double, StackX><<<g2, KT, 0, st>>>(SX, R, C, u + R, u, rpart, cpart);
  }
  k_op_reduce<<<nblk(R + C), KT, 0, st>>>(R, C, m, ntc, ntr, rpart, cpart, u, alpha, out);
}

static void gm_dot(const double* x, const double* y, int n, double* part, int nb, double* out,
                   cudaStream_t st) {
  k_dot_part<<<nb, KT, 0, st>>>(x, y, n, part);
  k_dot_final<<<1, 32, 0, st>>>(part, nb, out);
}

// block-diagonal split preconditioner for LSE (bd_lse_apply, krylov.hpp:253-287):
// m >= n through T1 = T(0:n, 0:n); n > m with U = [T1 T2; 0 I] and
// Y = [T1(n-p:m, n-p:m) T2(n-p:m, :); 0 I] (k = m - (n - p)) applied blockwise
template <class FT>
static void gm_bd(bool left, int m, int n, int p, double alpha, const FT* M, int64_t ld,
                  const Fac<FT>& FQ, const double* w, double* out, double* ta, double* tb,
                  double* ypart, cudaStream_t st, double* tc = nullptr) {
  const double ra = 1.0 / sqrt(alpha), sa = sqrt(alpha);
  const Mask up{1, 0, 0};
  const Mask none{0, 0, 0};
  if (n > m) {
    const int d = n - m, q0 = n - p, k = m - q0;  // Y's leading block: rows/cols q0 .. m of T
    double* o2 = out + m;
    double* o3 = out + m + p;
    if (left) {
      // o2 = Y (R^-1 w2): top T1(q0:m, q0:m) v_t + T2(q0:m, :) v_b, bottom v_b
      k_copy<double><<<nblk(p), KT, 0, st>>>(w + m, p, ta);
      trsv<FT, double>(M, ld, m, n - p, p, false, ta, st);
      gemv_n<FT, double>(M, ld, q0, k, q0, k, up, ta, o2, st);
      gemv_n<FT, double>(M, ld, q0, k, m, d, none, ta + k, tc, st);
      k_axpy<<<nblk(k), KT, 0, st>>>(1.0, tc, k, o2);
      k_copy<double><<<nblk(d), KT, 0, st>>>(ta + k, d, o2 + k);
      // o3 = U^-T (Q w3): top T1^T o_t = q_t, bottom q_b - T2^T o_t
      k_copy<double><<<nblk(n), KT, 0, st>>>(w + m + p, n, tb);
      apply_F<FT, double>(FQ, true, tb, ypart, st);
      trsv<FT, double>(M, ld, 0, 0, m, true, tb, st);
      gemv_h<FT, double>(M, ld, 0, m, m, d, none, tb, tc, st);
      k_sub<double><<<nblk(d), KT, 0, st>>>(tb + m, tc, d, tb + m);
      k_copy<double><<<nblk(n), KT, 0, st>>>(tb, n, o3);
    } else {
      // o2 = R^-T (Y^T w2): top T1(q0:m,q0:m)^T w_t, bottom T2(q0:m,:)^T w_t + w_b
      gemv_h<FT, double>(M, ld, q0, k, q0, k, up, w + m, ta, st);
      gemv_h<FT, double>(M, ld, q0, k, m, d, none, w + m, tc, st);
      k_copy<double><<<nblk(d), KT, 0, st>>>(w + m + k, d, ta + k);
      k_axpy<<<nblk(d), KT, 0, st>>>(1.0, tc, d, ta + k);
      trsv<FT, double>(M, ld, m, n - p, p, true, ta, st);
      k_copy<double><<<nblk(p), KT, 0, st>>>(ta, p, o2);
      // o3 = Q^T (U^-1 w3): bottom w_b, top T1^-1 (w_t - T2 w_b)
      k_copy<double><<<nblk(n), KT, 0, st>>>(w + m + p, n, tb);
      gemv_n<FT, double>(M, ld, 0, m, m, d, none, tb + m, tc, st);
      k_sub<double><<<nblk(m), KT, 0, st>>>(tb, tc, m, tb);
      trsv<FT, double>(M, ld, 0, 0, m, false, tb, st);
      apply_F<FT, double>(FQ, false, tb, ypart, st);
      k_copy<double><<<nblk(n), KT, 0, st>>>(tb, n, o3);
    }
    k_scal<<<nblk(m), KT, 0, st>>>(ra, w, m, out);
    k_scal<<<nblk(p), KT, 0, st>>>(ra, o2, p, o2);
    k_scal<<<nblk(n), KT, 0, st>>>(sa, o3, n, o3);
    return;
  }
  // the p-block (R solve) and the n-block (Q apply + T1 solve) are independent:
  // the p-block runs on the auxiliary stream when there is one
  cudaStream_t sp = CzAux::s ? CzAux::s : st;
  if (CzAux::s) {
    cudaEventRecord(CzAux::fork, st);
    cudaStreamWaitEvent(sp, CzAux::fork, 0);
  }
  if (left) {
    {
      CzLane ln(CzAux::s ? 1 : CzScratch::lane);
      k_copy<double><<<nblk(p), KT, 0, sp>>>(w + m, p, ta);
      trsv<FT, double>(M, ld, m, n - p, p, false, ta, sp);                 // t = R^-1 w2
      gemv_n<FT, double>(M, ld, n - p, p, n - p, p, up, ta, out + m, sp);  // o2 = T(n-p:n, n-p:n) t
      k_scal<<<nblk(p), KT, 0, sp>>>(ra, out + m, p, out + m);
    }
    k_copy<double><<<nblk(n), KT, 0, st>>>(w + m + p, n, tb);
    apply_F<FT, double>(FQ, true, tb, ypart, st);                        // q = Q w3
    trsv<FT, double>(M, ld, 0, 0, n, true, tb, st);                      // T1^T o3 = q
    k_scal<<<nblk(m), KT, 0, st>>>(ra, w, m, out);
    k_scal<<<nblk(n), KT, 0, st>>>(sa, tb, n, out + m + p);
  } else {
    {
      CzLane ln(CzAux::s ? 1 : CzScratch::lane);
      gemv_h<FT, double>(M, ld, n - p, p, n - p, p, up, w + m, ta, sp);    // t = T(..)^T w2
      trsv<FT, double>(M, ld, m, n - p, p, true, ta, sp);                  // R^T o2 = t
      k_scal<<<nblk(p), KT, 0, sp>>>(ra, ta, p, out + m);
    }
    k_copy<double><<<nblk(n), KT, 0, st>>>(w + m + p, n, tb);
    trsv<FT, double>(M, ld, 0, 0, n, false, tb, st);                     // T1 t3 = w3
    apply_F<FT, double>(FQ, false, tb, ypart, st);                       // o3 = Q^T t3
    k_scal<<<nblk(m), KT, 0, st>>>(ra, w, m, out);
    k_scal<<<nblk(n), KT, 0, st>>>(sa, tb, n, out + m + p);
  }
  if (CzAux::s) {
    cudaEventRecord(CzAux::join, sp);
    cudaStreamWaitEvent(st, CzAux::join, 0);
  }
}

// left preconditioner (left_lse_apply, krylov.hpp:209-230)
template <class FT>
static void gm_left(int m, int n, int p, double alpha, const FT* M, int64_t ld, const Fac<FT>& FZ,
                    const Fac<FT>& FQ, const double* w, double* out, double* const* cv,
                    double* ypart, cudaStream_t st) {
  const double ia = 1.0 / alpha;
  const Mask up{1, 0, 0};
  double *ta = cv[0], *tb = cv[1], *tc = cv[2], *td = cv[3], *te = cv[4], *tf = cv[5];
  // t = B^+ w2 = Q^T [0; R^-1 w2]
  k_copy<double><<<nblk(p), KT, 0, st>>>(w + m, p, ta);
  trsv<FT, double>(M, ld, m, n - p, p, false, ta, st);
  k_fill<double><<<nblk(n), KT, 0, st>>>(tb, n, 0.0);
  k_copy<double><<<nblk(p), KT, 0, st>>>(ta, p, tb + n - p);
  apply_F<FT, double>(FQ, false, tb, ypart, st);
  // h = w1 - A t, A t = Z T Q t
  k_copy<double><<<nblk(n), KT, 0, st>>>(tb, n, tc);
  apply_F<FT, double>(FQ, true, tc, ypart, st);
  gemv_n<FT, double>(M, ld, 0, m, 0, n, up, tc, td, st);
  apply_F<FT, double>(FZ, false, td, ypart, st);
  k_sub<double><<<nblk(m), KT, 0, st>>>(w, td, m, td);
  // g = w3 - (1/alpha) A^T h, A^T h = Q^T T^T Z^T h
  k_copy<double><<<nblk(m), KT, 0, st>>>(td, m, te);
  apply_F<FT, double>(FZ, true, te, ypart, st);
  gemv_h<FT, double>(M, ld, 0, m, 0, n, up, te, tf, st);
  apply_F<FT, double>(FQ, false, tf, ypart, st);
  k_scal<<<nblk(n), KT, 0, st>>>(-ia, tf, n, tf);
  k_axpy<<<nblk(n), KT, 0, st>>>(1.0, w + m + p, n, tf);
  // o2 = (B^+)^T g = R^-T (Q g)(n-p:n)
  apply_F<FT, double>(FQ, true, tf, ypart, st);
  trsv<FT, double>(M, ld, m, n - p, p, true, tf + (n - p), st);
  k_scal<<<nblk(m), KT, 0, st>>>(ia, td, m, out);
  k_copy<double><<<nblk(p), KT, 0, st>>>(tf + (n - p), p, out + m);
  k_copy<double><<<nblk(n), KT, 0, st>>>(tb, n, out + m + p);
}

// lse_correction_solve (lse.hpp:83-128) at binary64 on the widened factors
template <class FT>
static void gm_cascade(int m, int n, int p, const FT* M, int64_t ld, const Fac<FT>& FZ,
                       const Fac<FT>& FQ, const double* f1, const double* f2, const double* f3,
                       double* const* cv, double* ypart, double* dr, double* dv, double* dx,
                       cudaStream_t st) {
  const int k = n - p;
  const Mask none{0, 0, 0};
  double *u = cv[0], *w = cv[1], *y2 = cv[2], *q1 = cv[3], *t4 = cv[4], *y = cv[5], *tq = cv[7];
  k_copy<double><<<nblk(n), KT, 0, st>>>(f3, n, u);
  k_copy<double><<<nblk(m), KT, 0, st>>>(f1, m, w);
  k_copy<double><<<nblk(p), KT, 0, st>>>(f2, p, y2);
  apply_F<FT, double>(FQ, true, u, ypart, st);                   // u = Q f3
  apply_F<FT, double>(FZ, true, w, ypart, st);                   // w = Z^T f1
  trsv<FT, double>(M, ld, m, n - p, p, false, y2, st);           // R y2 = f2
  k_copy<double><<<nblk(k), KT, 0, st>>>(u, k, q1);
  trsv<FT, double>(M, ld, 0, 0, k, true, q1, st);                // T11^T q1 = u1
  gemv_n<FT, double>(M, ld, 0, k, k, p, none, y2, t4, st);
  gemv_n<FT, double>(M, ld, k, m - k, k, p, Mask{1, 0, 0}, y2, t4 + k, st);
  k_subsub<double><<<nblk(k), KT, 0, st>>>(w, q1, t4, k, y);
  k_copy<double><<<nblk(k), KT, 0, st>>>(q1, k, w);
  k_sub<double><<<nblk(m - k), KT, 0, st>>>(w + k, t4 + k, m - k, w + k);
  k_copy<double><<<nblk(m), KT, 0, st>>>(w, m, dr);
  k_copy<double><<<nblk(p), KT, 0, st>>>(y2, p, y + k);
  trsv<FT, double>(M, ld, 0, 0, k, false, y, st);
  apply_F<FT, double>(FQ, false, y, ypart, st);                  // dx = Q^T y
  apply_F<FT, double>(FZ, false, dr, ypart, st);                 // dr = Z q
  gemv_h<FT, double>(M, ld, 0, k, k, p, none, w, t4, st);
  gemv_h<FT, double>(M, ld, k, m - k, k, p, Mask{1, 0, 0}, w + k, tq, st);
  k_addsub<double><<<nblk(p), KT, 0, st>>>(t4, tq, u + k, p, t4);
  trsv<FT, double>(M, ld, m, n - p, p, true, t4, st);            // R^T dv = s
  k_copy<double><<<nblk(n), KT, 0, st>>>(y, n, dx);
  k_copy<double><<<nblk(p), KT, 0, st>>>(t4, p, dv);
}

// ---------------------------------------------------------- GMRES-IR (GLS)
// Augmented vectors are ordered [y-block (p); z-block (n); x-block (m)]
// (krylov.hpp:24-26).  In the packed GLS factors M (n x (m+p)): R = M[0:m, 0:m],
// T(i, j) = M[i, m + j]; F_Z (the driver's QR factor) is Q, F_Q (the RQ factor)
// is Z^H: Q x = apply_F(FZ, false), Q^T x = apply_F(FZ, true), Z x =
// apply_F(FQ, true), Z^T x = apply_F(FQ, false).

// out = op(u) (augmented_operator::apply, GLS branch); tmp holds [u3; u1]
static void gm_op_gls(int n, int m, int p, double alpha, const double* gW, const double* gV, int64_t ldw,
                      int64_t ldv, double sW, double sV, const double* u, double* out, double* tmp,
                      double* rpart, double* cpart, cudaStream_t st) {
  const int R = n, C = m + p;
  const int ntr = (R + RTR - 1) / RTR, ntc = (C + RTC - 1) / RTC;
  k_copy<double><<<nblk(m), KT, 0, st>>>(u + p + n, m, tmp);
  k_copy<double><<<nblk(p), KT, 0, st>>>(u, p, tmp + m);
  dim3 g2(ntr, ntc);
  if (sW == 1.0 && sV == 1.0) {
    const Stack<double> S{gW, gV, ldw, ldv, m, false, 1.0, 1.0};
    k_resid_stream<double><<<g2, KT, 0, st>>>(S, R, C, tmp, u + p, rpart, cpart);
  } else {
    const StackX SX{gW, gV, ldw, ldv, m, false, sW, sV};
    k_resid_tile<double, StackX><<<g2, KT, 0, st>>>(SX, R, C, tmp, u + p, rpart, cpart);
  }
  k_op_reduce_gls<<<nblk(p + n + m), KT, 0, st>>>(n, m, p, ntc, ntr, rpart, cpart, u, alpha, out);
}

// block-diagonal split preconditioner for GLS (bd_gls_apply, krylov.hpp:288-321),
// both cases: n <= p (T2 = T(0:n, p-n:p)) and n > p (U = [I T1; 0 T2],
// Y = [I T1(:, 0:k); 0 T2(0:k, 0:k)], k = m - (n - p), applied blockwise)
template <class FT>
static void gm_bd_gls(bool left, int n, int m, int p, double alpha, const FT* M, int64_t ld,
                      const Fac<FT>& FZ, const double* w, double* out, double* ta, double* tb,
                      double* tc, double* ypart, cudaStream_t st) {
  const double ra = 1.0 / sqrt(alpha), sa = sqrt(alpha);
  const Mask none{0, 0, 0};
  const int kk = std::min(n, p);
  const Mask rqm{2, n - kk, m + (p - kk)};
  double* o2 = out + p;
  double* o3 = out + p + n;
  k_copy<double><<<nblk(n), KT, 0, st>>>(w + p, n, ta);      // w2
  k_copy<double><<<nblk(m), KT, 0, st>>>(w + p + n, m, tb);  // w3
  if (n <= p) {
    if (left) {
      apply_F<FT, double>(FZ, true, ta, ypart, st);                  // q = Q^T w2
      trsv<FT, double>(M, ld, 0, m + p - n, n, false, ta, st);       // T2 o2 = q
      trsv<FT, double>(M, ld, 0, 0, m, true, tb, st);                // R^T t = w3
      gemv_h<FT, double>(M, ld, 0, m, m + p - n, m, rqm, tb, o3, st);  // o3 = T(0:m, p-n:p-n+m)^T t
      k_copy<double><<<nblk(n), KT, 0, st>>>(ta, n, o2);
    } else {
      trsv<FT, double>(M, ld, 0, m + p - n, n, true, ta, st);        // T2^T t = w2
      apply_F<FT, double>(FZ, false, ta, ypart, st);                 // o2 = Q t
      gemv_n<FT, double>(M, ld, 0, m, m + p - n, m, rqm, tb, o3, st);  // t3 = T(0:m, p-n:..) w3
      trsv<FT, double>(M, ld, 0, 0, m, false, o3, st);               // o3 = R^-1 t3
      k_copy<double><<<nblk(n), KT, 0, st>>>(ta, n, o2);
    }
  } else {
    const int d = n - p, k = m - d;
    if (left) {
      // o2 = U^-1 (Q^T w2): bottom T2 o_b = q_b, top o_t = q_t - T1 o_b
      apply_F<FT, double>(FZ, true, ta, ypart, st);
      trsv<FT, double>(M, ld, d, m, p, false, ta + d, st);
      gemv_n<FT, double>(M, ld, 0, d, m, p, none, ta + d, tc, st);
      k_sub<double><<<nblk(d), KT, 0, st>>>(ta, tc, d, ta);
      k_copy<double><<<nblk(n), KT, 0, st>>>(ta, n, o2);
      // o3 = Y^T (R^-T w3): top v_t, bottom T1(:,0:k)^T v_t + T2(0:k,0:k)^T v_b
      trsv<FT, double>(M, ld, 0, 0, m, true, tb, st);
      gemv_h<FT, double>(M, ld, 0, d, m, k, none, tb, tc, st);
      gemv_h<FT, double>(M, ld, d, k, m, k, rqm, tb + d, tc + k, st);
      k_copy<double><<<nblk(d), KT, 0, st>>>(tb, d, o3);
      k_fill<double><<<nblk(k), KT, 0, st>>>(o3 + d, k, 0.0);
      k_axpy<<<nblk(k), KT, 0, st>>>(1.0, tc, k, o3 + d);
      k_axpy<<<nblk(k), KT, 0, st>>>(1.0, tc + k, k, o3 + d);
    } else {
      // o2 = Q U^-T w2: top t_t = w2_t, bottom T2^T t_b = w2_b - T1^T t_t
      gemv_h<FT, double>(M, ld, 0, d, m, p, none, ta, tc, st);
      k_sub<double><<<nblk(p), KT, 0, st>>>(ta + d, tc, p, ta + d);
      trsv<FT, double>(M, ld, d, m, p, true, ta + d, st);
      apply_F<FT, double>(FZ, false, ta, ypart, st);
      k_copy<double><<<nblk(n), KT, 0, st>>>(ta, n, o2);
      // o3 = R^-1 (Y w3): top w3_t + T1(:,0:k) w3_b, bottom T2(0:k,0:k) w3_b
      gemv_n<FT, double>(M, ld, 0, d, m, k, none, tb + d, tc, st);
      gemv_n<FT, double>(M, ld, d, k, m, k, rqm, tb + d, o3 + d, st);
      k_copy<double><<<nblk(d), KT, 0, st>>>(tb, d, o3);
      k_axpy<<<nblk(d), KT, 0, st>>>(1.0, tc, d, o3);
      trsv<FT, double>(M, ld, 0, 0, m, false, o3, st);
    }
  }
  k_scal<<<nblk(p), KT, 0, st>>>(ra, w, p, out);
  k_scal<<<nblk(n), KT, 0, st>>>(sa, o2, n, o2);
  k_scal<<<nblk(m), KT, 0, st>>>(ra, o3, m, o3);
}

// left preconditioner for GLS (left_gls_apply, krylov.hpp:232-250)
template <class FT>
static void gm_left_gls(int n, int m, int p, double alpha, const FT* M, int64_t ld, const Fac<FT>& FZ,
                        const Fac<FT>& FQ, const double* w, double* out, double* const* cv, double* ypart,
                        cudaStream_t st) {
  const double ia = 1.0 / alpha;
  const int kk = std::min(n, p);
  const Mask rqm{2, n - kk, m + (p - kk)};
  double *t = cv[0], *q = cv[1], *h = cv[2], *g = cv[3], *u = cv[4];
  // t = W^+T w3 = Q [R^-T w3; 0]
  k_fill<double><<<nblk(n), KT, 0, st>>>(t, n, 0.0);
  k_copy<double><<<nblk(m), KT, 0, st>>>(w + p + n, m, t);
  trsv<FT, double>(M, ld, 0, 0, m, true, t, st);
  apply_F<FT, double>(FZ, false, t, ypart, st);
  // h = w1 - V^T t, V^T t = Z^T T^T Q^T t
  k_copy<double><<<nblk(n), KT, 0, st>>>(t, n, q);
  apply_F<FT, double>(FZ, true, q, ypart, st);
  gemv_h<FT, double>(M, ld, 0, n, m, p, rqm, q, h, st);
  apply_F<FT, double>(FQ, false, h, ypart, st);
  k_sub<double><<<nblk(p), KT, 0, st>>>(w, h, p, h);
  // g = w2 - (1/alpha) V h, V h = Q T Z h
  k_copy<double><<<nblk(p), KT, 0, st>>>(h, p, u);
  apply_F<FT, double>(FQ, true, u, ypart, st);
  gemv_n<FT, double>(M, ld, 0, n, m, p, rqm, u, g, st);
  apply_F<FT, double>(FZ, false, g, ypart, st);
  k_scal<<<nblk(n), KT, 0, st>>>(-ia, g, n, g);
  k_axpy<<<nblk(n), KT, 0, st>>>(1.0, w + p, n, g);
  // o3 = W^+ g = R^-1 (Q^T g)(0:m)
  apply_F<FT, double>(FZ, true, g, ypart, st);
  trsv<FT, double>(M, ld, 0, 0, m, false, g, st);
  k_scal<<<nblk(p), KT, 0, st>>>(ia, h, p, out);
  k_copy<double><<<nblk(n), KT, 0, st>>>(t, n, out + p);
  k_copy<double><<<nblk(m), KT, 0, st>>>(g, m, out + p + n);
}

// gls_correction_solve (Algorithm 3, gls.hpp:106-154) at binary64 on the widened
// factors: (f1 p, f2 n, f3 m) -> (dy p, dz n, dx m)
template <class FT>
static void gm_cascade_gls(int n, int m, int p, const FT* M, int64_t ld, const Fac<FT>& FZ,
                           const Fac<FT>& FQ, const double* f1, const double* f2, const double* f3,
                           double* const* cv, double* ypart, double* dy, double* dz, double* dx,
                           cudaStream_t st) {
  const int nm = n - m, kp = p - n + m;
  const int kk = std::min(n, p);
  const Mask none{0, 0, 0};
  const Mask rqm{2, n - kk, m + (p - kk)};
  double *u = cv[0], *w = cv[1], *h1 = cv[2], *g2 = cv[3], *t4 = cv[4], *r2 = cv[5], *g = cv[6],
         *r1v = cv[7], *tq = cv[8], *hh = cv[9];
  k_copy<double><<<nblk(n), KT, 0, st>>>(f2, n, u);
  k_copy<double><<<nblk(p), KT, 0, st>>>(f1, p, w);
  k_copy<double><<<nblk(m), KT, 0, st>>>(f3, m, h1);
  apply_F<FT, double>(FZ, true, u, ypart, st);                        // u = Q^T f2
  apply_F<FT, double>(FQ, true, w, ypart, st);                        // w = Z f1
  trsv<FT, double>(M, ld, 0, 0, m, true, h1, st);                     // R^T h1 = f3
  k_copy<double><<<nblk(nm), KT, 0, st>>>(u + m, nm, g2);
  trsv<FT, double>(M, ld, m, m + kp, nm, false, g2, st);              // T22 g2 = u2
  gemv_h<FT, double>(M, ld, 0, m, m + kp, nm, none, h1, t4, st);       // T12^T h1
  gemv_h<FT, double>(M, ld, 0, m, m, kp, rqm, h1, tq, st);             // T11^T h1
  k_subsub<double><<<nblk(nm), KT, 0, st>>>(w + kp, g2, t4, nm, r2);  // w2 - g2 - T12^T h1
  k_sub<double><<<nblk(kp), KT, 0, st>>>(w, tq, kp, g);               // g1 = w1 - T11^T h1
  k_copy<double><<<nblk(nm), KT, 0, st>>>(g2, nm, g + kp);
  trsv<FT, double>(M, ld, m, m + kp, nm, true, r2, st);               // T22^T h2 = ...
  k_copy<double><<<nblk(p), KT, 0, st>>>(g, p, hh);
  apply_F<FT, double>(FQ, false, hh, ypart, st);                       // dy = Z^T g
  gemv_n<FT, double>(M, ld, 0, m, m, kp, rqm, g, t4, st);              // T11 g1
  gemv_n<FT, double>(M, ld, 0, m, m + kp, nm, none, g2, tq, st);       // T12 g2
  k_sub2<double><<<nblk(m), KT, 0, st>>>(u, t4, tq, m, r1v);          // u1 - (T11 g1 + T12 g2)
  trsv<FT, double>(M, ld, 0, 0, m, false, r1v, st);                   // R dx = ...
  k_copy<double><<<nblk(m), KT, 0, st>>>(h1, m, u);
  k_copy<double><<<nblk(nm), KT, 0, st>>>(r2, nm, u + m);
  apply_F<FT, double>(FZ, false, u, ypart, st);                        // Q [h1; h2]
  k_copy<double><<<nblk(p), KT, 0, st>>>(hh, p, dy);
  k_scal<<<nblk(n), KT, 0, st>>>(-1.0, u, n, dz);                      // dz = -Q h
  k_copy<double><<<nblk(m), KT, 0, st>>>(r1v, m, dx);
}

// One GMRES step's MGS sweep as a single cooperative launch (k_mgs); false
// when it does not apply (MLSB_CASCADE_OLD, N beyond one 1024-row slice per
// SM, no scratch) and the per-vector dot/axpy launches run instead.
static bool mgs_fused(const double* Vb, int N, int k, double* w, double* h, double* part, int nb,
                      cudaStream_t st) {
  if (!cascade_on() || !CzScratch::cnt) return false;
  const int G = (N + 1023) / 1024;
  if (G > sm_count() || 2 * G > nb) return false;
  int* cnt = CzScratch::cnt + 2 * (2 * CZ_CNT) + CZ_CNT - 1;  // lane 2's last trsv flag slot
  if (cudaMemsetAsync(cnt, 0, sizeof(int), st) != cudaSuccess) return false;
  void* args[] = {(void*)&Vb, (void*)&N, (void*)&k, (void*)&w, (void*)&h, (void*)&part, (void*)&cnt};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_mgs), dim3(G), dim3(1024), args, 0, st) ==
         cudaSuccess;
}

// Full MGS-GMRES with Givens rotations (gmres, krylov.hpp:436-512; rel_tol
// 1e-6, max_iter N) on the augmented system: `lp` is the left preconditioner
// (or the split preconditioner's left half), `rp` the right half (kind 2);
// the solution is added to wacc.  Basis vectors live on the device, the
// Hessenberg column and the rotations on the host (one small D2H per step).
template <class OP, class LP, class RP>
static int gmres_core(int kind, int N, const double* rhs, double* wacc, const OP& op, const LP& lp,
                      const RP& rp, double* t2, double* t3, double* t4, double* part, int nb, double* hdev,
                      GmBuf& bas, int& cap, int64_t* its_out, cudaStream_t st) {
  cudaError_t e;
  auto grow = [&](int need) -> cudaError_t {
    if (need <= cap) return cudaSuccess;
    int nc = cap ? cap : 32;
    while (nc < need) nc *= 2;
    if (nc > N + 1) nc = N + 1;
    double* np_ = nullptr;
    cudaError_t ee = cudaMallocAsync(reinterpret_cast<void**>(&np_), sizeof(double) * size_t(N) * nc, st);
    if (ee) return ee;
    if (bas.p) {
      cudaMemcpyAsync(np_, bas.p, sizeof(double) * size_t(N) * cap, cudaMemcpyDeviceToDevice, st);
      cudaFreeAsync(bas.p, st);
    }
    bas.p = np_;
    bas.s = st;
    cap = nc;
    return cudaSuccess;
  };
  if ((e = grow(2))) return MLSB_ERR_CUDA;
  auto V = [&](int i) { return bas.p + size_t(i) * N; };
  lp(rhs, V(0));
  gm_dot(V(0), V(0), N, part, nb, hdev, st);
  double hb[2];
  cudaMemcpyAsync(hb, hdev, 8, cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st))) return MLSB_ERR_CUDA;
  const double beta = sqrt(hb[0]);
  int64_t its = 0;
  if (beta != 0.0) {
    k_scal<<<nblk(N), KT, 0, st>>>(1.0 / beta, V(0), N, V(0));
    std::vector<std::vector<double>> H;
    std::vector<double> gc, gs, g{beta}, hh;
    int k = 0;
    for (; k < N; ++k) {
      if ((e = grow(k + 2))) return MLSB_ERR_CUDA;
      if (kind == 2) {
        rp(V(k), t3);
        op(t3, t4);
      } else {
        op(V(k), t4);
      }
      lp(t4, t2);
      if (!mgs_fused(bas.p, N, k, t2, hdev, part, nb, st)) {
        for (int i = 0; i <= k; ++i) {  // modified Gram-Schmidt
          gm_dot(t2, V(i), N, part, nb, hdev + i, st);
          k_axpy_dev<<<nblk(N), KT, 0, st>>>(hdev + i, V(i), N, t2);
        }
        gm_dot(t2, t2, N, part, nb, hdev + k + 1, st);
      }
      hh.assign(k + 2, 0.0);
      cudaMemcpyAsync(hh.data(), hdev, sizeof(double) * (k + 2), cudaMemcpyDeviceToHost, st);
      if ((e = cudaStreamSynchronize(st))) return MLSB_ERR_CUDA;
      std::vector<double> h(hh);
      const double hk1 = sqrt(hh[k + 1]);
      h[k + 1] = hk1;
      const bool breakdown = hk1 <= 0x1p-52 * beta;
      for (int i = 0; i < k; ++i) {
        const double t = gc[i] * h[i] + gs[i] * h[i + 1];
        h[i + 1] = -gs[i] * h[i] + gc[i] * h[i + 1];
        h[i] = t;
      }
      const double r = std::hypot(h[k], h[k + 1]);
      const double c = r == 0.0 ? 1.0 : h[k] / r;
      const double s = r == 0.0 ? 0.0 : h[k + 1] / r;
      gc.push_back(c);
      gs.push_back(s);
      h[k] = r;
      h[k + 1] = 0.0;
      g.push_back(-s * g[k]);
      g[k] = c * g[k];
      H.push_back(std::move(h));
      its = k + 1;
      if (std::abs(g[k + 1]) <= 1e-6 * beta) {
        ++k;
        break;
      }
      if (breakdown) {
        ++k;
        break;
      }
      k_scal<<<nblk(N), KT, 0, st>>>(1.0 / hk1, t2, N, V(k + 1));
    }
    // back-substitute H y = g over the k columns, x = sum y_i V_i
    std::vector<double> y(k, 0.0);
    for (int jj = k; jj-- > 0;) {
      double sacc = g[jj];
      for (int i = jj + 1; i < k; ++i) sacc -= H[i][jj] * y[i];
      y[jj] = sacc / H[jj][jj];
    }
    k_fill<double><<<nblk(N), KT, 0, st>>>(t3, N, 0.0);
    for (int i = 0; i < k; ++i) k_axpy<<<nblk(N), KT, 0, st>>>(y[i], V(i), N, t3);
    if (kind == 2) {
      rp(t3, t4);
      k_axpy<<<nblk(N), KT, 0, st>>>(1.0, t4, N, wacc);
    } else {
      k_axpy<<<nblk(N), KT, 0, st>>>(1.0, t3, N, wacc);
    }
  }
  *its_out = its;
  return MLSB_OK;
}

// One GMRES-IR correction for LSE (krylov.hpp:640-681): rhs from the residual
// blocks, optional cascade initial guess (left), GMRES, and the state update.
template <class FT>
static int gmres_correction(int kind, int m, int n, int p, double alpha, const FT* M, int64_t ld,
                            const Fac<FT>& FZ, const Fac<FT>& FQ, const double* gA, const double* gB,
                            int64_t lda, int64_t ldb, double sA, double sB, const double* rout,
                            const double* cout, double* sw, double* su, double* rhs, double* wacc,
                            double* t1, double* t2, double* t3, double* t4, double* part, int nb,
                            double* hdev, GmBuf& bas, int& cap, double* const* cv, double* ypart,
                            double* rpart, double* cpart, int* flag, int64_t* its_out,
                            cudaStream_t st) {
  const int N = m + p + n;
  const double sqa = sqrt(alpha);
  cudaError_t e;
  k_scal<<<nblk(m + p), KT, 0, st>>>(sqa, rout, m + p, rhs);
  k_scal<<<nblk(n), KT, 0, st>>>(1.0 / sqa, cout, n, rhs + m + p);
  k_fill<double><<<nblk(N), KT, 0, st>>>(wacc, N, 0.0);
  auto op = [&](const double* in, double* o) {
    gm_op(m, n, p, alpha, gA, gB, lda, ldb, sA, sB, in, o, rpart, cpart, st);
  };
  if (kind == 1) {  // cascade initial guess: the left preconditioner is singular on null(B)
    gm_cascade<FT>(m, n, p, M, ld, FZ, FQ, rout, rout + m, cout, cv, ypart, t1, t1 + m, t1 + m + p, st);
    k_scal<<<nblk(m), KT, 0, st>>>(1.0 / sqa, t1, m, wacc);
    k_scal<<<nblk(p), KT, 0, st>>>(-1.0 / sqa, t1 + m, p, wacc + m);
    k_scal<<<nblk(n), KT, 0, st>>>(sqa, t1 + m + p, n, wacc + m + p);
    op(wacc, t2);
    k_axpy<<<nblk(N), KT, 0, st>>>(-1.0, t2, N, rhs);
  }
  auto lp = [&](const double* in, double* o) {
    if (kind == 2) gm_bd<FT>(true, m, n, p, alpha, M, ld, FQ, in, o, cv[8], cv[9], ypart, st, cv[7]);
    else gm_left<FT>(m, n, p, alpha, M, ld, FZ, FQ, in, o, cv, ypart, st);
  };
  auto rp = [&](const double* in, double* o) {
    gm_bd<FT>(false, m, n, p, alpha, M, ld, FQ, in, o, cv[8], cv[9], ypart, st, cv[7]);
  };
  if (int rc = gmres_core(kind, N, rhs, wacc, op, lp, rp, t2, t3, t4, part, nb, hdev, bas, cap, its_out, st))
    return rc;
  // r += sqa w1, v -= sqa w2, x += w3 / sqa (krylov.hpp:677-679), then the finite check
  k_axpy<<<nblk(m), KT, 0, st>>>(sqa, wacc, m, sw);
  k_axpy<<<nblk(p), KT, 0, st>>>(-sqa, wacc + m, p, sw + m);
  k_add_div<<<nblk(n), KT, 0, st>>>(wacc + m + p, sqa, n, su);
  k_finite_flag<<<nblk(m + p), KT, 0, st>>>(sw, m + p, flag);
  k_finite_flag<<<nblk(n), KT, 0, st>>>(su, n, flag);
  if ((e = cudaGetLastError())) return MLSB_ERR_CUDA;
  return MLSB_OK;
}

// One GMRES-IR correction for GLS (krylov.hpp:750-771): rhs = [sqa f1; f2/sqa;
// sqa f3]; left: the cascade's (dy, dz, dx) as initial guess; update
// y += sqa w1, z -= w2/sqa, x += sqa w3.  Driver layout: su = [x (m); y (p)],
// sw = z (n); residual blocks f1 = cout[m:], f2 = rout, f3 = cout[:m].
template <class FT>
static int gmres_correction_gls(int kind, int n, int m, int p, double alpha, const FT* M, int64_t ld,
                                const Fac<FT>& FZ, const Fac<FT>& FQ, const double* gW, const double* gV,
                                int64_t ldw, int64_t ldv, double sW, double sV, const double* rout,
                                const double* cout, double* sw, double* su, double* rhs, double* wacc,
                                double* t1, double* t2, double* t3, double* t4, double* part, int nb,
                                double* hdev, GmBuf& bas, int& cap, double* const* cv, double* ypart,
                                double* rpart, double* cpart, int* flag, int64_t* its_out,
                                cudaStream_t st) {
  const int N = p + n + m;
  const double sqa = sqrt(alpha);
  cudaError_t e;
  k_scal<<<nblk(p), KT, 0, st>>>(sqa, cout + m, p, rhs);
  k_scal<<<nblk(n), KT, 0, st>>>(1.0 / sqa, rout, n, rhs + p);
  k_scal<<<nblk(m), KT, 0, st>>>(sqa, cout, m, rhs + p + n);
  k_fill<double><<<nblk(N), KT, 0, st>>>(wacc, N, 0.0);
  double* tmp = t1;  // [u3; u1] staging of the operator; t1 is free once the initial guess is folded in
  auto op = [&](const double* in, double* o) {
    gm_op_gls(n, m, p, alpha, gW, gV, ldw, ldv, sW, sV, in, o, tmp, rpart, cpart, st);
  };
  if (kind == 1) {  // the cascade supplies the dz component the left preconditioner cannot see
    gm_cascade_gls<FT>(n, m, p, M, ld, FZ, FQ, cout + m, rout, cout, cv, ypart, t1, t1 + p, t1 + p + n, st);
    k_scal<<<nblk(p), KT, 0, st>>>(1.0 / sqa, t1, p, wacc);
    k_scal<<<nblk(n), KT, 0, st>>>(-sqa, t1 + p, n, wacc + p);
    k_scal<<<nblk(m), KT, 0, st>>>(1.0 / sqa, t1 + p + n, m, wacc + p + n);
    op(wacc, t2);
    k_axpy<<<nblk(N), KT, 0, st>>>(-1.0, t2, N, rhs);
  }
  auto lp = [&](const double* in, double* o) {
    if (kind == 2) gm_bd_gls<FT>(true, n, m, p, alpha, M, ld, FZ, in, o, cv[7], cv[8], cv[9], ypart, st);
    else gm_left_gls<FT>(n, m, p, alpha, M, ld, FZ, FQ, in, o, cv, ypart, st);
  };
  auto rp = [&](const double* in, double* o) {
    gm_bd_gls<FT>(false, n, m, p, alpha, M, ld, FZ, in, o, cv[7], cv[8], cv[9], ypart, st);
  };
  if (int rc = gmres_core(kind, N, rhs, wacc, op, lp, rp, t2, t3, t4, part, nb, hdev, bas, cap, its_out, st))
    return rc;
  k_axpy<<<nblk(p), KT, 0, st>>>(sqa, wacc, p, su + m);                  // y += sqa w1
  k_add_div<<<nblk(n), KT, 0, st>>>(wacc + p, -sqa, n, sw);              // z -= w2 / sqa
  k_axpy<<<nblk(m), KT, 0, st>>>(sqa, wacc + p + n, m, su);              // x += sqa w3
  k_finite_flag<<<nblk(m + p), KT, 0, st>>>(su, m + p, flag);
  k_finite_flag<<<nblk(n), KT, 0, st>>>(sw, n, flag);
  if ((e = cudaGetLastError())) return MLSB_ERR_CUDA;
  return MLSB_OK;
}

// debug: CTA-0 globaltimer stamps of the persistent apply (8 per block)
extern "C" int mlsb_debug_set_czstamps(void* buf) {
  unsigned long long* p = static_cast<unsigned long long*>(buf);
  return int(cudaMemcpyToSymbol(g_czstamp, &p, sizeof(p)));
}

// --------------------------------------------------------------- driver
template <class FT, class WT, class CT>
static int solve(const LargeProblem& P, cudaStream_t st, LargeOut* out) {
  const bool lse = P.kind == KIND_LSE;
  constexpr bool kReal = std::is_same<WT, double>::value;
  constexpr bool kGm = kReal && std::is_same<CT, double>::value;  // GMRES-IR instantiation
  const bool ext = kReal && P.u_r == 2;
  const int m = int(P.m), n = int(P.n), p = int(P.p);
  // GMRES-IR is built for real LSE with m >= n (the first case of the split
  // preconditioner, krylov.hpp:259-269; the reference's configs C1, C3)
  // GMRES-IR: LSE and GLS, both cases of the split preconditioners
  if (P.gmres && !kGm) return MLSB_ERR_UNSUPPORTED;
  const int R = lse ? m + p : n, C = lse ? n : m + p;
  const int64_t ld = R;
  const int kq = lse ? p : std::min(n, p);  // RQ reflectors
  const int kz = lse ? std::min(m, n) : m;  // QR reflectors
  const int nbz = (kz + NB - 1) / NB, nbq = (kq + NB - 1) / NB;
  const int obz = (kz + NBO - 1) / NBO, obq = (kq + NBO - 1) / NBO;  // outer blocks
  const int ntr = (R + RTR - 1) / RTR, ntc = (C + RTC - 1) / RTC;
  const int L = std::max(R, C);
  const size_t wn = size_t(NB) * std::max(R, C) * 64;  // split-K partials (st)
  const size_t wn2 = size_t(NBO) * NBO * 64;            // split-K partials (s2)
  const bool lows = P.u_s == 0;  // correction at u_s = low: one demotion scale (refine.hpp:103-119)
  const bool lowf = P.u_f == 0;  // pre-scaling only at u_f = low (lse.hpp:315-318, gls.hpp:287-289)

  // persistent cascade scratch: 2 x CZ_CNT ints, 2 x CZ_MAXB descriptors, and
  // the per-step partials of k_fac_apply (steps x CTAs x 128, the widest CT)
  const size_t cz_part = size_t(std::max(obz, obq)) * 160 * 128 * sizeof(cd);
  const size_t cz_bytes =
      CZ_LANES * (2 * CZ_CNT * sizeof(int) + cz_part + 256) + 2 * CZ_MAXB * sizeof(BlkD<FT>) + 1024;
  Arena ar;
  const size_t bytes = sizeof(FT) * (size_t(R) * C + size_t(obz) * R * NBO + size_t(obq) * C * NBO +
                                     size_t(nbz + nbq) * NB * NB + size_t(C + R) + 2 * size_t(L) * NBO +
                                     wn + 8 * size_t(L) + 2 * size_t(NB) * NBO + wn2 +
                                     size_t(1 + obz + obq) * NBO * NBO) +
                       sizeof(WT) * (size_t(R) * (6 + ntc) + size_t(C) * (5 + ntr)) +
                       (ext ? 16 * (size_t(ntc) * R + size_t(ntr) * C) + 8 * size_t(R) : 0) +
                       sizeof(CT) * (10 * size_t(L) + WYB * 256 + WYB + 4) +
                       (sizeof(CT) + sizeof(FT)) * size_t(L) * ((L + GNC - 1) / GNC) + 64 * 1024 + 64 * 256 +
                       cz_bytes;
  cudaError_t e = ar.init(bytes + bytes / 4 + (1 << 20), st);
  if (e) return MLSB_ERR_CUDA;
  FT* M = ar.take<FT>(size_t(R) * C);
  FT* VZ = ar.take<FT>(size_t(obz) * R * NBO);
  FT* VQ = ar.take<FT>(size_t(obq) * C * NBO);
  FT* TZ = ar.take<FT>(size_t(nbz) * NB * NB);
  FT* TQ = ar.take<FT>(size_t(nbq) * NB * NB);
  FT* tauZ = ar.take<FT>(C);
  FT* tauQ = ar.take<FT>(size_t(nbq) * NB + R);
  FT* W = ar.take<FT>(size_t(L) * NBO);
  FT* W2 = ar.take<FT>(size_t(L) * NBO);
  FT* gw = ar.take<FT>(wn);
  FT* Ws2 = ar.take<FT>(size_t(NB) * NBO);
  FT* W2s2 = ar.take<FT>(size_t(NB) * NBO);
  FT* gw2 = ar.take<FT>(wn2);
  FT* Gs2 = ar.take<FT>(size_t(NBO) * NBO);
  FT* TZb = ar.take<FT>(size_t(obz) * NBO * NBO);  // merged T per outer block
  FT* TQb = ar.take<FT>(size_t(obq) * NBO * NBO);
  FT* fv[8];
  for (int i = 0; i < 8; ++i) fv[i] = ar.take<FT>(L);
  WT* rinit = ar.take<WT>(R);
  WT* rrow = ar.take<WT>(R);  // row initialisers of the current pass
  WT* rout = ar.take<WT>(R);
  WT* sw = ar.take<WT>(R);
  WT* wvec = ar.take<WT>(R);
  WT* cinit = ar.take<WT>(C);
  WT* cout = ar.take<WT>(C);
  WT* su = ar.take<WT>(C);
  WT* rpart = ar.take<WT>(size_t(ntc) * R);
  WT* cpart = ar.take<WT>(size_t(ntr) * C);
  WT* gvec = ar.take<WT>(C);
  // u_r = extended (real only): double-double tile partials and the low
  // words of the row initialisers
  double2* rpartX = ext ? ar.take<double2>(size_t(ntc) * R) : nullptr;
  double2* cpartX = ext ? ar.take<double2>(size_t(ntr) * C) : nullptr;
  double* rlo = ext ? ar.take<double>(R) : nullptr;
  CT* cv[10];
  for (int i = 0; i < 10; ++i) cv[i] = ar.take<CT>(L);
  CT* ypart = ar.take<CT>(WYB * 256 + WYB + 4);  // partials | z | ticket
  const size_t gsn = size_t(L) * ((L + GNC - 1) / GNC);
  CT* gscr = ar.take<CT>(gsn);
  FT* gscr_f = ar.take<FT>(gsn);
  char* small = ar.take<char>(64 * 1024);
  if (!small) return MLSB_ERR_CUDA;
  unsigned long long* bits = reinterpret_cast<unsigned long long*>(small);  // [8]
  double* parts = reinterpret_cast<double*>(small + 1024);                   // [>= 2*grid]
  double* nsum = reinterpret_cast<double*>(small + 32 * 1024);               // [8]
  int* flags = reinterpret_cast<int*>(small + 33 * 1024);                    // [8]
  StopOut* so = reinterpret_cast<StopOut*>(small + 34 * 1024);
  cudaMemsetAsync(small, 0, 64 * 1024, st);
  cudaMemsetAsync(ypart, 0, sizeof(CT) * (WYB * 256 + WYB + 4), st);  // apply tickets start at 0
  int* cz_cnt = ar.take<int>(CZ_LANES * 2 * CZ_CNT);
  BlkD<FT>* cz_desc = ar.take<BlkD<FT>>(2 * CZ_MAXB);
  char* cz_p = ar.take<char>(CZ_LANES * cz_part);
  if (!cz_p) return MLSB_ERR_CUDA;
  CzScratchGuard czg(cz_cnt, cz_p, cz_part);
  GemvScratchGuard<CT> gsg_c(gscr, gsn);
  std::unique_ptr<GemvScratchGuard<FT>> gsg_f;
  if constexpr (!std::is_same<FT, CT>::value) gsg_f.reset(new GemvScratchGuard<FT>(gscr_f, gsn));

  const WT* gA = static_cast<const WT*>(P.A);
  const WT* gB = static_cast<const WT*>(P.B);
  const WT* gb = static_cast<const WT*>(P.b);
  const WT* gd = static_cast<const WT*>(P.d);
  cudaEvent_t ev[8];
  for (auto& x : ev) cudaEventCreate(&x);
  cudaEventRecord(ev[0], st);

  // ---------------------------------------------------------- pre-scaling
  const int rows1 = lse ? m : n, cols1 = lse ? n : m;  // A (LSE) / W (GLS)
  const int rows2 = lse ? p : n, cols2 = lse ? n : p;  // B / V
  const int grid = 148 * 4;
  k_maxabs<WT><<<grid, KT, 0, st>>>(gA, P.lda, rows1, cols1, bits + 0);
  k_maxabs<WT><<<grid, KT, 0, st>>>(gB, P.ldb, rows2, cols2, bits + 1);
  if (lse) k_maxabs<WT><<<grid, KT, 0, st>>>(gb, m, m, 1, bits + 2);
  else k_maxabs<WT><<<grid, KT, 0, st>>>(gd, n, n, 1, bits + 2);
  unsigned long long hb[3];
  cudaMemcpyAsync(hb, bits, sizeof(hb), cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st))) return MLSB_ERR_CUDA;
  auto asd = [](unsigned long long b) {
    double v;
    memcpy(&v, &b, 8);
    return v == 0.0 ? 1.0 : v;
  };
  double sA = lowf ? asd(hb[0]) : 1.0;
  const double c1 = lowf ? asd(hb[2]) : 1.0;
  double sB = lowf ? asd(hb[1]) : 1.0;
  if (P.gmres) {
    // the GMRES drivers balance the blocks by their Frobenius norms:
    // LSE s_B = s_A ||B||_F / ||A||_F (krylov.hpp:558-563), GLS s_W = s_V ||W||_F / ||V||_F (:685-688)
    k_cast<FT, WT><<<grid, KT, 0, st>>>(gA, P.lda, rows1, cols1, 1.0, M, ld, parts);
    k_sum_parts<<<1, 32, 0, st>>>(parts, grid, nsum + 0);
    k_cast<FT, WT><<<grid, KT, 0, st>>>(gB, P.ldb, rows2, cols2, 1.0, lse ? M + m : M + int64_t(m) * ld, ld,
                                        parts + grid);
    k_sum_parts<<<1, 32, 0, st>>>(parts + grid, grid, nsum + 1);
    double hr[2];
    cudaMemcpyAsync(hr, nsum, sizeof(hr), cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st))) return MLSB_ERR_CUDA;
    const double nAr = hr[0] > 0 ? sqrt(hr[0]) : 1.0, nBr = hr[1] > 0 ? sqrt(hr[1]) : 1.0;
    if (lse) sB = sA * nBr / nAr;
    else sA = sB * nAr / nBr;
  }
  const double c2 = lse ? sB * c1 / sA : c1;  // LSE c_d = s_B c_b / s_A ; GLS c_d
  // right-hand sides (exact division, lse.hpp:326-329)
  if (lse) {
    k_rhs_scale<WT><<<nblk(m), KT, 0, st>>>(gb, m, c1, rinit, nullptr);
    k_rhs_scale<WT><<<nblk(p), KT, 0, st>>>(gd, p, c2, rinit + m, flags + 0);
  } else {
    k_rhs_scale<WT><<<nblk(n), KT, 0, st>>>(gd, n, c2, rinit, nullptr);
  }
  // fp32 factor input and ||A_s||_F, ||B_s||_F
  if (lse) {
    k_cast<FT, WT><<<grid, KT, 0, st>>>(gA, P.lda, m, n, 1.0 / sA, M, ld, parts);
    k_sum_parts<<<1, 32, 0, st>>>(parts, grid, nsum + 0);
    k_cast<FT, WT><<<grid, KT, 0, st>>>(gB, P.ldb, p, n, 1.0 / sB, M + m, ld, parts + grid);
    k_sum_parts<<<1, 32, 0, st>>>(parts + grid, grid, nsum + 1);
  } else {
    k_cast<FT, WT><<<grid, KT, 0, st>>>(gA, P.lda, n, m, 1.0 / sA, M, ld, parts);
    k_sum_parts<<<1, 32, 0, st>>>(parts, grid, nsum + 0);
    k_cast<FT, WT><<<grid, KT, 0, st>>>(gB, P.ldb, n, p, 1.0 / sB, M + int64_t(m) * ld, ld, parts + grid);
    k_sum_parts<<<1, 32, 0, st>>>(parts + grid, grid, nsum + 1);
  }
  // ||b_s||, ||d_s|| through the stop kernel
  {
    StopIn si{};
    if (lse) {
      si.seg[0] = rinit;
      si.len[0] = m;
      si.seg[1] = rinit + m;
      si.len[1] = p;
    } else {
      si.seg[0] = rinit;
      si.len[0] = n;
    }
    k_stop<WT><<<1, 1024, 0, st>>>(si, so, bits + 3, flags + 0);
  }
  double hn[2];
  StopOut hso;
  cudaMemcpyAsync(hn, nsum, sizeof(hn), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&hso, so, sizeof(hso), cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st))) return MLSB_ERR_CUDA;
  if (lse && hso.bad) {
    out->err = MLSB_ERR_INVALID_INPUT;
    return MLSB_OK;
  }
  const double nA = sqrt(hn[0]), nB = sqrt(hn[1]);
  const double nb_ = lse ? hso.nrm[0] : 0.0, nd = lse ? hso.nrm[1] : hso.nrm[0];
  cudaEventRecord(ev[1], st);

  // ---------------------------------------------------------- GRQ / GQR
  Streams SS;
  SS.st = st;
  SS.ws[0] = WsBuf{W, W2, gw, wn};
  SS.ws[1] = WsBuf{Ws2, W2s2, gw2, wn2};
  SS.G = Gs2;
  {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&SS.s2, cudaStreamNonBlocking, hi);
    cudaEventCreateWithFlags(&SS.ev_upd, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&SS.ev_pan, cudaEventDisableTiming);
  }
  struct StreamsGuard {
    Streams& s;
    ~StreamsGuard() {
      cudaStreamDestroy(s.s2);
      cudaEventDestroy(s.ev_upd);
      cudaEventDestroy(s.ev_pan);
    }
  } sguard{SS};
  Fac<FT> FZ, FQ;  // QR factor (Z for LSE, Q for GLS) / RQ factor (Q^H for LSE, Z^H for GLS)
  if (lse) {
    if ((e = rq_stage<FT>(M, ld, m, p, 0, n, VQ, TQ, TQb, tauQ, FQ, SS))) return MLSB_ERR_CUDA;
    if ((e = qr_stage<FT>(M, ld, m, kz, n, VZ, TZ, TZb, tauZ, FZ, SS))) return MLSB_ERR_CUDA;
  } else {
    if ((e = qr_stage<FT>(M, ld, n, kz, m + p, VZ, TZ, TZb, tauZ, FZ, SS))) return MLSB_ERR_CUDA;
    if ((e = rq_stage<FT>(M, ld, 0, n, m, p, VQ, TQ, TQb, tauQ, FQ, SS))) return MLSB_ERR_CUDA;
  }
  if ((e = fac_upload<FT>(FZ, cz_desc, st)) || (e = fac_upload<FT>(FQ, cz_desc + CZ_MAXB, st)))
    return MLSB_ERR_CUDA;
  // the correction's independent applies / solves on three streams, when every
  // piece runs as a persistent launch (each lane owns its scratch)
  const int vec_rows = 32 * int(16 / sizeof(FT) > 0 ? 16 / sizeof(FT) : 1);
  const bool par = cascade_on() && FZ.dev && FQ.dev && int(FZ.hd.size()) <= CZ_CNT &&
                   int(FQ.hd.size()) <= CZ_CNT && (FZ.nrows + vec_rows - 1) / vec_rows <= sm_count() &&
                   (FQ.nrows + vec_rows - 1) / vec_rows <= sm_count() &&
                   (std::max({m, n, p}) + CZT - 1) / CZT <= sm_count() && !getenv("MLSB_CASCADE_SERIAL");
  cudaStream_t cs2 = nullptr, cs3 = nullptr;
  cudaEvent_t cev[6] = {};
  struct CzStreams {
    cudaStream_t& a;
    cudaStream_t& b;
    cudaEvent_t* ev;
    ~CzStreams() {
      if (a) cudaStreamDestroy(a);
      if (b) cudaStreamDestroy(b);
      for (int i = 0; i < 6; ++i)
        if (ev[i]) cudaEventDestroy(ev[i]);
    }
  } czs_guard{cs2, cs3, cev};
  if (par) {
    cudaStreamCreateWithFlags(&cs2, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&cs3, cudaStreamNonBlocking);
    for (int i = 0; i < 6; ++i) cudaEventCreateWithFlags(&cev[i], cudaEventDisableTiming);
  }
  struct CzAuxGuard {
    ~CzAuxGuard() {
      CzAux::s = nullptr;
      CzAux::fork = CzAux::join = nullptr;
    }
  } czaux_guard;
  if (par && P.gmres) {  // GMRES preconditioners: their independent halves on cs2
    CzAux::s = cs2;
    CzAux::fork = cev[4];
    CzAux::join = cev[5];
  }
  // zero pivots in the order of the reference's first failing trsv
  // (LSE: R at lse.hpp:53, then T11 at :60; GLS: T22 at gls.hpp:55, then R at :61)
  const int kl = lse ? n - p : p - n + m;  // LSE: size of T11 ; GLS: column split of T
  {
    k_fill<int><<<1, 32, 0, st>>>(flags + 1, 2, -1);
    if (lse) {
      k_pivot_scan<FT><<<nblk(p), KT, 0, st>>>(M, ld, m, n - p, p, flags + 1);
      k_pivot_scan<FT><<<nblk(kl), KT, 0, st>>>(M, ld, 0, 0, kl, flags + 2);
    } else {
      k_pivot_scan<FT><<<nblk(n - m), KT, 0, st>>>(M, ld, m, m + kl, n - m, flags + 1);
      k_pivot_scan<FT><<<nblk(m), KT, 0, st>>>(M, ld, 0, 0, m, flags + 2);
    }
    int hf[2];
    cudaMemcpyAsync(hf, flags + 1, sizeof(hf), cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st))) return MLSB_ERR_CUDA;
    if (hf[0] >= 0 || hf[1] >= 0) {
      out->err = MLSB_ERR_SINGULAR;
      out->sing = hf[0] >= 0 ? hf[0] : hf[1];
      return MLSB_OK;
    }
  }
  cudaEventRecord(ev[2], st);

  // ---------------------------------------------------------- initial solve at u_f
  FT* ypf = reinterpret_cast<FT*>(ypart);
  const Mask none{0, 0, 0};
  if (lse) {
    const int k = kl;
    FT *bf = fv[0], *y2 = fv[1], *c = fv[2], *t4 = fv[3], *y = fv[4], *rf = fv[5], *gf = fv[6];
    k_convert<WT, FT><<<nblk(m), KT, 0, st>>>(rinit, m, bf);
    k_convert<WT, FT><<<nblk(p), KT, 0, st>>>(rinit + m, p, y2);
    k_copy<FT><<<nblk(m), KT, 0, st>>>(bf, m, c);
    trsv<FT, FT>(M, ld, m, n - p, p, false, y2, st);      // R y2 = d
    apply_F<FT, FT>(FZ, true, c, ypf, st);                   // c = Z^H b
    gemv_n<FT, FT>(M, ld, 0, k, k, p, none, y2, t4, st);    // T12 y2
    k_sub<FT><<<nblk(k), KT, 0, st>>>(c, t4, k, y);
    k_copy<FT><<<nblk(p), KT, 0, st>>>(y2, p, y + k);
    trsv<FT, FT>(M, ld, 0, 0, k, false, y, st);             // T11 y1 = c1 - T12 y2
    apply_F<FT, FT>(FQ, false, y, ypf, st);                  // x = Q^H [y1; y2]  (F_Q = Q^H)
    {
      const int nt = (n + GNC - 1) / GNC;  // gscr_f / gscr hold L * ceil(L / GNC) entries
      FT* part = std::is_same<FT, CT>::value ? reinterpret_cast<FT*>(gscr) : gscr_f;
      k_rowgemv_cast<FT, WT><<<dim3((m + KT - 1) / KT, nt), KT, 0, st>>>(gA, P.lda, m, n, 1.0 / sA, y, part);
      k_rowgemv_red<FT><<<nblk(m), KT, 0, st>>>(part, m, nt, bf, rf);
    }
    k_convert<FT, WT><<<nblk(n), KT, 0, st>>>(y, n, su);
    k_convert<FT, WT><<<nblk(m), KT, 0, st>>>(rf, m, sw);
    // solve_v (lse.hpp:156-165): g = A^H r at u_r, sigma, Q g, R^H v = g(n-p:n)
    {
      Stack<WT> S{gA, gB, P.lda, P.ldb, m, true, 1.0 / sA, 1.0 / sB};
      k_fill<WT><<<nblk(n), KT, 0, st>>>(gvec, n, zero<WT>());
      dim3 g2((m + RTR - 1) / RTR, ntc);
      if constexpr (kReal) {
        if (ext) {  // g = A^T r accumulated in double-double (gemv_extended, matrix.hpp:157-170)
          const StackX SX{gA, gB, P.lda, P.ldb, m, true, sA, sB};
          k_resid_tile_dd<<<g2, KT, 0, st>>>(SX, m, n, gvec, sw, rpartX, cpartX);
          k_resid_reduce_dd<<<nblk(m + n), KT, 0, st>>>(m, n, ntc, (m + RTR - 1) / RTR, rpartX,
                                                         cpartX, nullptr, nullptr, nullptr, nullptr,
                                                         cout);
        }
      }
      if (!ext) {
        if constexpr (tr<WT>::cplx) k_resid_tile<WT><<<g2, KT, 0, st>>>(S, m, n, gvec, sw, rpart, cpart);  // complex128: register budget
      else k_resid_stream<WT><<<g2, KT, 0, st>>>(S, m, n, gvec, sw, rpart, cpart);
        k_resid_reduce<WT><<<nblk(m + n), KT, 0, st>>>(m, n, ntc, (m + RTR - 1) / RTR, rpart, cpart,
                                                       rinit, nullptr, rout, cout);
      }
      cudaMemsetAsync(bits + 4, 0, 8, st);
      k_vmax<WT><<<nblk(n), KT, 0, st>>>(cout, n, bits + 4);
      k_demote<WT, FT><<<nblk(n), KT, 0, st>>>(cout, n, bits + 4, gf);
      apply_F<FT, FT>(FQ, true, gf, ypf, st);                // Q g = F_Q^H g
      trsv<FT, FT>(M, ld, m, n - p, p, true, gf + (n - p), st);
      k_promote<WT, FT><<<nblk(p), KT, 0, st>>>(sw + m, p, gf + (n - p), bits + 4);
    }
  } else {
    const int nm = n - m;
    const int kk = std::min(n, p);
    FT *c = fv[0], *rhs = fv[1], *yv = fv[2], *g = fv[3], *zq = fv[4], *t = fv[5];
    k_convert<WT, FT><<<nblk(n), KT, 0, st>>>(rinit, n, c);
    apply_F<FT, FT>(FZ, true, c, ypf, st);                   // c = Q^H d
    trsv<FT, FT>(M, ld, m, m + kl, nm, false, c + m, st);   // T22 s2 = c2
    gemv_n<FT, FT>(M, ld, 0, m, m + kl, nm, none, c + m, t, st);
    k_sub<FT><<<nblk(m), KT, 0, st>>>(c, t, m, rhs);
    trsv<FT, FT>(M, ld, 0, 0, m, false, rhs, st);           // R x = c1 - T12 s2
    k_fill<FT><<<nblk(kl), KT, 0, st>>>(yv, kl, zero<FT>());
    k_copy<FT><<<nblk(nm), KT, 0, st>>>(c + m, nm, yv + kl);
    apply_F<FT, FT>(FQ, false, yv, ypf, st);                 // y = Z^H s  (F_Z = Z^H)
    // init_z: g = Z y, T22^H v = g2, z = Q [0; v]
    k_copy<FT><<<nblk(p), KT, 0, st>>>(yv, p, g);
    apply_F<FT, FT>(FQ, true, g, ypf, st);                   // Z y = F^H y
    trsv<FT, FT>(M, ld, m, m + kl, nm, true, g + kl, st);
    k_fill<FT><<<nblk(m), KT, 0, st>>>(zq, m, zero<FT>());
    k_copy<FT><<<nblk(nm), KT, 0, st>>>(g + kl, nm, zq + m);
    apply_F<FT, FT>(FZ, false, zq, ypf, st);                 // z = Q zq
    k_convert<FT, WT><<<nblk(m), KT, 0, st>>>(rhs, m, su);
    k_convert<FT, WT><<<nblk(p), KT, 0, st>>>(yv, p, su + m);
    k_convert<FT, WT><<<nblk(n), KT, 0, st>>>(zq, n, sw);
    (void)kk;
  }
  if ((e = cudaGetLastError())) return MLSB_ERR_CUDA;
  cudaEventRecord(ev[3], st);

  // ---------------------------------------------------------- refinement loop
  Stack<WT> S{gA, gB, P.lda, P.ldb, m, lse, 1.0 / sA, 1.0 / sB};
  double best = INFINITY;
  int status = 1;
  int64_t pass = 0;
  out->hist.clear();
  // ------------------------------------------------ GMRES-IR state (LSE)
  // Vectors of the augmented system, N = m + p + n, ordered [r-block; v-block;
  // x-block]; the Krylov basis grows on demand (full, unrestarted MGS-GMRES,
  // krylov.hpp:436-512, max_iter = N).
  const int N = m + p + n;
  GmBuf gbuf, gbas, gsc;
  const double* gAs = nullptr;  // GMRES operator: exactly scaled copies
  const double* gBs = nullptr;
  int64_t ldas = 0, ldbs = 0;
  double *g_rhs = nullptr, *g_w = nullptr, *g_t1 = nullptr, *g_t2 = nullptr, *g_t3 = nullptr,
         *g_t4 = nullptr, *g_part = nullptr, *g_h = nullptr;
  int g_cap = 0;
  double g_alpha = 1.0;
  const int g_nb = 148 * 2;
  if constexpr (kGm) {
    if (P.gmres) {
      gbuf.s = gbas.s = st;
      const size_t nv = size_t(N);
      if ((e = cudaMallocAsync(reinterpret_cast<void**>(&gbuf.p),
                               sizeof(double) * (6 * nv + g_nb + 2 * (size_t(N) + 2)), st)))
        return MLSB_ERR_CUDA;
      // exactly scaled copies of A, B (W, V) for the operator
      const int sr1 = lse ? m : n, sc1 = lse ? n : m, sr2 = lse ? p : n, sc2 = lse ? n : p;
      gsc.s = st;
      if ((e = cudaMallocAsync(reinterpret_cast<void**>(&gsc.p),
                               sizeof(double) * (size_t(sr1) * sc1 + size_t(sr2) * sc2), st)))
        return MLSB_ERR_CUDA;
      k_div_copy<<<148 * 8, KT, 0, st>>>(gA, P.lda, sr1, sc1, sA, gsc.p);
      k_div_copy<<<148 * 8, KT, 0, st>>>(gB, P.ldb, sr2, sc2, sB, gsc.p + size_t(sr1) * sc1);
      gAs = gsc.p;
      gBs = gsc.p + size_t(sr1) * sc1;
      ldas = sr1;
      ldbs = sr2;
      g_rhs = gbuf.p;
      g_w = g_rhs + nv;
      g_t1 = g_w + nv;
      g_t2 = g_t1 + nv;
      g_t3 = g_t2 + nv;
      g_t4 = g_t3 + nv;
      g_part = g_t4 + nv;
      g_h = g_part + g_nb;
      // alpha = alpha_scale * ||r0|| (LSE, krylov.hpp:613) | ||y0|| (GLS, :720)
      if (lse) k_dot_part<<<g_nb, KT, 0, st>>>(sw, sw, m, g_part);
      else k_dot_part<<<g_nb, KT, 0, st>>>(su + m, su + m, p, g_part);
      k_dot_final<<<1, 32, 0, st>>>(g_part, g_nb, g_h);
      double r2 = 0.0;
      cudaMemcpyAsync(&r2, g_h, 8, cudaMemcpyDeviceToHost, st);
      if ((e = cudaStreamSynchronize(st))) return MLSB_ERR_CUDA;
      g_alpha = P.alpha_scale * (r2 > 0.0 ? sqrt(r2) : 1.0);
    }
  }
  out->inner = 0;
  // MLSB_LOOP_PROF=1: CUDA-event split of the first refinement pass (stderr)
  static const bool loop_prof = getenv("MLSB_LOOP_PROF") != nullptr;
  std::vector<std::pair<const char*, cudaEvent_t>> pev;
  auto mark = [&](const char* name) {
    if (!loop_prof || pass != 1) return;
    cudaEvent_t e2;
    cudaEventCreate(&e2);
    cudaEventRecord(e2, st);
    pev.emplace_back(name, e2);
  };
  // per-pass phase events: [pass start, correction start, correction end]
  // -> trace.timing.residual (residual + stop test) and .correction | .gmres
  // (refine.hpp:45-52; lse.hpp:387, :416)
  std::vector<cudaEvent_t> pph;
  auto pmark = [&]() {
    cudaEvent_t e3;
    cudaEventCreate(&e3);
    cudaEventRecord(e3, st);
    pph.push_back(e3);
  };
  struct PphGuard {
    std::vector<cudaEvent_t>& v;
    ~PphGuard() {
      for (auto x : v) cudaEventDestroy(x);
    }
  } pph_guard{pph};
  for (pass = 1; pass <= P.maxit; ++pass) {
    mark("start");
    pmark();
    // row initialisers and weights of this pass
    if (lse) {
      k_sub<WT><<<nblk(m), KT, 0, st>>>(rinit, sw, m, rrow);                  // b - r
      k_copy<WT><<<nblk(p), KT, 0, st>>>(rinit + m, p, rrow + m);             // d
      k_copy<WT><<<nblk(R), KT, 0, st>>>(sw, R, wvec);
      k_neg<WT><<<nblk(m), KT, 0, st>>>(wvec, m);                              // [-r; v]
      k_fill<WT><<<nblk(C), KT, 0, st>>>(cinit, C, zero<WT>());
    } else {
      k_copy<WT><<<nblk(n), KT, 0, st>>>(rinit, n, rrow);                      // d
      k_copy<WT><<<nblk(n), KT, 0, st>>>(sw, n, wvec);                         // z
      k_fill<WT><<<nblk(m), KT, 0, st>>>(cinit, m, zero<WT>());
      k_copy<WT><<<nblk(p), KT, 0, st>>>(su + m, p, cinit + m);
      k_neg<WT><<<nblk(p), KT, 0, st>>>(cinit + m, p);                          // [0; -y]
    }
    dim3 g2(ntr, ntc);
    if constexpr (kReal) {
      if (ext) {  // lse.hpp:200-257 / gls.hpp:178-231
        if (lse) {
          k_sub_dd<<<nblk(m), KT, 0, st>>>(rinit, sw, m, rrow, rlo);  // TwoSum(b, -r)
          k_fill<double><<<nblk(p), KT, 0, st>>>(rlo + m, p, 0.0);
        } else {
          k_fill<double><<<nblk(n), KT, 0, st>>>(rlo, n, 0.0);
        }
        const StackX SX{gA, gB, P.lda, P.ldb, m, lse, sA, sB};
        k_resid_tile_dd<<<g2, KT, 0, st>>>(SX, R, C, su, wvec, rpartX, cpartX);
        k_resid_reduce_dd<<<nblk(R + C), KT, 0, st>>>(R, C, ntc, ntr, rpartX, cpartX, rrow, rlo, cinit,
                                                      rout, cout);
      }
    }
    if (!ext) {
      if constexpr (tr<WT>::cplx) k_resid_tile<WT><<<g2, KT, 0, st>>>(S, R, C, su, wvec, rpart, cpart);  // complex128: register budget
      else k_resid_stream<WT><<<g2, KT, 0, st>>>(S, R, C, su, wvec, rpart, cpart);
      k_resid_reduce<WT><<<nblk(R + C), KT, 0, st>>>(R, C, ntc, ntr, rpart, cpart, rrow, cinit, rout,
                                                     cout);
    }
    mark("residual");
    StopIn si{};
    if (lse) {  // f1, f2, f3 | r, v, x
      si.seg[0] = rout;       si.len[0] = m;
      si.seg[1] = rout + m;   si.len[1] = p;
      si.seg[2] = cout;       si.len[2] = n;
      si.seg[3] = sw;         si.len[3] = m;
      si.seg[4] = sw + m;     si.len[4] = p;
      si.seg[5] = su;         si.len[5] = n;
    } else {    // f1 = cout[m:], f2 = rout, f3 = cout[:m] | x, y, z
      si.seg[0] = cout + m;   si.len[0] = p;
      si.seg[1] = rout;       si.len[1] = n;
      si.seg[2] = cout;       si.len[2] = m;
      si.seg[3] = su;         si.len[3] = m;
      si.seg[4] = su + m;     si.len[4] = p;
      si.seg[5] = sw;         si.len[5] = n;
    }
    si.sigma_mask = 7;
    k_stop<WT><<<1, 1024, 0, st>>>(si, so, bits + 5, flags + 3);
    cudaMemcpyAsync(&hso, so, sizeof(hso), cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st))) return MLSB_ERR_CUDA;
    if (hso.bad) {  // the previous update went non-finite (lse.hpp:417-420)
      status = 2;
      --pass;
      break;
    }
    mark("stop+sync");
    const double g1 = hso.nrm[0], g2n = hso.nrm[1], g3 = hso.nrm[2];
    const double s3 = hso.nrm[3], s4 = hso.nrm[4], s5 = hso.nrm[5];
    double d1, d2, d3;
    if (lse) {  // lse.hpp:272-277, history :384-385
      d1 = nb_ + s3 + nA * s5;
      d2 = nd + nB * s5;
      d3 = nA * s3 + nB * s4;
      out->hist.push_back(g1 * c1);
      out->hist.push_back(g2n * c2);
      out->hist.push_back(g3 * sA * c1);
    } else {    // gls.hpp:246-251, history :343-344
      d1 = s4 + nB * s5;
      d2 = nd + nA * s3 + nB * s4;
      d3 = nA * s5;
      out->hist.push_back(g1 * c2 / sB);
      out->hist.push_back(g2n * c2);
      out->hist.push_back(g3 * sA * c2 / (sB * sB));
    }
    const double tol = P.tol;
    if (g1 <= tol * d1 && g2n <= tol * d2 && g3 <= tol * d3) {
      status = 0;
      break;
    }
    auto ratio = [](double num, double den) {
      if (den > 0.0) return num / den;
      return num == 0.0 ? 0.0 : INFINITY;
    };
    const double r1 = ratio(g1, d1), r2 = ratio(g2n, d2), r3 = ratio(g3, d3);
    const double t12 = r1 < r2 ? r2 : r1, sm = t12 < r3 ? r3 : t12;
    if (!std::isfinite(sm)) {
      status = 2;
      break;
    }
    if (sm < best) best = sm;
    if (sm >= 1e4 * best && best > 0.0) {
      status = 2;
      break;
    }

    pmark();  // correction (or GMRES) starts
    if constexpr (kGm) {
      if (P.gmres) {
        int64_t its = 0;
        int rc = lse ? gmres_correction(P.gmres, m, n, p, g_alpha, M, ld, FZ, FQ, gAs, gBs, ldas, ldbs, 1.0,
                                        1.0, rout, cout, sw, su, g_rhs, g_w, g_t1, g_t2, g_t3, g_t4, g_part,
                                        g_nb, g_h, gbas, g_cap, cv, ypart, rpart, cpart, flags + 3, &its,
                                        st)
                     : gmres_correction_gls(P.gmres, n, m, p, g_alpha, M, ld, FZ, FQ, gAs, gBs, ldas, ldbs,
                                            1.0, 1.0, rout, cout, sw, su, g_rhs, g_w, g_t1, g_t2, g_t3, g_t4,
                                            g_part, g_nb, g_h, gbas, g_cap, cv, ypart, rpart, cpart,
                                            flags + 3, &its, st);
        if (rc) return rc;
        out->inner += its;
        pmark();
        continue;
      }
    }
    // ---- correction at u_s (demotion by one sigma, refine.hpp:103-107)
    const unsigned long long* sb = lows ? bits + 5 : nullptr;
    if (lse && par) {  // Algorithm 1 (lse.hpp:83-128), independent pieces on three streams
      const int k = kl;
      CT *u = cv[0], *w = cv[1], *y2 = cv[2], *q1 = cv[3], *t4 = cv[4], *y = cv[5], *dr = cv[6],
         *tq = cv[7];
      k_demote<WT, CT><<<nblk(n), KT, 0, st>>>(cout, n, sb, u);
      k_demote<WT, CT><<<nblk(m), KT, 0, st>>>(rout, m, sb, w);
      k_demote<WT, CT><<<nblk(p), KT, 0, st>>>(rout + m, p, sb, y2);
      mark("demote");
      cudaEventRecord(cev[0], st);
      cudaStreamWaitEvent(cs2, cev[0], 0);
      cudaStreamWaitEvent(cs3, cev[0], 0);
      {
        CzLane ln(1);
        apply_F<FT, CT>(FQ, true, u, ypart, cs2);                 // u = Q f3 = F^H f3
        k_copy<CT><<<nblk(k), KT, 0, cs2>>>(u, k, q1);
        trsv<FT, CT>(M, ld, 0, 0, k, true, q1, cs2);              // T11^H q1 = u1
      }
      {
        CzLane ln(2);
        trsv<FT, CT>(M, ld, m, n - p, p, false, y2, cs3);         // R y2 = f2
        gemv_n<FT, CT>(M, ld, 0, k, k, p, none, y2, t4, cs3);      // T12 y2
        gemv_n<FT, CT>(M, ld, k, m - k, k, p, Mask{1, 0, 0}, y2, t4 + k, cs3);  // T22 y2
      }
      apply_F<FT, CT>(FZ, true, w, ypart, st);                    // w = Z^H f1
      cudaEventRecord(cev[1], cs2);
      cudaEventRecord(cev[2], cs3);
      cudaStreamWaitEvent(st, cev[1], 0);
      cudaStreamWaitEvent(st, cev[2], 0);
      mark("phaseA");
      k_subsub<CT><<<nblk(k), KT, 0, st>>>(w, q1, t4, k, y);      // y1 rhs = w1 - q1 - T12 y2
      k_copy<CT><<<nblk(k), KT, 0, st>>>(q1, k, w);               // q = [q1; w2 - T22 y2]
      k_sub<CT><<<nblk(m - k), KT, 0, st>>>(w + k, t4 + k, m - k, w + k);
      k_copy<CT><<<nblk(m), KT, 0, st>>>(w, m, dr);
      k_copy<CT><<<nblk(p), KT, 0, st>>>(y2, p, y + k);
      cudaEventRecord(cev[3], st);
      cudaStreamWaitEvent(cs2, cev[3], 0);
      cudaStreamWaitEvent(cs3, cev[3], 0);
      {
        CzLane ln(1);
        apply_F<FT, CT>(FZ, false, dr, ypart, cs2);               // dr = Z q = F q
      }
      {
        CzLane ln(2);
        gemv_h<FT, CT>(M, ld, 0, k, k, p, none, w, t4, cs3);       // T12^H q1
        gemv_h<FT, CT>(M, ld, k, m - k, k, p, Mask{1, 0, 0}, w + k, tq, cs3);  // T22^H q2
        k_addsub<CT><<<nblk(p), KT, 0, cs3>>>(t4, tq, u + k, p, t4);  // s = T12^H q1 + (T22^H q2 - u2)
        trsv<FT, CT>(M, ld, m, n - p, p, true, t4, cs3);           // R^H dv = s
      }
      trsv<FT, CT>(M, ld, 0, 0, k, false, y, st);                 // T11 y1 = ...
      apply_F<FT, CT>(FQ, false, y, ypart, st);                   // dx = Q^H y = F y
      cudaEventRecord(cev[4], cs2);
      cudaEventRecord(cev[5], cs3);
      cudaStreamWaitEvent(st, cev[4], 0);
      cudaStreamWaitEvent(st, cev[5], 0);
      mark("phaseB");
      k_promote_add<WT, CT><<<nblk(m), KT, 0, st>>>(sw, m, dr, sb, false, flags + 3);
      k_promote_add<WT, CT><<<nblk(p), KT, 0, st>>>(sw + m, p, t4, sb, false, flags + 3);
      k_promote_add<WT, CT><<<nblk(n), KT, 0, st>>>(su, n, y, sb, false, flags + 3);
    } else if (lse) {  // Algorithm 1 (lse.hpp:83-128)
      const int k = kl;
      CT *u = cv[0], *w = cv[1], *y2 = cv[2], *q1 = cv[3], *t4 = cv[4], *y = cv[5], *dr = cv[6],
         *tq = cv[7];
      k_demote<WT, CT><<<nblk(n), KT, 0, st>>>(cout, n, sb, u);
      k_demote<WT, CT><<<nblk(m), KT, 0, st>>>(rout, m, sb, w);
      k_demote<WT, CT><<<nblk(p), KT, 0, st>>>(rout + m, p, sb, y2);
      mark("demote");
      apply_F<FT, CT>(FQ, true, u, ypart, st);                  // u = Q f3 = F^H f3
      mark("applyQ");
      apply_F<FT, CT>(FZ, true, w, ypart, st);                  // w = Z^H f1
      mark("applyZ");
      trsv<FT, CT>(M, ld, m, n - p, p, false, y2, st);          // R y2 = f2
      mark("trsvR");
      k_copy<CT><<<nblk(k), KT, 0, st>>>(u, k, q1);
      trsv<FT, CT>(M, ld, 0, 0, k, true, q1, st);               // T11^H q1 = u1
      mark("trsvT11h");
      gemv_n<FT, CT>(M, ld, 0, k, k, p, none, y2, t4, st);       // T12 y2
      gemv_n<FT, CT>(M, ld, k, m - k, k, p, Mask{1, 0, 0}, y2, t4 + k, st);  // T22 y2
      mark("gemv_n x2");
      k_subsub<CT><<<nblk(k), KT, 0, st>>>(w, q1, t4, k, y);      // y1 rhs = w1 - q1 - T12 y2
      k_copy<CT><<<nblk(k), KT, 0, st>>>(q1, k, w);               // q = [q1; w2 - T22 y2]
      k_sub<CT><<<nblk(m - k), KT, 0, st>>>(w + k, t4 + k, m - k, w + k);
      k_copy<CT><<<nblk(m), KT, 0, st>>>(w, m, dr);
      k_copy<CT><<<nblk(p), KT, 0, st>>>(y2, p, y + k);
      mark("elementwise");
      trsv<FT, CT>(M, ld, 0, 0, k, false, y, st);               // T11 y1 = ...
      mark("trsvT11");
      apply_F<FT, CT>(FQ, false, y, ypart, st);                 // dx = Q^H y = F y
      mark("applyQh");
      apply_F<FT, CT>(FZ, false, dr, ypart, st);                // dr = Z q = F q
      mark("applyZh");
      gemv_h<FT, CT>(M, ld, 0, k, k, p, none, w, t4, st);        // T12^H q1
      gemv_h<FT, CT>(M, ld, k, m - k, k, p, Mask{1, 0, 0}, w + k, tq, st);  // T22^H q2
      mark("gemv_h x2");
      k_addsub<CT><<<nblk(p), KT, 0, st>>>(t4, tq, u + k, p, t4);  // s = T12^H q1 + (T22^H q2 - u2)
      trsv<FT, CT>(M, ld, m, n - p, p, true, t4, st);            // R^H dv = s
      mark("trsvRh");
      k_promote_add<WT, CT><<<nblk(m), KT, 0, st>>>(sw, m, dr, sb, false, flags + 3);
      k_promote_add<WT, CT><<<nblk(p), KT, 0, st>>>(sw + m, p, t4, sb, false, flags + 3);
      k_promote_add<WT, CT><<<nblk(n), KT, 0, st>>>(su, n, y, sb, false, flags + 3);
    } else if (par) {  // Algorithm 3 (gls.hpp:106-154), independent pieces on three streams
      const int nm = n - m, kp = kl;
      const int kk = std::min(n, p);
      const Mask rqm{2, n - kk, m + (p - kk)};
      CT *u = cv[0], *w = cv[1], *h1 = cv[2], *g2 = cv[3], *t4 = cv[4], *r2 = cv[5], *g = cv[6],
         *r1v = cv[7], *tq = cv[8], *hh = cv[9];
      k_demote<WT, CT><<<nblk(n), KT, 0, st>>>(rout, n, sb, u);       // f2
      k_demote<WT, CT><<<nblk(p), KT, 0, st>>>(cout + m, p, sb, w);   // f1
      k_demote<WT, CT><<<nblk(m), KT, 0, st>>>(cout, m, sb, h1);      // f3
      mark("demote");
      cudaEventRecord(cev[0], st);
      cudaStreamWaitEvent(cs2, cev[0], 0);
      cudaStreamWaitEvent(cs3, cev[0], 0);
      {
        CzLane ln(1);
        apply_F<FT, CT>(FZ, true, u, ypart, cs2);                       // u = Q^H f2
        k_copy<CT><<<nblk(nm), KT, 0, cs2>>>(u + m, nm, g2);
        trsv<FT, CT>(M, ld, m, m + kp, nm, false, g2, cs2);             // T22 g2 = u2
      }
      {
        CzLane ln(2);
        trsv<FT, CT>(M, ld, 0, 0, m, true, h1, cs3);                    // R^H h1 = f3
        gemv_h<FT, CT>(M, ld, 0, m, m + kp, nm, none, h1, t4, cs3);      // T12^H h1
        gemv_h<FT, CT>(M, ld, 0, m, m, kp, rqm, h1, tq, cs3);            // T11^H h1
      }
      apply_F<FT, CT>(FQ, true, w, ypart, st);                          // w = Z f1 = F^H f1
      cudaEventRecord(cev[1], cs2);
      cudaEventRecord(cev[2], cs3);
      cudaStreamWaitEvent(st, cev[1], 0);
      cudaStreamWaitEvent(st, cev[2], 0);
      mark("phaseA");
      k_subsub<CT><<<nblk(nm), KT, 0, st>>>(w + kp, g2, t4, nm, r2);  // w2 - g2 - T12^H h1
      k_sub<CT><<<nblk(kp), KT, 0, st>>>(w, tq, kp, g);               // g1 = w1 - T11^H h1
      k_copy<CT><<<nblk(nm), KT, 0, st>>>(g2, nm, g + kp);
      k_copy<CT><<<nblk(p), KT, 0, st>>>(g, p, hh);
      cudaEventRecord(cev[3], st);
      cudaStreamWaitEvent(cs2, cev[3], 0);
      cudaStreamWaitEvent(cs3, cev[3], 0);
      {
        CzLane ln(1);
        apply_F<FT, CT>(FQ, false, hh, ypart, cs2);                     // dy = Z^H g = F g
      }
      {
        CzLane ln(2);
        gemv_n<FT, CT>(M, ld, 0, m, m, kp, rqm, g, t4, cs3);             // T11 g1
        gemv_n<FT, CT>(M, ld, 0, m, m + kp, nm, none, g2, tq, cs3);      // T12 g2
        k_sub2<CT><<<nblk(m), KT, 0, cs3>>>(u, t4, tq, m, r1v);        // u1 - (T11 g1 + T12 g2)
        trsv<FT, CT>(M, ld, 0, 0, m, false, r1v, cs3);                  // R dx = ...
      }
      trsv<FT, CT>(M, ld, m, m + kp, nm, true, r2, st);                 // T22^H h2 = ...
      // [h1; h2] is assembled in w (free since the elementwise step above), not
      // in u as the serial order does: the third stream's k_sub2 still reads u
      k_copy<CT><<<nblk(m), KT, 0, st>>>(h1, m, w);
      k_copy<CT><<<nblk(nm), KT, 0, st>>>(r2, nm, w + m);
      apply_F<FT, CT>(FZ, false, w, ypart, st);                          // Q [h1; h2]
      cudaEventRecord(cev[4], cs2);
      cudaEventRecord(cev[5], cs3);
      cudaStreamWaitEvent(st, cev[4], 0);
      cudaStreamWaitEvent(st, cev[5], 0);
      mark("phaseB");
      k_promote_add<WT, CT><<<nblk(m), KT, 0, st>>>(su, m, r1v, sb, false, flags + 3);
      k_promote_add<WT, CT><<<nblk(p), KT, 0, st>>>(su + m, p, hh, sb, false, flags + 3);
      k_promote_add<WT, CT><<<nblk(n), KT, 0, st>>>(sw, n, w, sb, true, flags + 3);  // dz = -Q h
    } else {    // Algorithm 3 (gls.hpp:106-154)
      const int nm = n - m, kp = kl;
      const int kk = std::min(n, p);
      const Mask rqm{2, n - kk, m + (p - kk)};
      CT *u = cv[0], *w = cv[1], *h1 = cv[2], *g2 = cv[3], *t4 = cv[4], *r2 = cv[5], *g = cv[6],
         *r1v = cv[7], *tq = cv[8], *hh = cv[9];
      k_demote<WT, CT><<<nblk(n), KT, 0, st>>>(rout, n, sb, u);       // f2
      k_demote<WT, CT><<<nblk(p), KT, 0, st>>>(cout + m, p, sb, w);   // f1
      k_demote<WT, CT><<<nblk(m), KT, 0, st>>>(cout, m, sb, h1);      // f3
      mark("demote");
      apply_F<FT, CT>(FZ, true, u, ypart, st);                        // u = Q^H f2
      mark("applyQh");
      apply_F<FT, CT>(FQ, true, w, ypart, st);                        // w = Z f1 = F^H f1
      mark("applyZ");
      trsv<FT, CT>(M, ld, 0, 0, m, true, h1, st);                     // R^H h1 = f3
      mark("trsvRh");
      k_copy<CT><<<nblk(nm), KT, 0, st>>>(u + m, nm, g2);
      trsv<FT, CT>(M, ld, m, m + kp, nm, false, g2, st);              // T22 g2 = u2
      gemv_h<FT, CT>(M, ld, 0, m, m + kp, nm, none, h1, t4, st);       // T12^H h1
      gemv_h<FT, CT>(M, ld, 0, m, m, kp, rqm, h1, tq, st);             // T11^H h1
      k_subsub<CT><<<nblk(nm), KT, 0, st>>>(w + kp, g2, t4, nm, r2);  // w2 - g2 - T12^H h1
      k_sub<CT><<<nblk(kp), KT, 0, st>>>(w, tq, kp, g);               // g1 = w1 - T11^H h1
      k_copy<CT><<<nblk(nm), KT, 0, st>>>(g2, nm, g + kp);
      mark("T22+gemv");
      trsv<FT, CT>(M, ld, m, m + kp, nm, true, r2, st);               // T22^H h2 = ...
      k_copy<CT><<<nblk(p), KT, 0, st>>>(g, p, hh);
      mark("trsvT22h");
      apply_F<FT, CT>(FQ, false, hh, ypart, st);                       // dy = Z^H g = F g
      mark("applyZh");
      gemv_n<FT, CT>(M, ld, 0, m, m, kp, rqm, g, t4, st);              // T11 g1
      gemv_n<FT, CT>(M, ld, 0, m, m + kp, nm, none, g2, tq, st);       // T12 g2
      k_sub2<CT><<<nblk(m), KT, 0, st>>>(u, t4, tq, m, r1v);          // u1 - (T11 g1 + T12 g2)
      mark("gemv_n x2");
      trsv<FT, CT>(M, ld, 0, 0, m, false, r1v, st);                   // R dx = ...
      mark("trsvR");
      k_copy<CT><<<nblk(m), KT, 0, st>>>(h1, m, u);
      k_copy<CT><<<nblk(nm), KT, 0, st>>>(r2, nm, u + m);
      apply_F<FT, CT>(FZ, false, u, ypart, st);                        // Q [h1; h2]
      mark("applyQ");
      k_promote_add<WT, CT><<<nblk(m), KT, 0, st>>>(su, m, r1v, sb, false, flags + 3);
      k_promote_add<WT, CT><<<nblk(p), KT, 0, st>>>(su + m, p, hh, sb, false, flags + 3);
      k_promote_add<WT, CT><<<nblk(n), KT, 0, st>>>(sw, n, u, sb, true, flags + 3);  // dz = -Q h
    }
    if ((e = cudaGetLastError())) return MLSB_ERR_CUDA;
    pmark();
    mark("update");
    if (loop_prof && pass == 1) {
      cudaStreamSynchronize(st);
      for (size_t i = 1; i < pev.size(); ++i) {
        float ms2 = 0.f;
        cudaEventElapsedTime(&ms2, pev[i - 1].second, pev[i].second);
        fprintf(stderr, "[loop] %-12s %8.3f ms\n", pev[i].first, ms2);
      }
      for (auto& pe : pev) cudaEventDestroy(pe.second);
      pev.clear();
    }
  }
  if (pass > P.maxit) pass = P.maxit;
  if (status == 1) {
    // maxit reached: the last update's non-finite check (lse.hpp:417-420) has
    // not been read by a stop test yet
    int hbad = 0;
    cudaMemcpyAsync(&hbad, flags + 3, sizeof(int), cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st))) return MLSB_ERR_CUDA;
    if (hbad) status = 2;
  }
  cudaEventRecord(ev[4], st);
  // ---------------------------------------------------------- unscale outputs
  if (lse) {  // lse.hpp:424-426
    k_scale_out<WT><<<nblk(n), KT, 0, st>>>(su, n, c1 / sA, static_cast<WT*>(P.x));
    k_scale_out<WT><<<nblk(m), KT, 0, st>>>(sw, m, c1, static_cast<WT*>(P.r));
    k_scale_out<WT><<<nblk(p), KT, 0, st>>>(sw + m, p, sA * c1 / sB, static_cast<WT*>(P.v));
  } else {    // gls.hpp:382-384
    k_scale_out<WT><<<nblk(m), KT, 0, st>>>(su, m, c2 / sA, static_cast<WT*>(P.x));
    k_scale_out<WT><<<nblk(p), KT, 0, st>>>(su + m, p, c2 / sB, static_cast<WT*>(P.r));
    k_scale_out<WT><<<nblk(n), KT, 0, st>>>(sw, n, c2 / (sB * sB), static_cast<WT*>(P.v));
  }
  cudaEventRecord(ev[5], st);
  if ((e = cudaStreamSynchronize(st))) return MLSB_ERR_CUDA;
  float ms[5];
  for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1]);
  out->phases[5] = (ms[0] + ms[4]) * 1e-3;  // other
  out->phases[0] = ms[1] * 1e-3;            // factorization
  out->phases[1] = ms[2] * 1e-3;            // init
  // the loop split per pass: [start, corr) = residual + stop test, [corr, end)
  // = correction (classical) or GMRES; a pass that stopped has no correction
  double res_ms = 0.0, cor_ms = 0.0;
  for (size_t i = 0; i < pph.size(); i += 3) {
    float a = 0.f, b2 = 0.f;
    const bool has_corr = i + 2 < pph.size() || (i + 2 == pph.size() - 0 && false);
    if (i + 1 < pph.size()) {
      cudaEventElapsedTime(&a, pph[i], pph[i + 1]);
      if (i + 2 < pph.size()) cudaEventElapsedTime(&b2, pph[i + 1], pph[i + 2]);
    } else {  // final pass: residual + stop test up to the loop's end event
      cudaEventElapsedTime(&a, pph[i], ev[4]);
    }
    (void)has_corr;
    res_ms += a;
    cor_ms += b2;
  }
  // whatever of the loop interval the per-pass events do not cover (host-side
  // gaps between passes are on the device timeline too) goes to "residual"
  const double rest = ms[3] - res_ms - cor_ms;
  if (rest > 0.0) res_ms += rest;
  out->phases[2] = res_ms * 1e-3;                  // residual (+ stop test)
  out->phases[3] = P.gmres ? 0.0 : cor_ms * 1e-3;  // correction
  out->phases[4] = P.gmres ? cor_ms * 1e-3 : 0.0;  // gmres
  for (auto& x : ev) cudaEventDestroy(x);
  out->status = status;
  out->iters = pass;
  out->err = MLSB_OK;
  return MLSB_OK;
}

int large_solve(const LargeProblem& P, cudaStream_t st, LargeOut* out) {
  // the extended residual is real-only (the reference has no complex path)
  if (P.u_r == 2 && P.cplx) return MLSB_ERR_UNSUPPORTED;
  if (P.u_f != 0) {  // binary64 factors: FP64 panels and WY GEMMs (real; the reference has no complex path)
    if (P.cplx || P.gmres) return MLSB_ERR_UNSUPPORTED;
    return solve<double, double, double>(P, st, out);
  }
  if (P.cplx) {
    if (P.u_s != 0) return solve<cf, cd, cd>(P, st, out);
    return solve<cf, cd, cf>(P, st, out);
  }
  if (P.u_s != 0 || P.gmres) return solve<float, double, double>(P, st, out);  // GMRES: binary64 factors
  return solve<float, double, float>(P, st, out);
}

}  // namespace lg
}  // namespace mlsb
