// Panel factorization of the blocked GRQ/GQR: NB Householder reflectors of a
// tall panel, factored by ONE thread-block cluster of PCL CTAs (B200 allows 16
// with the non-portable attribute).  The panel (in its "QR view", see
// large_internal.h) is split by rows over the CTAs' shared memory; every
// reflector step needs ONE cluster-wide reduction, done through distributed
// shared memory with double-buffered partials (one cluster.sync per step):
//
//   partials over the CTA's rows r > q of column x = P[:, q]:
//     ||x||^2 (binary64), d_k = x^H P[:, k] for all k, and the pivot row P[q, :]
//   then every CTA forms (redundantly, identically) beta, tau, 1/(alpha-beta)
//   (xLARFG, householder.hpp:30-53), s_k = v^H P[:, k] = P[q,k] + conj(inv) d_k,
//   applies H^H to its rows of the trailing panel columns (householder.hpp:85-95)
//   and records the Gram entries v_k^H v_q = conj(P[q,k]) + inv conj(d_k) (k < q)
//   from which CTA 0 forms T (xLARFT, forward, columnwise) at the end.
//
// The RQ panels of the reference (rows bottom-up, reflectors applied from the
// right, householder.hpp:202-222) are the same computation on the conjugated,
// transposed and reversed row panel (zgerq2's conjugation), so one kernel serves
// both stages.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "large_common.cuh"
#include "large_internal.h"

namespace cg = cooperative_groups;

namespace mlsb {
namespace lg {

constexpr int PNT = 512, PNW = PNT / 32;

template <class T>
struct PanelArgs {
  T* M;
  int64_t ld, r0, c0;
  int L, nb, rc;  // panel rows, reflectors, rows per CTA
  int ncl;        // CTAs in the cluster
  bool rq;
  T* tau;
  T* V;
  int64_t ldv;
  T* Tm;
  int64_t vbase;  // RQ: M column of V row 0
};

template <class T>
__device__ __forceinline__ T ld_view(const PanelArgs<T>& a, int r, int q) {
  return a.rq ? conj_(a.M[(a.r0 - q) + (a.c0 - r) * a.ld]) : a.M[(a.r0 + r) + (a.c0 + q) * a.ld];
}
template <class T>
__device__ __forceinline__ void st_view(const PanelArgs<T>& a, int r, int q, T v) {
  if (a.rq) a.M[(a.r0 - q) + (a.c0 - r) * a.ld] = conj_(v);
  else a.M[(a.r0 + r) + (a.c0 + q) * a.ld] = v;
}

// complex / real xLARFG scalars from alpha and ss = ||x||^2 (binary64 sum)
__device__ __forceinline__ void larfg_s(float alpha, double ss, float& tau, float& inv, float& beta) {
  tau = 0.f;
  inv = 1.f;
  beta = alpha;
  if (ss != 0.0) {
    const float nrm = __fsqrt_rn(float(fma(double(alpha), double(alpha), ss)));
    const float bt = -copysignf(nrm, alpha);
    tau = __fdiv_rn(__fsub_rn(bt, alpha), bt);
    inv = __frcp_rn(__fsub_rn(alpha, bt));
    beta = bt;
  }
}
__device__ __forceinline__ void larfg_s(cf alpha, double ss, cf& tau, cf& inv, cf& beta) {
  tau = cf{0.f, 0.f};
  inv = cf{1.f, 0.f};
  beta = alpha;
  if (ss != 0.0 || alpha.y != 0.f) {
    const double ar = alpha.x, ai = alpha.y;
    const double bt = -copysign(sqrt(ar * ar + ai * ai + ss), ar);
    tau = cf{float((bt - ar) / bt), float(-ai / bt)};
    // 1 / (alpha - beta)
    const double dr = ar - bt, di = ai, den = dr * dr + di * di;
    inv = cf{float(dr / den), float(-di / den)};
    beta = cf{float(bt), 0.f};
  }
}

template <class T>
__global__ void __launch_bounds__(PNT, 1) panel_kernel(PanelArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = int(cl.block_rank());
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int nb = a.nb, L = a.L, rc = a.rc;
  const int rb = rank * rc, re = max(rb, min(L, rb + rc));  // my rows [rb, re)
  const int ldp = rc;
  // smem: P chunk | parts[2] | totals | G | coef
  T* P = reinterpret_cast<T*>(smem);
  const int NV = 2 * NB;  // d (NB) + prow (NB)
  double* partd = reinterpret_cast<double*>(smem + size_t(ldp) * NB * sizeof(T));  // [2] nrm2
  T* part = reinterpret_cast<T*>(partd + 2);                                       // [2][NV]
  T* tot = part + 2 * NV;                                                            // [NV]
  double* totd = reinterpret_cast<double*>(tot + NV);                                // [1]
  T* G = reinterpret_cast<T*>(totd + 2);                                             // [NB][NB]
  T* coef = G + NB * NB;                                                             // [NB]
  T* taus = coef + NB;                                                               // [NB]
  T* wpart = taus + NB;                                                              // [PNW][NB]
  double* wnrm = reinterpret_cast<double*>(wpart + PNW * NB);                        // [PNW]

  // load my rows of the panel (q fastest: coalesced for the RQ view)
  for (int e = tid; e < rc * nb; e += PNT) {
    const int q = a.rq ? e % nb : e / rc;
    const int r = a.rq ? rb + e / nb : rb + e % rc;
    P[(r - rb) + q * ldp] = (r < re) ? ld_view(a, r, q) : zero<T>();
  }
  for (int e = tid; e < NB * NB; e += PNT) G[e] = zero<T>();
  __syncthreads();

  for (int q = 0; q < nb; ++q) {
    const int par = q & 1;
    // ---- local partials: d_k = sum_{r>q} conj(x_r) P[r][k], ||x||^2, pivot row
    const int rlo = max(rb, q + 1);
    const T* xq = P + q * ldp;
    for (int k = w; k < nb; k += PNW) {
      const T* pk = P + k * ldp;
      T acc = zero<T>();
      double an = 0.0;
      for (int r = rlo + l; r < re; r += 32) {
        const T x = xq[r - rb];
        mac(acc, conj_(x), pk[r - rb]);
        if (k == q) an += abs2d(x);
      }
      acc = wsum(acc);
      if (k == q) an = wsum(an);
      if (l == 0) {
        part[par * NV + k] = acc;
        if (k == q) partd[par] = an;
      }
    }
    if (tid < nb) part[par * NV + NB + tid] = (q >= rb && q < re) ? P[(q - rb) + tid * ldp] : zero<T>();
    cl.sync();
    // ---- cluster totals in fixed rank order (identical in every CTA)
    if (tid < 2 * NB) {
      const int k = tid < NB ? tid : tid - NB;
      if (k < nb) {
        T v[PCL];
#pragma unroll
        for (int c = 0; c < PCL; ++c) v[c] = c < a.ncl ? cl.map_shared_rank(part, c)[par * NV + tid] : zero<T>();
        T s = zero<T>();
#pragma unroll
        for (int c = 0; c < PCL; ++c)
          if (c < a.ncl) s = s + v[c];
        tot[tid] = s;
      }
    } else if (tid == 2 * NB) {
      double v[PCL];
#pragma unroll
      for (int c = 0; c < PCL; ++c) v[c] = c < a.ncl ? cl.map_shared_rank(partd, c)[par] : 0.0;
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < PCL; ++c)
        if (c < a.ncl) s += v[c];
      totd[0] = s;
    }
    __syncthreads();
    // ---- reflector scalars (redundant per thread, identical values)
    T tau, inv, beta;
    larfg_s(tot[NB + q], totd[0], tau, inv, beta);
    if (tid < nb) {
      const int k = tid;
      const T dk = tot[k], pk = tot[NB + k];
      if (k > q) {
        const T s = pk + conj_(inv) * dk;  // v^H P[:, k]
        coef[k] = conj_(tau) * s;          // H^H = I - conj(tau) v v^H
      } else if (k < q) {
        G[k + NB * q] = conj_(pk) + inv * conj_(dk);  // v_k^H v_q
      }
      if (k == q) taus[q] = tau;
    }
    __syncthreads();
    // ---- apply H^H to my rows of columns k > q (warp per column, lanes over rows)
    const bool has_tau = !(tau == zero<T>());
    if (has_tau) {
      for (int k = q + 1 + w; k < nb; k += PNW) {
        const T ck = coef[k];
        T* pk = P + k * ldp;
        for (int r = max(rb, q) + l; r < re; r += 32) {
          if (r == q) pk[r - rb] = pk[r - rb] - ck;
          else pk[r - rb] = pk[r - rb] - ck * (inv * xq[r - rb]);
        }
      }
    }
    __syncthreads();
    for (int r = max(rb, q) + tid; r < re; r += PNT) {
      T* pe = P + (r - rb) + q * ldp;
      if (r == q) *pe = beta;
      else if (has_tau) *pe = inv * (*pe);
    }
    __syncthreads();
  }
  // ---- write back the factored panel, the dense reflector block and tau / T
  for (int e = tid; e < rc * nb; e += PNT) {
    const int q = a.rq ? e % nb : e / rc;
    const int r = a.rq ? rb + e / nb : rb + e % rc;
    if (r >= re) continue;
    const T pv = P[(r - rb) + q * ldp];
    st_view(a, r, q, pv);
    const T vv = r < q ? zero<T>() : (r == q ? one<T>() : pv);
    const int64_t vi = a.rq ? (a.c0 - r - a.vbase) : r;
    a.V[vi + q * a.ldv] = vv;
  }
  if (rank == 0) {
    if (tid < nb) a.tau[tid] = taus[tid];
    if (w == 0) {
      // T[q][q] = tau_q ; T[0:q, q] = -tau_q T[0:q, 0:q] G[0:q, q]; lane l owns row l
      T Tr[NB];
#pragma unroll
      for (int k = 0; k < NB; ++k) Tr[k] = zero<T>();
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        if (q < nb) {
          T t = zero<T>();
#pragma unroll
          for (int k = 0; k < q; ++k) mac(t, Tr[k], G[k + NB * q]);
          const T tq = taus[q];
          Tr[q] = l < q ? -(tq * t) : (l == q ? tq : zero<T>());
        }
      }
      if (l < nb)
#pragma unroll
        for (int q = 0; q < NB; ++q)
          if (q < nb) a.Tm[l + q * NB] = Tr[q];
    }
  }
  cl.sync();  // no CTA may exit while others still read its shared memory
}

template <class T>
static size_t panel_smem(int rc) {
  const int NV = 2 * NB;
  return size_t(rc) * NB * sizeof(T) + 2 * sizeof(double) + 2 * NV * sizeof(T) + NV * sizeof(T) +
         2 * sizeof(double) + (NB * NB + 2 * NB + PNW * NB) * sizeof(T) + PNW * sizeof(double) + 64;
}

template <class T>
cudaError_t panel_factor(T* M, int64_t ld, int64_t r0, int64_t c0, int L, int nb, bool rq, T* tau,
                         T* V, int64_t ldv, T* Tm, int64_t vbase, cudaStream_t st) {
  if (nb <= 0 || nb > NB || L < nb) return cudaErrorInvalidValue;
  PanelArgs<T> a;
  a.M = M;
  a.ld = ld;
  a.r0 = r0;
  a.c0 = c0;
  a.L = L;
  a.nb = nb;
  // 16 CTAs (B200's non-portable maximum): the per-step work is the rows each
  // CTA owns, measured cheaper than the extra cluster-barrier cost
  a.ncl = PCL;
  a.rc = (L + PCL - 1) / PCL;
  a.rq = rq;
  a.tau = tau;
  a.V = V;
  a.ldv = ldv;
  a.Tm = Tm;
  a.vbase = vbase;
  const size_t sm = panel_smem<T>(a.rc);
  auto kern = panel_kernel<T>;
  cudaError_t e;
  static bool attr_done[2] = {false, false};
  if (!attr_done[sizeof(T) == 8]) {
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1))) return e;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)))
      return e;
    attr_done[sizeof(T) == 8] = true;
  }
  if (sm > 227 * 1024) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.ncl);
  cfg.blockDim = dim3(PNT);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = a.ncl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template cudaError_t panel_factor<float>(float*, int64_t, int64_t, int64_t, int, int, bool, float*,
                                         float*, int64_t, float*, int64_t, cudaStream_t);
template cudaError_t panel_factor<cf>(cf*, int64_t, int64_t, int64_t, int, int, bool, cf*, cf*,
                                      int64_t, cf*, int64_t, cudaStream_t);

}  // namespace lg
}  // namespace mlsb
