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

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "large_common.cuh"
#include "large_internal.h"
#include "../../include/mixedls_b200_tools.h"

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
  long long* probe = nullptr;  // clock64 stamps of CTA 0 thread 0 (measurement builds only)
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
// binary64 factors (u_f = working): the reference's make_reflector in double
__device__ __forceinline__ void larfg_s(double alpha, double ss, double& tau, double& inv, double& beta) {
  tau = 0.0;
  inv = 1.0;
  beta = alpha;
  if (ss != 0.0) {
    const double bt = -copysign(sqrt(fma(alpha, alpha, ss)), alpha);
    tau = (bt - alpha) / bt;
    inv = 1.0 / (alpha - bt);
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

// ---------------------------------------------------------------------------
// Register-resident binary32 panel (the large path's critical chain: one
// panel per NB reflectors, 160 panels at C3).  Every thread of the cluster
// owns RPT whole rows of the panel in registers (P[i][0..NB)), so a
// reflector step touches shared memory only for its reductions:
//
//   1. per thread: d_k = sum_{own rows r > q} x_r P[r][k] for all k (and
//      ||x||^2 in binary64) -- RPT*NB register FMAs;
//   2. warp: transposed butterfly (31 shuffles) leaves lane k with the warp's
//      d_k; CTA: 16 warp partials summed in warp order by thread k;
//   3. cluster: each CTA PUSHES its partials (d, pivot row, norm) into slot
//      [rank] of every CTA's exchange buffer (remote st.shared::cluster, no
//      remote-load round trip), one barrier.cluster, then sums the slots in
//      rank order -- identical totals in every CTA;
//   4. per thread: xLARFG scalars, coef_k = tau (p_k + inv d_k), and the
//      rank-1 update of its own rows, all in registers.
//
// Two CTA barriers and one cluster barrier per reflector; the q loop is fully
// unrolled so every register index is static.
__device__ __forceinline__ uint32_t cl_addr(const void* p, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(r)
               : "r"(uint32_t(__cvta_generic_to_shared(p))), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cl(uint32_t a, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void st_cl(uint32_t a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
// remote store that signals the destination CTA's mbarrier on arrival
__device__ __forceinline__ void st_async(uint32_t a, float v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f32 [%0], %1, [%2];" ::"r"(a), "f"(v),
               "r"(bar)
               : "memory");
}
__device__ __forceinline__ void st_async(uint32_t a, float4 v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(a),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void st_async(uint32_t a, double v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(a), "d"(v),
               "r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(const void* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(uint32_t(__cvta_generic_to_shared(bar))),
      "r"(parity)
      : "memory");
}
// all threads of the cluster; orders the remote shared stores before the wait
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// element (r, q) of the panel view at base(r) + q * stride (QR: down a column
// of M with stride ld; RQ: along a row of M, conjugated, stride -1)
template <class T>
__device__ __forceinline__ void view_row(const PanelArgs<T>& a, int r, T*& base, int64_t& stride) {
  if (a.rq) {
    base = a.M + a.r0 + (a.c0 - r) * a.ld;
    stride = -1;
  } else {
    base = a.M + (a.r0 + r) + a.c0 * a.ld;
    stride = a.ld;
  }
}

template <int RPT, int NT>
__global__ void __launch_bounds__(NT, 1) panel_reg_kernel(PanelArgs<float> a) {
  constexpr int NW = NT / 32;
  __shared__ float wpart[NW][NB];
  __shared__ double wnorm[NW];
  __shared__ __align__(16) float prow_s[NB];
  __shared__ __align__(16) float xd[2][PCL][NB];  // [parity][rank] CTA partials of d
  __shared__ __align__(16) float xp[2][NB];       // [parity] pivot row (from its owner CTA)
  __shared__ double xn[2][PCL];                   // [parity][rank] CTA partials of ||x||^2
  __shared__ __align__(8) unsigned long long xbar[2];  // exchange arrivals, per parity
  __shared__ uint32_t rbase[PCL];                      // cluster address of xd in CTA c
  __shared__ __align__(16) float coef_s[NB];
  __shared__ float scal[2];
  __shared__ __align__(16) float G[NB * NB];
  __shared__ float taus[NB];

  cg::cluster_group cl = cg::this_cluster();
  const int rank = int(cl.block_rank()), ncl = a.ncl;
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int nb = a.nb;
  const int rb = rank * a.rc, re = min(a.L, rb + a.rc);

  long long* pk0 = (a.probe && rank == 0 && tid == 0) ? a.probe + 8 * NB : nullptr;  // kernel-level stamps
  if (pk0) pk0[0] = clock64();
  float P[RPT][NB];
  int row[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    row[i] = rb + tid + NT * i;
    const bool own = row[i] < re;
    float* pb;
    int64_t ps;
    view_row(a, own ? row[i] : rb, pb, ps);  // running pointer: no per-load address arithmetic
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      P[i][k] = (own && k < nb) ? *pb : 0.f;
      pb += ps;
    }
    if (!own) row[i] = -1;  // never > q, never == q
  }
  for (int e = tid; e < NB * NB; e += NT) G[e] = 0.f;
  const uint32_t xd0 = uint32_t(__cvta_generic_to_shared(&xd[0][0][0]));
  if (tid < PCL) rbase[tid] = tid < ncl ? cl_addr(&xd[0][0][0], tid) : 0u;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(uint32_t(__cvta_generic_to_shared(&xbar[0]))));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(uint32_t(__cvta_generic_to_shared(&xbar[1]))));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_barrier();  // every exchange barrier initialised before any remote signal
  const uint32_t xbytes = uint32_t(ncl) * (NB * sizeof(float) + sizeof(double)) + NB * sizeof(float);
  if (pk0) pk0[1] = clock64();
  // exchange buffers and barrier as offsets from xd (the same in every CTA)
  const uint32_t off_d = uint32_t(__cvta_generic_to_shared(&xd[0][rank][0])) - xd0;
  const uint32_t off_p = uint32_t(__cvta_generic_to_shared(&xp[0][0])) - xd0;
  const uint32_t off_n = uint32_t(__cvta_generic_to_shared(&xn[0][rank])) - xd0;
  const uint32_t off_bar = uint32_t(__cvta_generic_to_shared(&xbar[0])) - xd0;
  constexpr uint32_t par_d = sizeof(xd[0]), par_p = sizeof(xp[0]), par_n = sizeof(xn[0]);

  // Rotating frame: at step q, P[i][f] holds column (q + f) mod NB, so the
  // current column is always P[i][0] and the step is the same code for every
  // q (a real loop: the unrolled 32-step body does not fit the i-cache).
#pragma unroll 1
  for (int q = 0; q < nb; ++q) {
    const int par = q & 1;
    long long* pq = (a.probe && rank == 0 && tid == 0) ? a.probe + 8 * q : nullptr;
    if (pq) pq[0] = clock64();
    // ---- 1. thread partials (frame order)
    float d[NB];
#pragma unroll
    for (int f = 0; f < NB; ++f) d[f] = 0.f;
    double nn = 0.0;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      if (row[i] > q) {
        const float x = P[i][0];
        nn = fma(double(x), double(x), nn);
#pragma unroll
        for (int f = 0; f < NB; ++f) d[f] = fmaf(x, P[i][f], d[f]);
      } else if (row[i] == q) {
#pragma unroll
        for (int f = 0; f < NB; ++f) prow_s[f] = P[i][f];
      }
    }
    // ---- 2. warp transposed reduction: lane l ends with the warp sum of d[l]
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      const bool up = (l & s) != 0;
#pragma unroll
      for (int j = 0; j < s; ++j) {
        const float send = up ? d[j] : d[j + s];
        const float keep = up ? d[j + s] : d[j];
        d[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
      }
    }
    nn = wsum(nn);
    wpart[w][l] = d[0];
    if (l == 0) wnorm[w] = nn;
    if (pq) pq[1] = clock64();
    __syncthreads();
    if (pq) pq[2] = clock64();
    // ---- 3. CTA partials pushed into slot [rank] of every CTA's exchange
    //         buffer by st.async, each landing store counted on the
    //         destination's mbarrier (no fence, no cluster barrier)
    if (tid == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       uint32_t(__cvta_generic_to_shared(&xbar[par]))),
                   "r"(xbytes)
                   : "memory");
    {
      // one 16-byte chunk per (destination, chunk) pair: threads u = 8 c + j
      const uint32_t bo = off_bar + 8 * par;
      for (int u = tid; u < 8 * ncl; u += NT) {
        const int c = u >> 3, j = u & 7;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int ww = 0; ww < NW; ++ww) {
          const float4 t = *reinterpret_cast<const float4*>(&wpart[ww][4 * j]);
          v.x += t.x, v.y += t.y, v.z += t.z, v.w += t.w;
        }
        st_async(rbase[c] + off_d + par * par_d + 16 * j, v, rbase[c] + bo);
      }
      if (q >= rb && q < re)  // this CTA owns the pivot row
        for (int u = tid; u < 8 * ncl; u += NT) {
          const int c = u >> 3, j = u & 7;
          st_async(rbase[c] + off_p + par * par_p + 16 * j, *reinterpret_cast<const float4*>(&prow_s[4 * j]),
                   rbase[c] + bo);
        }
      if (tid < ncl) {
        double t[NW];
#pragma unroll
        for (int ww = 0; ww < NW; ++ww) t[ww] = wnorm[ww];
        double v = 0.0;
#pragma unroll
        for (int ww = 0; ww < NW; ++ww) v += t[ww];
        st_async(rbase[tid] + off_n + par * par_n, v, rbase[tid] + bo);
      }
    }
    // ---- 4. warp 0: totals in rank order (lane f: d_f, p_f), xLARFG, the
    //         update coefficients coef_f = tau v^T P[:, f] and Gram entries
    if (pq) pq[3] = clock64();
    if (w == 0) {
      mbar_wait(&xbar[par], (q >> 1) & 1);
      if (pq) pq[4] = clock64();
      float td[PCL];
      double tn[PCL];
#pragma unroll
      for (int c = 0; c < PCL; ++c) {
        const bool in = c < ncl;
        td[c] = in ? xd[par][c][l] : 0.f;
        tn[c] = in ? xn[par][c] : 0.0;
      }
      const float pk = xp[par][l];
      // fixed pairwise tree over the ranks (absent ranks add exact zeros)
#pragma unroll
      for (int h = PCL / 2; h >= 1; h >>= 1)
#pragma unroll
        for (int c = 0; c < h; ++c) {
          td[c] += td[c + h];
          tn[c] += tn[c + h];
        }
      const float dk = td[0];
      const double nrm = tn[0];
      float tau, inv, beta;
      larfg_s(__shfl_sync(0xffffffffu, pk, 0), nrm, tau, inv, beta);
      const float s = fmaf(inv, dk, pk);  // v^T P[:, f]
      coef_s[l] = (l >= 1 && l < nb - q) ? tau * s : 0.f;
      if (l >= NB - q) G[(q + l - NB) + NB * q] = s;  // v_k^T v_q, k = q + l - NB < q
      if (l == 0) {
        scal[0] = inv;
        scal[1] = beta;
        taus[q] = tau;
      }
    }
    if (pq) pq[5] = clock64();
    __syncthreads();
    if (pq) pq[6] = clock64();
    // ---- 5. rank-1 update of my rows, in registers, then rotate the frame
    const float inv = scal[0], beta = scal[1];
    float v[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) v[i] = row[i] == q ? 1.f : (row[i] > q ? inv * P[i][0] : 0.f);
#pragma unroll
    for (int f4 = 0; f4 < NB; f4 += 4) {
      const float4 c4 = *reinterpret_cast<const float4*>(&coef_s[f4]);
      const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (f4 + t >= 1)
#pragma unroll
          for (int i = 0; i < RPT; ++i) P[i][f4 + t] = fmaf(-cc[t], v[i], P[i][f4 + t]);
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const float p0 = row[i] == q ? beta : (row[i] > q ? v[i] : P[i][0]);
#pragma unroll
      for (int f = 0; f < NB - 1; ++f) P[i][f] = P[i][f + 1];
      P[i][NB - 1] = p0;
    }
    if (pq) pq[7] = clock64();
  }
  if (pk0) pk0[2] = clock64();
  __syncthreads();
  if (pk0) pk0[3] = clock64();
  // ---- T of the panel first (rank 0, warp 0), overlapping the other warps'
  //      write-back; then every thread writes its rows back through running
  //      pointers (frame index f holds column (nb + f) mod NB after nb steps)
  if (rank == 0) {
    if (tid < nb) a.tau[tid] = taus[tid];
    if (w == 0) {
      // T[q][q] = tau_q ; T[0:q, q] = -tau_q T[0:q, 0:q] G[0:q, q]; lane l owns row l
      float Tr[NB];
#pragma unroll
      for (int k2 = 0; k2 < NB; ++k2) Tr[k2] = 0.f;
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        if (q < nb) {
          // column q of G as eight broadcast 16-byte loads, issued before the
          // (unchanged, sequential) dot so no load latency sits on it
          float gq[NB];
#pragma unroll
          for (int k4 = 0; k4 < NB; k4 += 4) {
            const float4 g4 = *reinterpret_cast<const float4*>(&G[k4 + NB * q]);
            gq[k4] = g4.x, gq[k4 + 1] = g4.y, gq[k4 + 2] = g4.z, gq[k4 + 3] = g4.w;
          }
          float t = 0.f;
#pragma unroll
          for (int k2 = 0; k2 < NB; ++k2)
            if (k2 < q) t = fmaf(Tr[k2], gq[k2], t);
          const float tq = taus[q];
          Tr[q] = l < q ? -(tq * t) : (l == q ? tq : 0.f);
        }
      }
      if (l < nb)
#pragma unroll
        for (int q = 0; q < NB; ++q)
          if (q < nb) a.Tm[l + q * NB] = Tr[q];
    }
  }
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int r = row[i];
    if (r < 0) continue;
    const int64_t vi = a.rq ? (a.c0 - r - a.vbase) : r;
    float* pb;
    int64_t ps;
    view_row(a, r, pb, ps);
    float* pv = a.V + vi;
#pragma unroll
    for (int f = 0; f < NB; ++f) {
      const int kc = (nb + f) & (NB - 1);
      if (kc < nb) {
        pb[kc * ps] = P[i][f];
        pv[kc * a.ldv] = r < kc ? 0.f : (r == kc ? 1.f : P[i][f]);
      }
    }
  }
  if (pk0) pk0[4] = clock64();
  cluster_barrier();
}

template <int RPT, int NT>
__global__ void __launch_bounds__(NT, 1) panel_reg_kernel_c(PanelArgs<cf> a) {
  constexpr int NW = NT / 32;
  __shared__ cf wpart[NW][NB];
  __shared__ double wnorm[NW];
  __shared__ __align__(16) cf prow_s[NB];
  __shared__ __align__(16) cf xd[2][PCL][NB];  // [parity][rank] CTA partials of d
  __shared__ __align__(16) cf xp[2][NB];       // [parity] pivot row (from its owner CTA)
  __shared__ double xn[2][PCL];                   // [parity][rank] CTA partials of ||x||^2
  __shared__ __align__(8) unsigned long long xbar[2];  // exchange arrivals, per parity
  __shared__ uint32_t rbase[PCL];                      // cluster address of xd in CTA c
  __shared__ __align__(16) cf coef_s[NB];
  __shared__ cf scal[2];
  __shared__ cf G[NB * NB];
  __shared__ cf taus[NB];

  cg::cluster_group cl = cg::this_cluster();
  const int rank = int(cl.block_rank()), ncl = a.ncl;
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int nb = a.nb;
  const int rb = rank * a.rc, re = min(a.L, rb + a.rc);

  cf P[RPT][NB];
  int row[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    row[i] = rb + tid + NT * i;
    const bool own = row[i] < re;
    cf* pb;
    int64_t ps;
    view_row(a, own ? row[i] : rb, pb, ps);
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      P[i][k] = (own && k < nb) ? (a.rq ? conj_(*pb) : *pb) : zero<cf>();
      pb += ps;
    }
    if (!own) row[i] = -1;  // never > q, never == q
  }
  for (int e = tid; e < NB * NB; e += NT) G[e] = zero<cf>();
  const uint32_t xd0 = uint32_t(__cvta_generic_to_shared(&xd[0][0][0]));
  if (tid < PCL) rbase[tid] = tid < ncl ? cl_addr(&xd[0][0][0], tid) : 0u;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(uint32_t(__cvta_generic_to_shared(&xbar[0]))));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(uint32_t(__cvta_generic_to_shared(&xbar[1]))));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_barrier();  // every exchange barrier initialised before any remote signal
  const uint32_t xbytes = uint32_t(ncl) * (NB * sizeof(cf) + sizeof(double)) + NB * sizeof(cf);
  // exchange buffers and barrier as offsets from xd (the same in every CTA)
  const uint32_t off_d = uint32_t(__cvta_generic_to_shared(&xd[0][rank][0])) - xd0;
  const uint32_t off_p = uint32_t(__cvta_generic_to_shared(&xp[0][0])) - xd0;
  const uint32_t off_n = uint32_t(__cvta_generic_to_shared(&xn[0][rank])) - xd0;
  const uint32_t off_bar = uint32_t(__cvta_generic_to_shared(&xbar[0])) - xd0;
  constexpr uint32_t par_d = sizeof(xd[0]), par_p = sizeof(xp[0]), par_n = sizeof(xn[0]);

  // Rotating frame: at step q, P[i][f] holds column (q + f) mod NB, so the
  // current column is always P[i][0] and the step is the same code for every
  // q (a real loop: the unrolled 32-step body does not fit the i-cache).
#pragma unroll 1
  for (int q = 0; q < nb; ++q) {
    const int par = q & 1;
    long long* pq = (a.probe && rank == 0 && tid == 0) ? a.probe + 8 * q : nullptr;
    if (pq) pq[0] = clock64();
    // ---- 1. thread partials (frame order)
    cf d[NB];
#pragma unroll
    for (int f = 0; f < NB; ++f) d[f] = zero<cf>();
    double nn = 0.0;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      if (row[i] > q) {
        const cf x = P[i][0];
        nn += abs2d(x);
        const cf xc = conj_(x);
#pragma unroll
        for (int f = 0; f < NB; ++f) mac(d[f], xc, P[i][f]);
      } else if (row[i] == q) {
#pragma unroll
        for (int f = 0; f < NB; ++f) prow_s[f] = P[i][f];
      }
    }
    // ---- 2. warp transposed reduction: lane l ends with the warp sum of d[l]
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      const bool up = (l & s) != 0;
#pragma unroll
      for (int j = 0; j < s; ++j) {
        const cf send = up ? d[j] : d[j + s];
        const cf keep = up ? d[j + s] : d[j];
        d[j] = keep + cf{__shfl_xor_sync(0xffffffffu, send.x, s), __shfl_xor_sync(0xffffffffu, send.y, s)};
      }
    }
    nn = wsum(nn);
    wpart[w][l] = d[0];
    if (l == 0) wnorm[w] = nn;
    if (pq) pq[1] = clock64();
    __syncthreads();
    if (pq) pq[2] = clock64();
    // ---- 3. CTA partials pushed into slot [rank] of every CTA's exchange
    //         buffer by st.async, each landing store counted on the
    //         destination's mbarrier (no fence, no cluster barrier)
    if (tid == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       uint32_t(__cvta_generic_to_shared(&xbar[par]))),
                   "r"(xbytes)
                   : "memory");
    {
      // one 16-byte chunk (two complex values) per (destination, chunk) pair:
      // threads u = 16 c + j
      const uint32_t bo = off_bar + 8 * par;
      for (int u = tid; u < 16 * ncl; u += NT) {
        const int c = u >> 4, j = u & 15;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int ww = 0; ww < NW; ++ww) {
          const float4 t = *reinterpret_cast<const float4*>(&wpart[ww][2 * j]);
          v.x += t.x, v.y += t.y, v.z += t.z, v.w += t.w;
        }
        st_async(rbase[c] + off_d + par * par_d + 16 * j, v, rbase[c] + bo);
      }
      if (q >= rb && q < re)  // this CTA owns the pivot row
        for (int u = tid; u < 16 * ncl; u += NT) {
          const int c = u >> 4, j = u & 15;
          st_async(rbase[c] + off_p + par * par_p + 16 * j, *reinterpret_cast<const float4*>(&prow_s[2 * j]),
                   rbase[c] + bo);
        }
      if (tid < ncl) {
        double t[NW];
#pragma unroll
        for (int ww = 0; ww < NW; ++ww) t[ww] = wnorm[ww];
        double v = 0.0;
#pragma unroll
        for (int ww = 0; ww < NW; ++ww) v += t[ww];
        st_async(rbase[tid] + off_n + par * par_n, v, rbase[tid] + bo);
      }
    }
    // ---- 4. warp 0: totals in rank order (lane f: d_f, p_f), xLARFG, the
    //         update coefficients coef_f = tau v^T P[:, f] and Gram entries
    if (pq) pq[3] = clock64();
    if (w == 0) {
      mbar_wait(&xbar[par], (q >> 1) & 1);
      if (pq) pq[4] = clock64();
      cf td[PCL];
      double tn[PCL];
#pragma unroll
      for (int c = 0; c < PCL; ++c) {
        const bool in = c < ncl;
        td[c] = in ? xd[par][c][l] : zero<cf>();
        tn[c] = in ? xn[par][c] : 0.0;
      }
      const cf pk = xp[par][l];
#pragma unroll
      for (int h = PCL / 2; h >= 1; h >>= 1)
#pragma unroll
        for (int c = 0; c < h; ++c) {
          td[c] = td[c] + td[c + h];
          tn[c] += tn[c + h];
        }
      const cf dk = td[0];
      const double nrm = tn[0];
      cf tau, inv, beta;
      larfg_s(cf{__shfl_sync(0xffffffffu, pk.x, 0), __shfl_sync(0xffffffffu, pk.y, 0)}, nrm, tau, inv, beta);
      const cf sv = pk + conj_(inv) * dk;  // v^H P[:, f]
      coef_s[l] = (l >= 1 && l < nb - q) ? conj_(tau) * sv : zero<cf>();  // H^H = I - conj(tau) v v^H
      if (l >= NB - q) G[(q + l - NB) + NB * q] = conj_(pk) + inv * conj_(dk);  // v_k^H v_q
      if (l == 0) {
        scal[0] = inv;
        scal[1] = beta;
        taus[q] = tau;
      }
    }
    if (pq) pq[5] = clock64();
    __syncthreads();
    if (pq) pq[6] = clock64();
    // ---- 5. rank-1 update of my rows, in registers, then rotate the frame
    const cf inv = scal[0], beta = scal[1];
    cf v[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) v[i] = row[i] == q ? one<cf>() : (row[i] > q ? inv * P[i][0] : zero<cf>());
#pragma unroll
    for (int f2 = 0; f2 < NB; f2 += 2) {
      const float4 c4 = *reinterpret_cast<const float4*>(&coef_s[f2]);
      const cf cc[2] = {cf{c4.x, c4.y}, cf{c4.z, c4.w}};
#pragma unroll
      for (int t = 0; t < 2; ++t)
        if (f2 + t >= 1)
#pragma unroll
          for (int i = 0; i < RPT; ++i) P[i][f2 + t] = P[i][f2 + t] - cc[t] * v[i];
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const cf p0 = row[i] == q ? beta : (row[i] > q ? v[i] : P[i][0]);
#pragma unroll
      for (int f = 0; f < NB - 1; ++f) P[i][f] = P[i][f + 1];
      P[i][NB - 1] = p0;
    }
    if (pq) pq[7] = clock64();
  }
  __syncthreads();
  // ---- T first (rank 0, warp 0), then the write-back through running pointers
  if (rank == 0) {
    if (tid < nb) a.tau[tid] = taus[tid];
    if (w == 0) {
      cf Tr[NB];
#pragma unroll
      for (int k2 = 0; k2 < NB; ++k2) Tr[k2] = zero<cf>();
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        if (q < nb) {
          cf t = zero<cf>();
#pragma unroll
          for (int k2 = 0; k2 < NB; ++k2)
            if (k2 < q) mac(t, Tr[k2], G[k2 + NB * q]);
          const cf tq = taus[q];
          Tr[q] = l < q ? -(tq * t) : (l == q ? tq : zero<cf>());
        }
      }
      if (l < nb)
#pragma unroll
        for (int q = 0; q < NB; ++q)
          if (q < nb) a.Tm[l + q * NB] = Tr[q];
    }
  }
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int r = row[i];
    if (r < 0) continue;
    const int64_t vi = a.rq ? (a.c0 - r - a.vbase) : r;
    cf* pb;
    int64_t ps;
    view_row(a, r, pb, ps);
    cf* pv = a.V + vi;
#pragma unroll
    for (int f = 0; f < NB; ++f) {
      const int kc = (nb + f) & (NB - 1);
      if (kc < nb) {
        pb[kc * ps] = a.rq ? conj_(P[i][f]) : P[i][f];
        pv[kc * a.ldv] = r < kc ? zero<cf>() : (r == kc ? one<cf>() : P[i][f]);
      }
    }
  }
  cluster_barrier();
}

template <class T>
static size_t panel_smem(int rc) {
  const int NV = 2 * NB;
  return size_t(rc) * NB * sizeof(T) + 2 * sizeof(double) + 2 * NV * sizeof(T) + NV * sizeof(T) +
         2 * sizeof(double) + (NB * NB + 2 * NB + PNW * NB) * sizeof(T) + PNW * sizeof(double) + 64;
}

template <class T>
cudaError_t panel_factor(T* M, int64_t ld, int64_t r0, int64_t c0, int L, int nb, bool rq, T* tau,
                         T* V, int64_t ldv, T* Tm, int64_t vbase, cudaStream_t st, long long* probe) {
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
  a.probe = probe;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(PNT);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  static const bool smem_panel = getenv("MLSB_PANEL_SMEM") != nullptr;  // A/B comparisons
  if constexpr (std::is_same<T, float>::value) {
    // register-resident rows: 256 threads x 2 rows per CTA while 16 CTAs hold
    // the panel, else 512 x 2
    if (L <= PCL * 512 * 2 && !smem_panel) {
      const bool small = L <= PCL * 128 * 4;
      // 256 threads x 2 rows per CTA: two warps per scheduler hide each other's
      // latency (ncu: the 128 x 4 form runs at IPC 0.69 with one warp per
      // scheduler, ~760 instructions per warp and reflector at ~5.8 cycles
      // each).  Measured at 8192 x 32: 61.8 us (128 x 4), 57.6 us (256 x 2),
      // 68.5 us (512 x 1); C3 factorization 24.9 / 23.4 / 24.9 ms.
      // MLSB_PANEL_256=0 / 2 select the other two forms (A/B).
      static const int pvar = getenv("MLSB_PANEL_256") ? atoi(getenv("MLSB_PANEL_256")) : 1;
      const bool p256 = pvar == 1, p512 = pvar == 2;
      const int per = small ? 128 * 4 : 512 * 2;
      const int ncl = std::min(PCL, (L + per - 1) / per);
      a.ncl = ncl;
      a.rc = (L + ncl - 1) / ncl;
      auto kern = small ? (p256 ? panel_reg_kernel<2, 256> : (p512 ? panel_reg_kernel<1, 512> : panel_reg_kernel<4, 128>))
                        : panel_reg_kernel<2, 512>;
      static bool attr_reg = false;
      if (!attr_reg) {
        if ((e = cudaFuncSetAttribute(panel_reg_kernel<2, 256>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)))
          return e;
        if ((e = cudaFuncSetAttribute(panel_reg_kernel<1, 512>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)))
          return e;
        if ((e = cudaFuncSetAttribute(panel_reg_kernel<4, 128>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)))
          return e;
        if ((e = cudaFuncSetAttribute(panel_reg_kernel<2, 512>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)))
          return e;
        attr_reg = true;
      }
      cfg.gridDim = dim3(ncl);
      cfg.blockDim = dim3(small ? (p256 ? 256 : (p512 ? 512 : 128)) : 512);
      cfg.dynamicSmemBytes = 0;
      attr[0].val.clusterDim.x = ncl;
      return cudaLaunchKernelEx(&cfg, kern, a);
    }
  }
  if constexpr (std::is_same<T, cf>::value) {
    // complex64: 256 threads x 1 row per CTA while 16 CTAs hold the panel
    if (L <= PCL * 256 && !smem_panel) {
      const int ncl = std::min(PCL, (L + 255) / 256);
      a.ncl = ncl;
      a.rc = (L + ncl - 1) / ncl;
      static bool attr_c = false;
      if (!attr_c) {
        if ((e = cudaFuncSetAttribute(panel_reg_kernel_c<1, 256>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)))
          return e;
        attr_c = true;
      }
      cfg.gridDim = dim3(ncl);
      cfg.blockDim = dim3(256);
      cfg.dynamicSmemBytes = 0;
      attr[0].val.clusterDim.x = ncl;
      return cudaLaunchKernelEx(&cfg, panel_reg_kernel_c<1, 256>, a);
    }
  }
  const size_t sm = panel_smem<T>(a.rc);
  auto kern = panel_kernel<T>;
  static bool attr_done = false;  // per instantiation
  if (!attr_done) {
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1))) return e;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)))
      return e;
    attr_done = true;
  }
  if (sm > 227 * 1024) return cudaErrorInvalidValue;
  cfg.gridDim = dim3(a.ncl);
  cfg.dynamicSmemBytes = sm;
  attr[0].val.clusterDim.x = a.ncl;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template cudaError_t panel_factor<float>(float*, int64_t, int64_t, int64_t, int, int, bool, float*,
                                         float*, int64_t, float*, int64_t, cudaStream_t, long long*);
template cudaError_t panel_factor<cf>(cf*, int64_t, int64_t, int64_t, int, int, bool, cf*, cf*,
                                      int64_t, cf*, int64_t, cudaStream_t, long long*);
template cudaError_t panel_factor<double>(double*, int64_t, int64_t, int64_t, int, int, bool, double*,
                                          double*, int64_t, double*, int64_t, cudaStream_t, long long*);

}  // namespace lg
}  // namespace mlsb

extern "C" int mlsb_panel_f32(float* M, int64_t ld, int64_t r0, int64_t c0, int L, int nb, float* tau,
                              float* V, int64_t ldv, float* T, void* stream) {
  return int(mlsb::lg::panel_factor<float>(M, ld, r0, c0, L, nb, false, tau, V, ldv, T, 0,
                                           static_cast<cudaStream_t>(stream)));
}
extern "C" int mlsb_panel_c64(float* M, int64_t ld, int64_t r0, int64_t c0, int L, int nb, float* tau, float* V,
                              int64_t ldv, float* T, void* stream) {
  using mlsb::lg::cf;
  return int(mlsb::lg::panel_factor<cf>(reinterpret_cast<cf*>(M), ld, r0, c0, L, nb, false,
                                        reinterpret_cast<cf*>(tau), reinterpret_cast<cf*>(V), ldv,
                                        reinterpret_cast<cf*>(T), 0, static_cast<cudaStream_t>(stream)));
}
extern "C" int mlsb_panel_probe_f32(float* M, int64_t ld, int L, int nb, float* tau, float* V, float* T,
                                    long long* probe, void* stream) {
  return int(mlsb::lg::panel_factor<float>(M, ld, 0, 0, L, nb, false, tau, V, L, T, 0,
                                           static_cast<cudaStream_t>(stream), probe));
}
