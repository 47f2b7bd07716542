// Whole-factor reflector applications and whole triangular solves of the
// large path's refinement cascade as ONE persistent (cooperative) launch each.
//
// Why: the correction solves of lse_correction_solve / gls_correction_solve
// (inc/lse.hpp:83-128, inc/gls.hpp:106-154) apply F = P_0 ... P_last (xORMQR
// with compact-WY blocks of 128 reflectors) and run xTRSV on the 128-row
// diagonal blocks of T and R.  Per block, the work is a few MB of V (HBM
// streaming) but the blocks are strictly sequential: block-per-launch costs
// two launches and a full grid drain per 128 reflectors (round 1: ~900
// launches, 2.2 ms per C3 correction, 0.02 of HBM).  Here the sequencing
// stays on the device:
//
//  * k_fac_apply: CTA c owns rows [c RB, c RB + RB) of x for the whole launch
//    (x in shared memory).  Per block: each thread holds its row's slice of
//    V_b in registers (loaded once, prefetched during the previous block's
//    barrier), dots y_c = V_b^H x_c (transposed warp reductions + a fixed-
//    order sum over row groups), publishes its partial, meets the other
//    active CTAs at a per-block counter (release/acquire), sums the partials
//    in CTA order (bitwise identical y in every CTA), forms z = T' y
//    redundantly and updates its rows with the same registers.  One grid
//    barrier per 128 reflectors and one HBM read of V.
//  * k_trsv_chain: CTA j owns the 128-row block j of U x = b (or U^H x = b):
//    it prefetches its diagonal block into shared memory, subtracts the
//    contributions of the already solved blocks as their flags arrive (in a
//    fixed order: bitwise reproducible), solves its diagonal block with the
//    lane-owned-row chain of k_trsv_diag128 and publishes x_j with a flag.
//    The critical path is one 128-step chain per block plus one flag hop.
//
// Both need all CTAs co-resident (spin-waits), hence cooperative launches of
// at most one CTA per SM.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "large_common.cuh"

namespace mlsb {
namespace lg {

template <class FT>
struct BlkD {
  const FT* V;
  const FT* T;
  int64_t ldv;
  int L, nbk, voff, ldt;
};

constexpr int CZ_NT = 512;
constexpr int CZ_MAXB = 192;  // blocks per factor handled by one launch

__device__ __forceinline__ float ldcg_(const float* p) { return __ldcg(p); }
__device__ __forceinline__ double ldcg_(const double* p) { return __ldcg(p); }
__device__ __forceinline__ cf ldcg_(const cf* p) {
  const float2 v = __ldcg(reinterpret_cast<const float2*>(p));
  return cf{v.x, v.y};
}
__device__ __forceinline__ cd ldcg_(const cd* p) {
  const double2 v = __ldcg(reinterpret_cast<const double2*>(p));
  return cd{v.x, v.y};
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(smem_dst))),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Arrive on a step counter (zeroed before the launch) and wait until `need`
// CTAs have arrived.  The CTA's prior global writes are released by thread
// 0's fence after the CTA barrier; readers acquire and then use ld.cg.
__device__ __forceinline__ void cz_barrier(int* cnt, int need) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(cnt) : "memory");
    while (ld_acquire(cnt) < need) {
    }
  }
  __syncthreads();
}

// Split form: arrive right after the CTA's partials are written (the release
// then covers only those stores), issue the independent prefetches, then wait.
// A release placed after the prefetch loads would wait for them to land.
__device__ __forceinline__ void cz_arrive(int* cnt) {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(cnt) : "memory");
}
__device__ __forceinline__ void cz_wait(const int* cnt, int need) {
  if (threadIdx.x == 0)
    while (ld_acquire(cnt) < need) {
    }
  __syncthreads();
}

// debug: globaltimer stamps of CTA 0 (mlsb_debug_set_czstamps), null in production
__device__ unsigned long long* g_czstamp = nullptr;
__device__ __forceinline__ void czstamp_any(int k) {
  unsigned long long* p = g_czstamp;
  if (p != nullptr && threadIdx.x == 0 && k < 512) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    p[k] = t;
  }
}
__device__ __forceinline__ void czstamp(int k) {
  unsigned long long* p = g_czstamp;
  if (p != nullptr && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0 && k < 512) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    p[k] = t;
  }
}

// Transposed butterfly over 32 lanes of NV per-lane values: lane l returns the
// warp sum of value index (l >> (5 - log2 NV)) (fixed order, every lane of a
// group gets the same bits).
template <int NV, class CT>
__device__ __forceinline__ CT tsum_lanes(CT (&d)[NV], int l) {
  int n = NV;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    if (n > 1) {
      const int h = n >> 1;
      const bool b = l & o;
#pragma unroll
      for (int i = 0; i < NV / 2; ++i)
        if (i < h) {
          const CT send = b ? d[i] : d[i + h], keep = b ? d[i + h] : d[i];
          d[i] = keep + shfl_xor(send, o);
        }
      n = h;
    } else {
      d[0] = d[0] + shfl_xor(d[0], o);
    }
  }
  return d[0];
}

// vector loads of V: VEC consecutive rows per lane (one 16-byte load per
// column when V's columns are 16-byte aligned)
template <class FT> struct VecOf;
template <> struct VecOf<float> { using T = float4; };
template <> struct VecOf<double> { using T = double2; };
template <> struct VecOf<cf> { using T = float4; };
template <> struct VecOf<cd> { using T = double2; };  // one element (VEC = 1)

// x := F^H x (HERM: blocks first to last, T^H) or F x (last to first, T), with
// F = prod_b (I - V_b T_b V_b^H) over the `nb` blocks.  x has `nrows` entries;
// CTA c owns rows [c RB, c RB + RB), RB = 32 VEC: lane l holds rows
// VEC l .. VEC l + VEC - 1 of its CTA and warp w the 8 columns 8w .. 8w + 7
// of every block (VEC x 8 values of V in registers).  part: nb * gridDim.x *
// 128 CT scratch; cnt: nb ints, zero at launch.  Dynamic shared memory: the
// staged T_b.  ALIGNED: every column of every V_b starts 16-byte aligned at
// the CTA's first row (16-byte loads), else scalar loads.
template <class FT, class CT, bool HERM, bool ALIGNED>
__global__ void __launch_bounds__(CZ_NT, 1) k_fac_apply(const BlkD<FT>* blks, int nb, CT* x, int nrows,
                                                        CT* part, int* cnt) {
  constexpr int VEC = 16 / int(sizeof(FT)) > 0 ? 16 / int(sizeof(FT)) : 1;
  constexpr int RB = 32 * VEC;
  constexpr int PER = 16 / int(sizeof(FT)) > 0 ? 16 / int(sizeof(FT)) : 1;  // FT per 16-byte chunk
  constexpr int TLDS = 128 + PER;  // padded column stride of the staged T
  __shared__ BlkD<FT> sb[CZ_MAXB];
  __shared__ CT xs[RB];
  __shared__ CT zq[4][128];
  __shared__ CT ys[128], zs[128];
  __shared__ CT ured[16][RB];
  extern __shared__ __align__(16) unsigned char czap_[];
  FT* Ts = reinterpret_cast<FT*>(czap_);  // Ts[k * TLDS + q] = T(q, k)
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int c = blockIdx.x, G = gridDim.x;
  const int row0 = c * RB, r0l = VEC * l, rq = row0 + r0l;  // the lane's first row
  for (int i = tid; i < nb; i += CZ_NT) sb[i] = blks[HERM ? i : nb - 1 - i];
  for (int i = tid; i < RB; i += CZ_NT) xs[i] = row0 + i < nrows ? x[row0 + i] : zero<CT>();
  // T entries outside a block's nbk x nbk stay finite (zero or an earlier T):
  // they only ever meet y_k = 0 (k >= nbk) or outputs masked below
  for (int i = tid; i < 128 * TLDS; i += CZ_NT) Ts[i] = zero<FT>();
  __syncthreads();

  auto active = [&](const BlkD<FT>& b) {
    return c >= b.voff / RB && c < min(G, (b.voff + b.L + RB - 1) / RB);
  };
  auto next_active = [&](int s) {
    for (; s < nb; ++s)
      if (active(sb[s])) return s;
    return nb;
  };
  // v[cc][i] = V_b(rq + i - voff, 8 w + cc)
  auto load_v = [&](const BlkD<FT> b, FT (&v)[8][VEC]) {
    const int lr = rq - b.voff;
    const FT* vp = b.V + lr + int64_t(8 * w) * b.ldv;
    if (ALIGNED && lr >= 0 && lr + VEC <= b.L && rq + VEC <= nrows) {
      using V4 = typename VecOf<FT>::T;
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        if (8 * w + cc < b.nbk) {
          const V4 t = *reinterpret_cast<const V4*>(vp + int64_t(cc) * b.ldv);
          const FT* tf = reinterpret_cast<const FT*>(&t);
#pragma unroll
          for (int i = 0; i < VEC; ++i) v[cc][i] = tf[i];
        } else {
#pragma unroll
          for (int i = 0; i < VEC; ++i) v[cc][i] = zero<FT>();
        }
      }
    } else {
#pragma unroll
      for (int cc = 0; cc < 8; ++cc)
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
          const bool ok = lr + i >= 0 && lr + i < b.L && rq + i < nrows && 8 * w + cc < b.nbk;
          v[cc][i] = ok ? vp[i + int64_t(cc) * b.ldv] : zero<FT>();
        }
    }
  };

  FT v[8][VEC];
  int s = next_active(0);
  if (s < nb) load_v(sb[s], v);
  while (s < nb) {
    const BlkD<FT> b = sb[s];
    const int lo = b.voff / RB, hi = min(G, (b.voff + b.L + RB - 1) / RB);
    czstamp(8 * s + 0);
    CT* ps = part + (int64_t(s) * G) * 128;
    // ---- partial y_c = V_b^H x over this CTA's rows: 8 column sums per lane,
    // one transposed reduction; lane l holds column 8 w + (l >> 2)
    {
      CT d[8];
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        CT a = zero<CT>();
#pragma unroll
        for (int i = 0; i < VEC; ++i) mac(a, conj_(widen_to<CT>(v[cc][i])), xs[r0l + i]);
        d[cc] = a;
      }
      const CT t = tsum_lanes<8, CT>(d, l);
      if ((l & 3) == 0) ps[int64_t(c) * 128 + 8 * w + (l >> 2)] = t;
    }
    czstamp(8 * s + 6);
    cz_arrive(cnt + s);
    czstamp(8 * s + 7);
    // stage T_b while waiting (warp per column, lane per 16-byte chunk)
    for (int k = w; k < b.nbk; k += CZ_NT / 32)
      for (int q0 = l * PER; q0 < b.nbk; q0 += 32 * PER) cp_async16(Ts + k * TLDS + q0, b.T + int64_t(b.ldt) * k + q0);
    // prefetch the next active block's V slice (independent of the barrier)
    const int sn = next_active(s + 1);
    FT vn[8][VEC];
    if (sn < nb) load_v(sb[sn], vn);
    czstamp(8 * s + 1);
    cz_wait(cnt + s, hi - lo);
    czstamp(8 * s + 2);
    // ---- y = sum of the partials in CTA order (identical in every CTA)
    {
      const int q = tid & 127, h = tid >> 7;
      CT a = zero<CT>();
      for (int c2 = lo + h; c2 < hi; c2 += 64) {
        CT t[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int cc = c2 + 4 * u;
          t[u] = cc < hi ? ldcg_(ps + int64_t(cc) * 128 + q) : zero<CT>();
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) a = a + t[u];
      }
      zq[h][q] = a;
    }
    cp_async_wait_all();
    __syncthreads();
    czstamp(8 * s + 3);
    if (tid < 128) ys[tid] = ((zq[0][tid] + zq[1][tid]) + zq[2][tid]) + zq[3][tid];
    __syncthreads();
    // ---- z = T' y (T upper; HERM: T^H), k in quarters, T from shared memory
    {
      const int q = tid & 127, h = tid >> 7, qq = q - 32 * h;
      const FT* tp = HERM ? Ts + q * TLDS + 32 * h : Ts + (32 * h) * TLDS + q;
      CT a = zero<CT>();
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const FT tv = HERM ? tp[u] : tp[u * TLDS];
        const bool ok = HERM ? (u <= qq) : (u >= qq);  // k <= q | k >= q
        mac(a, HERM ? conj_(widen_to<CT>(ok ? tv : zero<FT>())) : widen_to<CT>(ok ? tv : zero<FT>()),
            ys[32 * h + u]);
      }
      zq[h][q] = a;
    }
    __syncthreads();
    if (tid < 128) zs[tid] = tid < b.nbk ? ((zq[0][tid] + zq[1][tid]) + zq[2][tid]) + zq[3][tid] : zero<CT>();
    __syncthreads();
    // ---- x_r -= V_b(r, :) z with the same registers; column groups in order
    {
#pragma unroll
      for (int i = 0; i < VEC; ++i) {
        CT acc = zero<CT>();
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) mac(acc, widen_to<CT>(v[cc][i]), zs[8 * w + cc]);
        ured[w][r0l + i] = acc;
      }
    }
    __syncthreads();
    czstamp(8 * s + 4);
    if (tid < RB) {
      CT a = ured[0][tid];
#pragma unroll
      for (int g = 1; g < 16; ++g) a = a + ured[g][tid];
      xs[tid] = xs[tid] - a;
    }
    __syncthreads();
    czstamp(8 * s + 5);
    if (sn < nb)
#pragma unroll
      for (int cc = 0; cc < 8; ++cc)
#pragma unroll
        for (int i = 0; i < VEC; ++i) v[cc][i] = vn[cc][i];
    s = sn;
  }
  for (int i = tid; i < RB; i += CZ_NT)
    if (row0 + i < nrows) x[row0 + i] = xs[i];
}

// ---------------------------------------------------------------- TRSV
// U = M[r0 : r0+k, c0 : c0+k] upper triangular; !HERM: U x = b (blocks last to
// first), HERM: U^H x = b (first to last).  x holds b on entry.  flags: one int
// per 128-row block, zero at launch.  One CTA per block (grid = ceil(k/128)).
constexpr int CZT = 128;

template <class FT, class CT, bool HERM>
__global__ void __launch_bounds__(CZ_NT, 1) k_trsv_chain(const FT* M, int64_t ld, int64_t r0, int64_t c0,
                                                         int k, CT* x, int* flags) {
  extern __shared__ __align__(16) unsigned char czsm_[];
  constexpr int LU = CZT + 4;  // 16-byte aligned columns (4-row vector loads)
  // diagonal block: !HERM Ud[i + j LU] = U(i, j) (upper); HERM Ud[i + j LU] =
  // conj(U(j, i)) (the lower triangle of U^H), so both solves read a column of
  // four consecutive rows per lane
  FT* Ud = reinterpret_cast<FT*>(czsm_);
  CT* xs = reinterpret_cast<CT*>(Ud + CZT * LU);        // b_j, then x_j
  CT* xi = xs + CZT;                                     // a solved block x_i
  CT* red = xi + CZT;                                    // [4][CZT] partials
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int K = gridDim.x;
  const int j = HERM ? int(blockIdx.x) : K - 1 - int(blockIdx.x);  // early CTAs take the chain head
  const int i0 = CZT * j, bs = min(CZT, k - i0);
  const int rr = tid & (CZT - 1), h = tid >> 7;
  // diagonal block into shared memory (upper triangle; 32 loads in flight per thread)
  {
    const FT* mp = M + (r0 + i0 + rr) + (c0 + i0 + h) * ld;
    FT t[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const int jj = h + 4 * u;
      t[u] = (rr <= jj && jj < bs) ? mp[int64_t(4 * u) * ld] : zero<FT>();
    }
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      if (!HERM) Ud[rr + (h + 4 * u) * LU] = t[u];
      else Ud[(h + 4 * u) + rr * LU] = conj_(t[u]);
    }
  }
  if (tid < CZT) xs[tid] = tid < bs ? x[i0 + tid] : zero<CT>();

  // Contributions of the solved blocks i, nearest-first (the flags' arrival
  // order; a fixed order, so the result is bitwise reproducible).
  //  !HERM: xs[r] -= sum_c U(i0 + r, ib + c) x_i[c]: thread (row rr, column
  //         quarter h), 32 coalesced column loads.
  //   HERM: xs[c] -= sum_r conj(U(ib + r, i0 + c)) x_i[r]: warp w owns columns
  //         8w .. 8w+7, lane l rows l + 32 t (coalesced), one transposed
  //         reduction of the 8 column sums.
  const int nsrc = HERM ? j : K - 1 - j;
  auto src_of = [&](int t) { return HERM ? t : K - 1 - t; };
  auto load_u = [&](int i, FT (&u)[32]) {
    const int ib = CZT * i, ibs = min(CZT, k - ib);
    if (!HERM) {
      const bool rok = rr < bs;
      const FT* mp = M + (r0 + i0 + (rok ? rr : 0)) + (c0 + ib + 32 * h) * ld;
      const int cmax = rok ? ibs - 32 * h : 0;
#pragma unroll
      for (int u2 = 0; u2 < 32; ++u2) u[u2] = u2 < cmax ? mp[int64_t(u2) * ld] : zero<FT>();
    } else {
      // u[8 t + cc] = U(ib + l + 32 t, i0 + 8 w + cc)
      const FT* mp = M + (r0 + ib + l) + (c0 + i0 + 8 * w) * ld;
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          const bool ok = l + 32 * t < ibs && 8 * w + cc < bs;
          u[8 * t + cc] = ok ? mp[32 * t + int64_t(cc) * ld] : zero<FT>();
        }
    }
  };
  FT u[32];
  if (nsrc > 0) load_u(src_of(0), u);
  __syncthreads();
  czstamp_any(4 * j + 0);
  for (int t = 0; t < nsrc; ++t) {
    const int i = src_of(t);
    FT un[32];
    if (t + 1 < nsrc) load_u(src_of(t + 1), un);
    if (tid == 0)
      while (ld_acquire(flags + i) == 0) {
      }
    __syncthreads();
    if (t + 1 == nsrc) czstamp_any(256 + 2 * j);
    if (tid < CZT) {
      const int ib = CZT * i;
      xi[tid] = ib + tid < k ? ldcg_(x + ib + tid) : zero<CT>();
    }
    __syncthreads();
    if (!HERM) {
      CT acc = zero<CT>();
#pragma unroll
      for (int u2 = 0; u2 < 32; ++u2) mac(acc, widen_to<CT>(u[u2]), xi[32 * h + u2]);
      red[h * CZT + rr] = acc;
      __syncthreads();
      if (tid < CZT)
        xs[tid] = xs[tid] - (((red[tid] + red[CZT + tid]) + red[2 * CZT + tid]) + red[3 * CZT + tid]);
    } else {
      CT d[8];
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        CT a = zero<CT>();
#pragma unroll
        for (int t2 = 0; t2 < 4; ++t2) mac(a, conj_(widen_to<CT>(u[8 * t2 + cc])), xi[l + 32 * t2]);
        d[cc] = a;
      }
      const CT sum = tsum_lanes<8, CT>(d, l);  // lane l: column 8 w + (l >> 2)
      if ((l & 3) == 0) xs[8 * w + (l >> 2)] = xs[8 * w + (l >> 2)] - sum;
    }
    __syncthreads();
    if (t + 1 < nsrc)
#pragma unroll
      for (int u2 = 0; u2 < 32; ++u2) u[u2] = un[u2];
  }

  czstamp_any(4 * j + 1);
  // diagonal block: ONE warp; lane l owns the four consecutive rows 4l .. 4l+3
  // in registers.  Group g (rows 4g .. 4g+3, last to first for U, first to
  // last for U^H): lane g solves its 4 x 4 triangle serially in registers,
  // broadcasts the four values, every lane still to update subtracts their
  // column block from its rows.  The chain per four rows is one 4 x 4 solve
  // plus four shuffles (round 1 / earlier round 2: one shuffle per row); the
  // 16 coupling entries of the next group are loaded while the current one
  // runs (conflict-free 16-byte loads of four consecutive rows).
  if (w == 0) {
    CT xv[4];
    const int rq0 = 4 * l;
#pragma unroll
    for (int i = 0; i < 4; ++i) xv[i] = rq0 + i < bs ? xs[rq0 + i] : zero<CT>();
    // the lane's own 4 x 4 diagonal block (A[i][c] = Ud row rq0+i, col rq0+c),
    // pivots 1 for rows past bs
    CT dg[4][4], rpv[4], pvv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) dg[i][c] = widen_to<CT>(Ud[(rq0 + i) + (rq0 + c) * LU]);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      pvv[i] = rq0 + i < bs ? dg[i][i] : one<CT>();
      rpv[i] = recip(pvv[i]);
    }
    auto cload = [&](int g, CT (&u)[4][4]) {  // u[i][c] = Ud(rq0 + i, 4g + c)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const FT* cp = Ud + rq0 + (4 * g + c) * LU;
        if constexpr (sizeof(FT) == 4) {
          const float4 t4 = *reinterpret_cast<const float4*>(cp);
          u[0][c] = widen_to<CT>(t4.x), u[1][c] = widen_to<CT>(t4.y);
          u[2][c] = widen_to<CT>(t4.z), u[3][c] = widen_to<CT>(t4.w);
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) u[i][c] = widen_to<CT>(cp[i]);
        }
      }
    };
    constexpr int NG = CZT / 4;
    // binary32 compute: the next group's entries are loaded one group ahead;
    // wider types load them at the group start (registers), still ahead of
    // the owner's 4 x 4 solve
    constexpr bool AHEAD = sizeof(CT) == 4;
    CT ucur[4][4];
    if (AHEAD) cload(HERM ? 0 : NG - 1, ucur);
#pragma unroll 4
    for (int gg = 0; gg < NG; ++gg) {
      const int g = HERM ? gg : NG - 1 - gg;
      CT unext[AHEAD ? 4 : 1][AHEAD ? 4 : 1];
      if (!AHEAD) cload(g, ucur);
      if (AHEAD && gg + 1 < NG) cload(HERM ? g + 1 : g - 1, reinterpret_cast<CT(&)[4][4]>(unext));
      if (l == g) {  // the 4 x 4 triangle: backward (U) or forward (U^H)
        if (!HERM) {
#pragma unroll
          for (int i = 3; i >= 0; --i) {
            CT a = xv[i];
#pragma unroll
            for (int c = 3; c > i; --c) a = a - dg[i][c] * xv[c];
            xv[i] = qdiv(a, pvv[i], rpv[i]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            CT a = xv[i];
#pragma unroll
            for (int c = 0; c < i; ++c) a = a - dg[i][c] * xv[c];
            xv[i] = qdiv(a, pvv[i], rpv[i]);
          }
        }
      }
      CT xg[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) xg[c] = shfl_idx(xv[c], g);
      // rows still to update: !HERM lanes above the group, HERM lanes below
      const bool upd = !HERM ? (l < g) : (l > g);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        CT a = xv[i];
#pragma unroll
        for (int c = 0; c < 4; ++c) a = a - ucur[i][c] * xg[c];
        if (upd) xv[i] = a;
      }
      if (AHEAD && gg + 1 < NG)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int c = 0; c < 4; ++c) ucur[i][c] = reinterpret_cast<CT(&)[4][4]>(unext)[i][c];
    }
    // publish x_j straight from the registers: the release by lane 0 after the
    // warp barrier covers the whole warp's stores
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (rq0 + i < bs) x[i0 + rq0 + i] = xv[i];
    __syncwarp();
    if (l == 0) st_release(flags + j, 1);
  }
  czstamp_any(4 * j + 2);
}

// ------------------------------------------------------------------ MGS
// The modified Gram-Schmidt sweep of one GMRES step (gmres, krylov.hpp:436-512)
// in one cooperative launch: for i = 0 .. k, h_i = <w, V_i>, w -= h_i V_i
// (sequential in i, as MGS is), then h_{k+1} = <w, w>.  Thread e of the grid
// owns entry e of w in a register; each dot is a warp butterfly, a fixed-
// order sum over the CTA's warps, a per-step partial per CTA, one counter
// barrier, and the partials summed in CTA order by every CTA (so all CTAs
// subtract the same h_i).  V_{i+1}'s entry is loaded before the barrier.
// part: 2 x gridDim.x doubles (double-buffered by step parity); cnt: one
// int, zero at launch (arrival targets grow by gridDim.x per step).
__global__ void __launch_bounds__(1024, 1) k_mgs(const double* Vb, int N, int k, double* w, double* h,
                                                 double* part, int* cnt) {
  __shared__ double red[32];
  __shared__ double hsh;
  const int tid = threadIdx.x, l = tid & 31, wi = tid >> 5;
  const int c = blockIdx.x, G = gridDim.x;
  const int e = c * 1024 + tid;
  const bool in = e < N;
  double we = in ? w[e] : 0.0;
  double ve = (in && k >= 0) ? Vb[e] : 0.0;
  for (int i = 0; i <= k + 1; ++i) {
    const double y = i <= k ? ve : we;
    double s = we * y;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (l == 0) red[wi] = s;
    __syncthreads();
    double* ps = part + (i & 1) * G;
    if (tid == 0) {
      double t = 0.0;
#pragma unroll 8
      for (int q = 0; q < 32; ++q) t += red[q];
      ps[c] = t;
      asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(cnt) : "memory");
    }
    // the next basis vector's entry does not depend on this step
    const double vn = (in && i + 1 <= k) ? Vb[int64_t(i + 1) * N + e] : 0.0;
    if (tid == 0) {
      while (ld_acquire(cnt) < (i + 1) * G) {
      }
      double hs = 0.0;
      for (int q = 0; q < G; ++q) hs += ldcg_(ps + q);
      hsh = hs;
      if (c == 0) h[i] = hs;
    }
    __syncthreads();
    const double hi = hsh;
    if (i <= k) we = fma(-hi, ve, we);
    ve = vn;
  }
  if (in) w[e] = we;
}

}  // namespace lg
}  // namespace mlsb
