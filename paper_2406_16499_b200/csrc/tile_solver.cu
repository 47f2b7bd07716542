// Fused tile solver: ONE CTA solves ONE LSE or GLS problem end to end --
// pre-scaling, GRQ/GQR factorization at u_f held in shared memory, the
// initial solve, and every refinement pass (fp64 / double-double residual
// streamed from HBM, correction cascade at u_s against the shared-memory
// factors, stop test, divergence test) -- so a batch of problems is one
// launch with no host round trip.
//
// Reference semantics followed (paths relative to
// /root/reference/proj/include/mixedls):
//   pre-scaling                   lse.hpp:314-329, gls.hpp:287-297
//   reflector (xLARFG, fp64 norm) householder.hpp:30-53
//   RQ bottom-up, right-applied   householder.hpp:202-222 (+ factor.hpp:45 A Q^T)
//   QR left-applied               householder.hpp:173-190 (+ factor.hpp:65-67 Q^T V)
//   initial solve                 lse.hpp:346-366 (lse_direct_x :48-65, solve_v :156-173)
//                                 gls.hpp:313-326 (gls_direct_xy :47-65, init_z :71-82)
//   residuals                     lse.hpp:181-258, gls.hpp:161-232
//   stop test / divergence        lse.hpp:272-290, gls.hpp:246-264, refine.hpp:79-91
//   correction cascades           lse.hpp:83-128 (Alg. 1), gls.hpp:106-154 (Alg. 3)
//   demote / promote              refine.hpp:103-119
//   history (unscaled), status    lse.hpp:382-396, gls.hpp:341-355
//   unscale                       lse.hpp:424-426, gls.hpp:382-384
//
// Stacked storage in shared memory (column-major, odd leading dimension so
// both row and column sweeps are bank-conflict free):
//   LSE  M = [A; B]  ((m+p) x n): RQ of rows m..m+p-1 applied to every row
//        above (this is rq(B) followed by C = A Q^T), then QR of M[0:m, 0:n].
//   GLS  M = [W  V]  (n x (m+p)): QR of columns 0..m-1 applied to every
//        column to the right (qr(W) followed by Q^T V), then RQ of M[:, m:].
// Reflectors are stored LAPACK-packed (below the diagonal for QR, left of
// the pivot for RQ) with the unit entry implicit.
//
// Numerics differ from the reference only in summation order (tree and
// FMA instead of sequential), and the scaled fp64 data is formed as
// a * (1/s) instead of a / s (<= 1 ulp of the scaled entry).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "device_common.cuh"
#include "mlsb_internal.h"

namespace mlsb {

constexpr int NT = 512;
constexpr int NW = NT / 32;
constexpr int RPL = 2;         // rows per lane in a residual chunk
constexpr int CH = 32 * RPL;   // rows per residual chunk
constexpr int NWORK = 8;       // solve-precision work vectors
constexpr size_t kStaticSmem = 512;  // qr_stage's static mbarrier ring, counted against the limit

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

struct Layout {
  int R, C, ld, L;
  size_t oM, oTau1, oTau2, oRinit, oRinitC, oRout, oSw, oCout, oCacc, oCaccC, oSu, oWork,
      oPart, oRed, oScal, total;
};

__host__ __device__ inline Layout make_layout(int kind, int64_t m, int64_t n, int64_t p,
                                              int fsz, int csz, bool ext, bool m_global = false) {
  Layout L;
  L.R = int(kind == KIND_LSE ? m + p : n);
  L.C = int(kind == KIND_LSE ? n : m + p);
  L.ld = L.R | 1;
  L.L = L.R > L.C ? L.R : L.C;
  size_t o = 0;
  L.oM = o;       o = al16(o + (m_global ? 0 : size_t(L.ld) * L.C * fsz));
  L.oTau1 = o;    o = al16(o + size_t(L.C) * fsz);
  L.oTau2 = o;    o = al16(o + size_t(L.R) * fsz);
  L.oRinit = o;   o = al16(o + size_t(L.R) * 8);
  L.oRinitC = o;  o = al16(o + size_t(ext ? L.R : 0) * 8);
  L.oRout = o;    o = al16(o + size_t(L.R) * 8);
  L.oSw = o;      o = al16(o + size_t(L.R) * 8);
  L.oCout = o;    o = al16(o + size_t(L.C) * 8);
  L.oCacc = o;    o = al16(o + size_t(L.C) * 8);
  L.oCaccC = o;   o = al16(o + size_t(ext ? L.C : 0) * 8);
  L.oSu = o;      o = al16(o + size_t(L.C) * 8);
  L.oWork = o;    o = al16(o + size_t(NWORK) * L.L * (csz > fsz ? csz : fsz));
  L.oPart = o;    o = al16(o + size_t(NW) * CH * 8 * (ext ? 2 : 1));
  L.oRed = o;     o = al16(o + size_t(NW) * 8 * 8);
  L.oScal = o;    o = al16(o + 64 * 8);
  L.total = o;
  return L;
}

// scalar slots in the shared `scal` array
enum Slot {
  S_SA = 0, S_SB, S_CB, S_CD, S_NB, S_ND, S_NA, S_NBF,  // scales and problem norms
  S_SIG, S_BEST, S_BETA, S_TMP,                         // sigma, divergence min, reflector beta
  S_RED0 = 16,                                          // block-reduction results (8)
  S_FLAG = 32,                                          // int flags (stored as double bits)
};

// ====================== reflector-factor vector applies =====================
// QR-type factor Q = H_0 ... H_{k-1}; H_j = I - tau_j v v^T, v = [1; M[j+1:rend, j]]
// (householder.hpp:114-129).  One warp; x in shared memory.
//
// Reflectors go two at a time: one pass over the rows accumulates v1.x, v2.x
// and v1.v2, then x -= b1 v1 + b2 v2 with b1 = t1 (v1.x), b2 = t2 (v2.x -
// b1 v1.v2) -- the same product H2 H1 x with one warp reduction and one
// update sweep per pair instead of per reflector.
template <class FT, class CT>
__device__ void qrf_apply(const FT* M, int ld, const FT* tau, int k, int rend, CT* x, bool herm,
                          int lane) {
  int s0 = 0;
  for (; s0 + 1 < k; s0 += 2) {
    const int j1 = herm ? s0 : (k - 1 - s0), j2 = herm ? s0 + 1 : (k - 2 - s0);
    const CT t1 = CT(tau[j1]), t2 = CT(tau[j2]);
    const int lo = j1 < j2 ? j1 : j2, hi = lo + 1;
    const FT* v1 = M + size_t(j1) * ld;
    const FT* v2 = M + size_t(j2) * ld;
    CT a1 = CT(0), a2 = CT(0), gg = CT(0);
    for (int i = hi + 1 + lane; i < rend; i += 32) {
      const CT xi = x[i], e1 = CT(v1[i]), e2 = CT(v2[i]);
      a1 += e1 * xi;
      a2 += e2 * xi;
      gg += e1 * e2;
    }
    const CT xlo = x[lo], xhi = hi < rend ? x[hi] : CT(0);
    const CT mh = hi < rend ? CT(M[hi + size_t(lo) * ld]) : CT(0);  // v_lo at row hi
    a1 = warp_sum(a1);
    a2 = warp_sum(a2);
    gg = warp_sum(gg);
    // full dots: v_lo = [1 at lo, mh at hi, ...], v_hi = [0 at lo, 1 at hi, ...]
    const bool f_lo = j1 == lo;
    const CT dlo = (f_lo ? a1 : a2) + xlo + mh * xhi, dhi = (f_lo ? a2 : a1) + xhi;
    const CT d1 = f_lo ? dlo : dhi, d2 = f_lo ? dhi : dlo;
    const CT b1 = t1 * d1, b2 = t2 * (d2 - b1 * (gg + mh));
    const CT blo = f_lo ? b1 : b2, bhi = f_lo ? b2 : b1;
    __syncwarp();
    if (lane == 0) {
      x[lo] = xlo - blo;
      if (hi < rend) x[hi] = xhi - (blo * mh + bhi);
    }
    for (int i = hi + 1 + lane; i < rend; i += 32) x[i] -= b1 * CT(v1[i]) + b2 * CT(v2[i]);
    __syncwarp();
  }
  for (int s = s0; s < k; ++s) {
    const int j = herm ? s : (k - 1 - s);
    const CT t = CT(tau[j]);
    if (t == CT(0)) continue;
    const FT* v = M + size_t(j) * ld;
    CT acc = CT(0);
    for (int i = j + 1 + lane; i < rend; i += 32) acc += CT(v[i]) * x[i];
    acc = warp_sum(acc);
    acc = (acc + x[j]) * t;
    __syncwarp();
    if (lane == 0) x[j] -= acc;
    for (int i = j + 1 + lane; i < rend; i += 32) x[i] -= acc * CT(v[i]);
    __syncwarp();
  }
}

// RQ-type factor Z = H_0 ... H_{kk-1}; reflector j lives in row rtop+j, entries
// at columns c0+t for t < ptop+j, unit at t = ptop+j (householder.hpp:202-222).
// Two reflectors per step as in qrf_apply (columns reversed: v_lo has its
// unit at pc_lo, v_hi its unit at pc_lo + 1 and a stored entry at pc_lo).
template <class FT, class CT>
__device__ void rqf_apply(const FT* M, int ld, const FT* tau, int kk, int rtop, int c0, int ptop,
                          CT* x, bool herm, int lane) {
  int s0 = 0;
  for (; s0 + 1 < kk; s0 += 2) {
    const int j1 = herm ? s0 : (kk - 1 - s0), j2 = herm ? s0 + 1 : (kk - 2 - s0);
    const CT t1 = CT(tau[j1]), t2 = CT(tau[j2]);
    const int jl = j1 < j2 ? j1 : j2;
    const int pl = ptop + jl, ph = pl + 1;
    const FT* v1 = M + (rtop + j1) + size_t(c0) * ld;
    const FT* v2 = M + (rtop + j2) + size_t(c0) * ld;
    CT a1 = CT(0), a2 = CT(0), gg = CT(0);
    for (int q = lane; q < pl; q += 32) {
      const CT xq = x[q], e1 = CT(v1[size_t(q) * ld]), e2 = CT(v2[size_t(q) * ld]);
      a1 += e1 * xq;
      a2 += e2 * xq;
      gg += e1 * e2;
    }
    const bool f_lo = j1 == jl;
    const CT xl = x[pl], xh = x[ph];
    const CT mh = CT((f_lo ? v2 : v1)[size_t(pl) * ld]);  // v_hi at column pl
    a1 = warp_sum(a1);
    a2 = warp_sum(a2);
    gg = warp_sum(gg);
    const CT dlo = (f_lo ? a1 : a2) + xl, dhi = (f_lo ? a2 : a1) + mh * xl + xh;
    const CT d1 = f_lo ? dlo : dhi, d2 = f_lo ? dhi : dlo;
    const CT b1 = t1 * d1, b2 = t2 * (d2 - b1 * (gg + mh));
    const CT blo = f_lo ? b1 : b2, bhi = f_lo ? b2 : b1;
    __syncwarp();
    if (lane == 0) {
      x[pl] = xl - (blo + bhi * mh);
      x[ph] = xh - bhi;
    }
    for (int q = lane; q < pl; q += 32)
      x[q] -= b1 * CT(v1[size_t(q) * ld]) + b2 * CT(v2[size_t(q) * ld]);
    __syncwarp();
  }
  for (int s = s0; s < kk; ++s) {
    const int j = herm ? s : (kk - 1 - s);
    const CT t = CT(tau[j]);
    if (t == CT(0)) continue;
    const int pc = ptop + j;
    const FT* vrow = M + (rtop + j) + size_t(c0) * ld;
    CT acc = CT(0);
    for (int q = lane; q < pc; q += 32) acc += CT(vrow[size_t(q) * ld]) * x[q];
    acc = warp_sum(acc);
    acc = (acc + x[pc]) * t;
    __syncwarp();
    if (lane == 0) x[pc] -= acc;
    for (int q = lane; q < pc; q += 32) x[q] -= acc * CT(vrow[size_t(q) * ld]);
    __syncwarp();
  }
}

// ========================= triangular solves (one warp) =====================
// U = M[r0:r0+k, c0:c0+k] upper triangular; x overwritten.  Returns false and
// sets *bad to the block-relative pivot index on an exact zero pivot, in the
// same sweep order as trsv_sub (matrix.hpp:242-267).
// Columns go two at a time (same operations in the same order as one at a
// time, so bitwise equal): one update sweep and two warp syncs per pair.
template <class FT, class CT>
__device__ bool trsv_n(const FT* M, int ld, int r0, int c0, int k, CT* x, int lane, int* bad) {
  int jj = k - 1;
  for (; jj >= 1; jj -= 2) {
    const FT* col = M + size_t(c0 + jj) * ld + r0;
    const FT* cl1 = col - ld;
    const CT piv = CT(col[jj]), piv1 = CT(cl1[jj - 1]);
    if (piv == CT(0) || piv1 == CT(0)) break;  // the single-column loop reports it
    const CT xj = x[jj] / piv;
    const CT xj1 = (x[jj - 1] - xj * CT(col[jj - 1])) / piv1;
    __syncwarp();
    if (lane == 0) {
      x[jj] = xj;
      x[jj - 1] = xj1;
    }
    for (int i = lane; i < jj - 1; i += 32) x[i] = (x[i] - xj * CT(col[i])) - xj1 * CT(cl1[i]);
    __syncwarp();
  }
  for (; jj >= 0; --jj) {
    const FT* col = M + size_t(c0 + jj) * ld + r0;
    const CT piv = CT(col[jj]);
    if (piv == CT(0)) {
      if (lane == 0) *bad = jj;
      __syncwarp();
      return false;
    }
    const CT xj = x[jj] / piv;
    __syncwarp();
    if (lane == 0) x[jj] = xj;
    for (int i = lane; i < jj; i += 32) x[i] -= xj * CT(col[i]);
    __syncwarp();
  }
  return true;
}
// U^T x = b as a forward column sweep over the rows of U
template <class FT, class CT>
__device__ bool trsv_t(const FT* M, int ld, int r0, int c0, int k, CT* x, int lane, int* bad) {
  int j = 0;
  for (; j + 1 < k; j += 2) {
    const FT* row = M + (r0 + j) + size_t(c0) * ld;
    const FT* rw1 = row + 1;
    const CT piv = CT(row[size_t(j) * ld]), piv1 = CT(rw1[size_t(j + 1) * ld]);
    if (piv == CT(0) || piv1 == CT(0)) break;  // the single-row loop reports it
    const CT xj = x[j] / piv;
    const CT xj1 = (x[j + 1] - CT(row[size_t(j + 1) * ld]) * xj) / piv1;
    __syncwarp();
    if (lane == 0) {
      x[j] = xj;
      x[j + 1] = xj1;
    }
    for (int i = j + 2 + lane; i < k; i += 32)
      x[i] = (x[i] - CT(row[size_t(i) * ld]) * xj) - CT(rw1[size_t(i) * ld]) * xj1;
    __syncwarp();
  }
  for (; j < k; ++j) {
    const FT* row = M + (r0 + j) + size_t(c0) * ld;
    const CT piv = CT(row[size_t(j) * ld]);
    if (piv == CT(0)) {
      if (lane == 0) *bad = j;
      __syncwarp();
      return false;
    }
    const CT xj = x[j] / piv;
    __syncwarp();
    if (lane == 0) x[j] = xj;
    for (int i = j + 1 + lane; i < k; i += 32) x[i] -= CT(row[size_t(i) * ld]) * xj;
    __syncwarp();
  }
  return true;
}

// ============================= block GEMVs ================================
// Entries of the stacked matrix that hold packed reflectors read as zero.
struct NoMask {
  __device__ bool zero(int, int) const { return false; }
};
struct LowerMask {  // QR region: rows below the diagonal hold reflectors
  __device__ bool zero(int i, int j) const { return i > j; }
};
struct RqMask {  // RQ region of GLS: row r >= rtop, column c < c0 + (r - rtop) + ptop
  int rtop, c0, ptop;
  __device__ bool zero(int i, int j) const { return i >= rtop && j < c0 + (i - rtop) + ptop; }
};

// y[i] = sum_j M(r0+i, c0+j) x[j], thread-per-row over threads [t0, t0+nth)
template <class FT, class CT, class Mk>
__device__ void gemv_n(const FT* M, int ld, int r0, int rows, int c0, int cols, const CT* x,
                       CT* y, Mk mk, int t, int nth) {
  for (int i = t; i < rows; i += nth) {
    CT acc = CT(0);
    const FT* rowp = M + (r0 + i) + size_t(c0) * ld;
    for (int j = 0; j < cols; ++j)
      if (!mk.zero(r0 + i, c0 + j)) acc += CT(rowp[size_t(j) * ld]) * x[j];
    y[i] = acc;
  }
}
// y[j] = sum_i M(r0+i, c0+j) x[i], thread-per-column
template <class FT, class CT, class Mk>
__device__ void gemv_t(const FT* M, int ld, int r0, int rows, int c0, int cols, const CT* x,
                       CT* y, Mk mk, int t, int nth) {
  for (int j = t; j < cols; j += nth) {
    CT acc = CT(0);
    const FT* colp = M + size_t(c0 + j) * ld + r0;
    for (int i = 0; i < rows; ++i)
      if (!mk.zero(r0 + i, c0 + j)) acc += CT(colp[i]) * x[i];
    y[j] = acc;
  }
}

// ============================ factorization ================================
// xLARFG on a column held by one warp: x = col[j+1:rend], alpha = col[j].
template <class FT>
__device__ void gen_col_reflector(FT* col, int j, int rend, FT* tau_j, int lane) {
  __syncwarp();
  double ss = 0.0;
  for (int i = j + 1 + lane; i < rend; i += 32) {
    const double t = double(col[i]);
    ss = fma(t, t, ss);
  }
  ss = warp_sum(ss);
  const double xn = sqrt(ss);
  const FT alpha = col[j];
  if (xn == 0.0) {
    if (lane == 0) *tau_j = FT(0);
    __syncwarp();
    return;
  }
  const double a = double(alpha);
  // binary32 data cannot overflow a binary64 a^2 + ss: one sqrt instead of
  // sqrt + hypot on the reflector chain
  const double beta = -copysign(sizeof(FT) == 4 ? sqrt(fma(a, a, ss)) : hypot(a, xn), a);
  const FT tj = FT((beta - a) / beta);
  const FT inv = FT(1.0 / (a - beta));
  for (int i = j + 1 + lane; i < rend; i += 32) col[i] = col[i] * inv;
  __syncwarp();
  if (lane == 0) {
    *tau_j = tj;
    col[j] = FT(beta);
  }
  __syncwarp();
}

// Four warp sums at once, bitwise equal to four warp_sum() butterflies (same
// pairs at every level) in 10 shuffles instead of 20: the first two levels
// halve the number of live values per lane (transposed reduction), the last
// three are a plain butterfly, and the totals are broadcast back.
template <class FT>
__device__ __forceinline__ void warp_sum4(FT s[4], int lane) {
  const bool h = lane & 16, g = lane & 8;
  const FT y0 = __shfl_xor_sync(0xffffffffu, h ? s[0] : s[2], 16);
  const FT y1 = __shfl_xor_sync(0xffffffffu, h ? s[1] : s[3], 16);
  const FT t0 = (h ? s[2] : s[0]) + y0;  // column 2h
  const FT t1 = (h ? s[3] : s[1]) + y1;  // column 2h + 1
  const FT y = __shfl_xor_sync(0xffffffffu, g ? t0 : t1, 8);
  FT u = (g ? t1 : t0) + y;  // column 2h + g
  u += __shfl_xor_sync(0xffffffffu, u, 4);
  u += __shfl_xor_sync(0xffffffffu, u, 2);
  u += __shfl_xor_sync(0xffffffffu, u, 1);
#pragma unroll
  for (int c = 0; c < 4; ++c) s[c] = __shfl_sync(0xffffffffu, u, (c >> 1) * 16 + (c & 1) * 8);
}

// H_j applied to a group of CG columns c, c+NW, ... of one warp (columns past
// cend are clamped and not written): one pass for the CG dots, one
// transposed reduction per four columns, one update pass.
template <class FT, int CG>
__device__ __forceinline__ void qr_cols(FT* M, int ld, const FT* v, int c, int cend, int j,
                                        int rend, FT tj, int lane) {
  FT s[CG];
  FT* cc[CG];
#pragma unroll
  for (int u = 0; u < CG; ++u) {
    s[u] = FT(0);
    cc[u] = M + size_t(min(c + u * NW, cend - 1)) * ld;
  }
#pragma unroll 4
  for (int i = j + 1 + lane; i < rend; i += 32) {
    const FT vi = v[i];
#pragma unroll
    for (int u = 0; u < CG; ++u) s[u] += vi * cc[u][i];
  }
  FT cj[CG];
#pragma unroll
  for (int u = 0; u < CG; ++u) cj[u] = cc[u][j];
#pragma unroll
  for (int g = 0; g < CG; g += 4) warp_sum4(s + g, lane);
  __syncwarp();  // every lane has read cc[u][j] before lane 0 rewrites it
  bool live[CG];
#pragma unroll
  for (int u = 0; u < CG; ++u) {
    live[u] = c + u * NW < cend;
    s[u] = (s[u] + cj[u]) * tj;
    if (lane == 0 && live[u]) cc[u][j] = cj[u] - s[u];
  }
  // one pass over the rows for all columns: v[i] read once, the column loads
  // independent of each other (no per-column latency chain)
#pragma unroll 4
  for (int i = j + 1 + lane; i < rend; i += 32) {
    const FT vi = v[i];
#pragma unroll
    for (int u = 0; u < CG; ++u)
      if (live[u]) cc[u][i] -= s[u] * vi;
  }
}

// QR of columns [0, k) over rows [0, rend), applied to columns < cend.
// One reflector per step; column c is owned by warp c % NW, and the owner of
// column j+1 generates reflector j+1 right after applying H_j to it
// (look-ahead), so each step costs one CTA barrier.
//
// Reflector j is published through a ring of mbarriers (one arrival: the
// owner warp's lane 0 after a __syncwarp) instead of a CTA barrier per step:
// a warp waits only for the reflector it applies next, so the owner of column
// j+1 never waits for the slowest warp's bulk updates.  Every warp owns a
// column every NW steps, so no warp lags more than NW steps: a ring of 2 NW
// barriers cannot wrap onto a pending phase.
template <class FT, bool WIDE = false>
__device__ __forceinline__ void qr_stage(FT* M, int ld, int rend, int k, int cend, FT* tau, int warp, int lane) {
  if (k <= 0) return;
  constexpr int NQB = 2 * NW;
  __shared__ uint64_t qbar[NQB];
  if (warp == 0 && lane < NQB) mbar_init(&qbar[lane], 1);
  __syncthreads();
  if (warp == 0) {
    gen_col_reflector(M, 0, rend, &tau[0], lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&qbar[0]);
  }
  for (int j = 0; j < k; ++j) {
    mbar_wait(&qbar[j % NQB], (j / NQB) & 1);
    const FT tj = tau[j];
    const FT* v = M + size_t(j) * ld;
    int c = j + 1 + ((warp - (j + 1)) % NW + NW) % NW;
    // the owner's column j+1 first (it feeds the next reflector), then the
    // warp's other columns four at a time so their warp sums overlap
    if (c == j + 1 && c < cend) {
      FT* cc = M + size_t(c) * ld;
      if (tj != FT(0)) {
        FT s = FT(0);
        for (int i = j + 1 + lane; i < rend; i += 32) s += v[i] * cc[i];
        s = warp_sum(s);
        s = (s + cc[j]) * tj;
        __syncwarp();
        if (lane == 0) cc[j] -= s;
        for (int i = j + 1 + lane; i < rend; i += 32) cc[i] -= s * v[i];
      }
      if (c < k) {
        gen_col_reflector(cc, c, rend, &tau[c], lane);
        __syncwarp();  // the warp's writes of v_{j+1} and tau before lane 0's release
        if (lane == 0) mbar_arrive(&qbar[c % NQB]);
      }
      c += NW;
    }
    if (tj != FT(0)) {
      // eight binary32 columns fit the register budget with shared-memory
      // (32-bit) addressing; 64-bit global pointers would spill
      if constexpr (WIDE && sizeof(FT) == 4)
        for (; c + 7 * NW < cend; c += 8 * NW) qr_cols<FT, 8>(M, ld, v, c, cend, j, rend, tj, lane);
      for (; c < cend; c += 4 * NW) qr_cols<FT, 4>(M, ld, v, c, cend, j, rend, tj, lane);
    }
  }
  __syncthreads();
}

// RQ of the block rows [rb, rb+rr) x columns [c0, c0+cc); reflector j is
// generated from row rb+rr-kk+j and applied from the right to every row
// above it.  The reference's sequential row-dot order is kept per thread.
template <class FT>
__device__ __forceinline__ void rq_stage(FT* M, int ld, int rb, int rr, int c0, int cc, FT* tau, double* scal,
                         int tid, int warp, int lane) {
  const int kk = rr < cc ? rr : cc;
  for (int j = kk - 1; j >= 0; --j) {
    const int row = rb + rr - kk + j, pc = cc - kk + j;
    FT* vrow = M + row + size_t(c0) * ld;
    if (warp == 0) {
      double ss = 0.0;
      for (int q = lane; q < pc; q += 32) {
        const double t = double(vrow[size_t(q) * ld]);
        ss = fma(t, t, ss);
      }
      ss = warp_sum(ss);
      const double xn = sqrt(ss);
      const FT alpha = vrow[size_t(pc) * ld];
      FT tj = FT(0), beta = alpha;
      if (xn != 0.0) {
        const double a = double(alpha);
        const double bt = -copysign(sizeof(FT) == 4 ? sqrt(fma(a, a, ss)) : hypot(a, xn), a);
        tj = FT((bt - a) / bt);
        const FT inv = FT(1.0 / (a - bt));
        for (int q = lane; q < pc; q += 32) vrow[size_t(q) * ld] = vrow[size_t(q) * ld] * inv;
        beta = FT(bt);
      }
      if (lane == 0) {
        tau[j] = tj;
        scal[S_BETA] = double(beta);
      }
    }
    __syncthreads();
    const FT tj = tau[j];
    if (tj != FT(0)) {
      // 4 threads per row (adjacent lanes), each with every fourth column of
      // the row's dot: chains of ~pc/4 FMAs instead of pc, every thread of
      // the CTA busy; the phases are combined as (p0 + p1) + (p2 + p3) (same
      // in every lane).  Two rows (i, i + NT/4) per thread when both passes are live,
      // so each v element is loaded once for both.
      // Thread (r8, c) of a warp takes row wrow + 4 r8 and columns c, c+4, ...:
      // banks (4 r8 + c ld) mod 32 are distinct for any odd ld, so the
      // 8 rows x 4 column phases of a warp access are conflict-free.
      const int c = lane & 3, r8 = lane >> 2;
      const int qa = min(pc, c), qb = pc;
      const size_t st = size_t(4) * ld;
      const int wrow = 32 * (warp >> 2) + (warp & 3);
      const FT* vq = vrow + size_t(qa) * ld;
      FT* Mc = M + size_t(c0) * ld;  // column block of this stage
      for (int i0 = 0; i0 + wrow < row; i0 += NT / 2) {
        const int i = i0 + wrow + 4 * r8;
        const bool ok = i < row;
        if (i0 + NT / 4 + wrow < row) {  // warp-uniform: second pass live
          const bool ok2 = i + NT / 4 < row;
          FT* a1 = Mc + i + size_t(qa) * ld;
          FT* a2 = Mc + (ok2 ? i + NT / 4 : i) + size_t(qa) * ld;
          const FT apc1 = Mc[i + size_t(pc) * ld];
          const FT apc2 = ok2 ? Mc[i + NT / 4 + size_t(pc) * ld] : FT(0);
          FT w1 = FT(0), w2 = FT(0);
          {
            const FT *v = vq, *p1 = a1, *p2 = a2;
#pragma unroll 4
            for (int q = qa; q < qb; q += 4, v += st, p1 += st, p2 += st) {
              const FT vv = *v;
              w1 += vv * *p1;
              w2 += vv * *p2;
            }
          }
          w1 += __shfl_xor_sync(0xffffffffu, w1, 1);
          w2 += __shfl_xor_sync(0xffffffffu, w2, 1);
          w1 += __shfl_xor_sync(0xffffffffu, w1, 2);
          w2 += __shfl_xor_sync(0xffffffffu, w2, 2);
          w1 += apc1;
          w2 += apc2;
          {
            const FT* v = vq;
            FT *p1 = a1, *p2 = a2;
#pragma unroll 4
            for (int q = qa; q < qb; q += 4, v += st, p1 += st, p2 += st) {
              const FT tv = tj * *v;
              *p1 -= tv * w1;
              if (ok2) *p2 -= tv * w2;
            }
          }
          if (c == 0) {
            Mc[i + size_t(pc) * ld] = apc1 - tj * w1;
            if (ok2) Mc[i + NT / 4 + size_t(pc) * ld] = apc2 - tj * w2;
          }
        } else {
          FT* arow = Mc + (ok ? i : 0);
          FT w = FT(0);
          const FT apc = ok ? arow[size_t(pc) * ld] : FT(0);
          if (ok) {
            const FT* v = vq;
            const FT* p1 = arow + size_t(qa) * ld;
#pragma unroll 4
            for (int q = qa; q < qb; q += 4, v += st, p1 += st) w += *v * *p1;
          }
          w += __shfl_xor_sync(0xffffffffu, w, 1);
          w += __shfl_xor_sync(0xffffffffu, w, 2);
          w += apc;
          if (ok) {
            const FT* v = vq;
            FT* p1 = arow + size_t(qa) * ld;
#pragma unroll 4
            for (int q = qa; q < qb; q += 4, v += st, p1 += st) *p1 -= (tj * *v) * w;
            if (c == 0) arow[size_t(pc) * ld] = apc - tj * w;
          }
        }
      }
    }
    if (tid == 0) vrow[size_t(pc) * ld] = FT(scal[S_BETA]);
    __syncthreads();
  }
}

// ============================== kernel =====================================
// MG: factors in the global workspace (a.gws) instead of shared memory; a
// template parameter so that the shared-memory instantiation addresses M
// with LDS/STS instead of generic loads.
template <int KIND, class FT, class CT, bool EXT, bool MG>
__global__ void __launch_bounds__(NT, 1) tile_solve_kernel(TileArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t pid = blockIdx.x;
  const int m = int(a.m), n = int(a.n), p = int(a.p);
  const Layout Ly = make_layout(KIND, m, n, p, sizeof(FT), sizeof(CT), EXT, MG);
  const int R = Ly.R, C = Ly.C, ld = Ly.ld;
  constexpr bool LOWF = sizeof(FT) == 4;
  constexpr bool LOWS = sizeof(CT) == 4;

  // the stacked factor matrix lives in shared memory, or -- when it does not
  // fit -- in a per-problem global workspace that stays L2-resident
  FT* M = MG ? reinterpret_cast<FT*>(a.gws) + size_t(pid) * size_t(ld) * C
             : reinterpret_cast<FT*>(smem + Ly.oM);
  FT* tau1 = reinterpret_cast<FT*>(smem + Ly.oTau1);
  FT* tau2 = reinterpret_cast<FT*>(smem + Ly.oTau2);
  double* rinit = reinterpret_cast<double*>(smem + Ly.oRinit);
  double* rinitc = reinterpret_cast<double*>(smem + Ly.oRinitC);
  double* rout = reinterpret_cast<double*>(smem + Ly.oRout);
  double* sw = reinterpret_cast<double*>(smem + Ly.oSw);
  double* cout = reinterpret_cast<double*>(smem + Ly.oCout);
  double* cacc = reinterpret_cast<double*>(smem + Ly.oCacc);
  double* caccc = reinterpret_cast<double*>(smem + Ly.oCaccC);
  double* su = reinterpret_cast<double*>(smem + Ly.oSu);
  unsigned char* work = smem + Ly.oWork;
  const size_t wstride = size_t(Ly.L) * (sizeof(CT) > sizeof(FT) ? sizeof(CT) : sizeof(FT));
  auto WC = [&](int i) { return reinterpret_cast<CT*>(work + i * wstride); };
  auto WF = [&](int i) { return reinterpret_cast<FT*>(work + i * wstride); };
  double* part = reinterpret_cast<double*>(smem + Ly.oPart);
  double* red = reinterpret_cast<double*>(smem + Ly.oRed);
  double* scal = reinterpret_cast<double*>(smem + Ly.oScal);
  int* iflag = reinterpret_cast<int*>(scal + S_FLAG);  // [0] error code, [1] pivot index

  const double* gA = a.A + pid * a.sA;
  const double* gB = a.B + pid * a.sB;
  const double* gb = (KIND == KIND_LSE) ? a.b + pid * a.sb : nullptr;
  const double* gd = a.d + pid * a.sd;

  uint64_t t_last = 0;
  double ph[6] = {0, 0, 0, 0, 0, 0};
  auto lap = [&](int slot) {
    if (tid == 0) {
      const uint64_t t = globaltimer_ns();
      ph[slot] += double(t - t_last) * 1e-9;
      t_last = t;
    }
  };
  if (tid == 0) t_last = globaltimer_ns();
  if (a.stamps && pid == 0 && tid == 0) a.stamps[0] = t_last;  // debug: kernel start
  if (tid == 0) {
    iflag[0] = 0;
    iflag[1] = -1;
  }

  // stacked global element (i, j) of M and its scale reciprocal
  auto gval = [&](int i, int j) -> double {
    if (KIND == KIND_LSE)
      return i < m ? __ldg(gA + i + size_t(j) * a.lda) : __ldg(gB + (i - m) + size_t(j) * a.ldb);
    else
      return j < m ? __ldg(gA + i + size_t(j) * a.lda) : __ldg(gB + i + size_t(j - m) * a.ldb);
  };

  // ---------------- pre-scaling (lse.hpp:314-329 / gls.hpp:287-297) ----------
  double invA = 1.0, invB = 1.0;  // reciprocals of s_A, s_B (s_W, s_V)
  {
    double mx[3] = {0.0, 0.0, 0.0};
    if (LOWF) {
      for (int j = warp; j < C; j += NW)
        for (int i = lane; i < R; i += 32) {
          const double t = fabs(gval(i, j));
          const bool first = (KIND == KIND_LSE) ? (i < m) : (j < m);
          if (first) mx[0] = nanskip_max(mx[0], t);
          else mx[1] = nanskip_max(mx[1], t);
        }
      if (KIND == KIND_LSE)
        for (int i = tid; i < m; i += NT) mx[2] = nanskip_max(mx[2], fabs(__ldg(gb + i)));
      else
        for (int i = tid; i < n; i += NT) mx[2] = nanskip_max(mx[2], fabs(__ldg(gd + i)));
    }
    block_max(mx, red, scal + S_RED0);
    if (tid == 0) {
      double sA = 1.0, sB = 1.0, c1 = 1.0, c2 = 1.0;
      if (LOWF) {
        sA = scal[S_RED0] == 0.0 ? 1.0 : scal[S_RED0];
        sB = scal[S_RED0 + 1] == 0.0 ? 1.0 : scal[S_RED0 + 1];
        c1 = scal[S_RED0 + 2] == 0.0 ? 1.0 : scal[S_RED0 + 2];
        c2 = (KIND == KIND_LSE) ? sB * c1 / sA : c1;
      }
      scal[S_SA] = sA;
      scal[S_SB] = sB;
      scal[S_CB] = c1;  // LSE c_b ; GLS c_d
      scal[S_CD] = c2;  // LSE c_d ; GLS c_d
    }
    __syncthreads();
    if (LOWF) {
      invA = 1.0 / scal[S_SA];
      invB = 1.0 / scal[S_SB];
    }
  }
  auto sval = [&](int i, int j) -> double {  // scaled fp64 entry of the stacked matrix
    const double g = gval(i, j);
    if (!LOWF) return g;
    const bool first = (KIND == KIND_LSE) ? (i < m) : (j < m);
    return g * (first ? invA : invB);
  };

  // scaled right-hand sides and the state-independent row initialisers
  if (KIND == KIND_LSE) {
    const double cb = scal[S_CB], cd = scal[S_CD];
    for (int i = tid; i < R; i += NT) rinit[i] = i < m ? __ldg(gb + i) / cb : __ldg(a.d + pid * a.sd + (i - m)) / cd;
  } else {
    const double cd = scal[S_CD];
    for (int i = tid; i < n; i += NT) rinit[i] = __ldg(gd + i) / cd;
  }
  __syncthreads();
  if (KIND == KIND_LSE) {
    // "rhs scaling overflowed" (lse.hpp:328-329)
    int bad = 0;
    for (int i = m + tid; i < R; i += NT) bad |= !isfinite(rinit[i]);
    bad = __syncthreads_or(bad);
    if (bad) {
      if (tid == 0) iflag[0] = 2;
      goto finish;
    }
  }

  // ---------------- cast to u_f + problem Frobenius norms ---------------------
  {
    double ss[2] = {0.0, 0.0};
    for (int j = warp; j < C; j += NW)
      for (int i = lane; i < R; i += 32) {
        const double t = sval(i, j);
        const bool first = (KIND == KIND_LSE) ? (i < m) : (j < m);
        if (first) ss[0] = fma(t, t, ss[0]); else ss[1] = fma(t, t, ss[1]);
        M[i + size_t(j) * ld] = FT(t);
      }
    double nv[2] = {0.0, 0.0};
    // rhs norm (||b|| for LSE plus ||d||; ||d|| for GLS)
    for (int i = tid; i < R; i += NT) {
      const double t = rinit[i];
      const bool first = (KIND == KIND_LSE) ? (i < m) : true;
      if (first) nv[0] = fma(t, t, nv[0]); else nv[1] = fma(t, t, nv[1]);
    }
    double all4[4] = {ss[0], ss[1], nv[0], nv[1]};
    block_sum(all4, red, scal + S_RED0);
    if (tid == 0) {
      scal[S_NA] = sqrt(scal[S_RED0]);       // ||A_s||_F  (GLS ||W_s||_F)
      scal[S_NBF] = sqrt(scal[S_RED0 + 1]);  // ||B_s||_F  (GLS ||V_s||_F)
      if (KIND == KIND_LSE) {
        scal[S_NB] = sqrt(scal[S_RED0 + 2]);  // ||b_s||
        scal[S_ND] = sqrt(scal[S_RED0 + 3]);  // ||d_s||
      } else {
        scal[S_ND] = sqrt(scal[S_RED0 + 2]);  // ||d_s||
      }
    }
  }
  __syncthreads();
  lap(5);
  if (a.stamps && pid == 0 && tid == 0) a.stamps[29] = globaltimer_ns();  // debug: factorization start

  // ---------------- GRQ / GQR at u_f ------------------------------------------
  if (KIND == KIND_LSE) {
    rq_stage<FT>(M, ld, m, p, 0, n, tau2, scal, tid, warp, lane);
    qr_stage<FT, !MG>(M, ld, m, m < n ? m : n, n, tau1, warp, lane);
  } else {
    qr_stage<FT, !MG>(M, ld, n, m, m + p, tau1, warp, lane);
    if (a.stamps && pid == 0 && tid == 0) a.stamps[30] = globaltimer_ns();  // debug: QR stage done
    rq_stage<FT>(M, ld, 0, n, m, p, tau2, scal, tid, warp, lane);
    if (a.stamps && pid == 0 && tid == 0) a.stamps[31] = globaltimer_ns();  // debug: RQ stage done
  }
  __syncthreads();
  lap(0);

  // ---------------- initial solve at u_f ---------------------------------------
  if (KIND == KIND_LSE) {
    const int k = n - p;
    const int kz = m < n ? m : n;
    FT* bf = WF(0);
    FT* y2 = WF(1);
    FT* c = WF(2);
    FT* rhs = WF(3);
    FT* y = WF(4);
    FT* rf = WF(5);
    for (int i = tid; i < m; i += NT) {
      bf[i] = FT(rinit[i]);
      c[i] = bf[i];
    }
    for (int i = tid; i < p; i += NT) y2[i] = FT(rinit[m + i]);
    __syncthreads();
    if (warp == 0) {  // R y2 = d
      if (!trsv_n<FT, FT>(M, ld, m, n - p, p, y2, lane, &iflag[1]) && lane == 0) iflag[0] = 3;
    } else if (warp == 1) {  // c = Z^T b
      qrf_apply<FT, FT>(M, ld, tau1, kz, m, c, true, lane);
    }
    __syncthreads();
    if (iflag[0]) goto finish;
    // rhs = c1 - T12 y2
    gemv_n<FT, FT>(M, ld, 0, k, k, p, y2, rhs, NoMask{}, tid, NT);
    __syncthreads();
    for (int i = tid; i < k; i += NT) rhs[i] = c[i] - rhs[i];
    __syncthreads();
    if (warp == 0) {
      if (!trsv_n<FT, FT>(M, ld, 0, 0, k, rhs, lane, &iflag[1]) && lane == 0) iflag[0] = 3;
      __syncwarp();
      for (int i = lane; i < k; i += 32) y[i] = rhs[i];
      for (int i = lane; i < p; i += 32) y[k + i] = y2[i];
      __syncwarp();
      rqf_apply<FT, FT>(M, ld, tau2, p, m, 0, n - p, y, true, lane);  // x = Q^T [y1; y2]
    }
    __syncthreads();
    if (iflag[0]) goto finish;
    // r_f = b_f - A_f x_f, A_f = fl32(A / s_A) re-read from HBM
    for (int i = tid; i < m; i += NT) {
      FT acc = FT(0);
      for (int j = 0; j < n; ++j) acc += y[j] * FT(sval(i, j));
      rf[i] = bf[i] - acc;
    }
    for (int j = tid; j < n; j += NT) su[j] = double(y[j]);
    __syncthreads();
    for (int i = tid; i < m; i += NT) sw[i] = double(rf[i]);
    __syncthreads();
    // solve_v: g = A^T r at u_r (lse.hpp:156-173)
    for (int j = warp; j < n; j += NW) {
      if (EXT) {
        dd acc{0.0, 0.0};
        for (int i = lane; i < m; i += 32) dd_fma(acc, sval(i, j), sw[i]);
        acc = warp_dd_sum(acc);
        if (lane == 0) cout[j] = acc.s + acc.c;
      } else {
        double acc = 0.0;
        for (int i = lane; i < m; i += 32) acc = fma(sval(i, j), sw[i], acc);
        acc = warp_sum(acc);
        if (lane == 0) cout[j] = acc;
      }
    }
    __syncthreads();
    {
      double mx[1] = {0.0};
      if (LOWF)
        for (int j = tid; j < n; j += NT) mx[0] = nanskip_max(mx[0], fabs(cout[j]));
      block_max(mx, red, scal + S_RED0);
    }
    const double sg = LOWF ? (scal[S_RED0] == 0.0 ? 1.0 : scal[S_RED0]) : 1.0;
    FT* gf = WF(6);
    for (int j = tid; j < n; j += NT) gf[j] = FT(cout[j] / sg);
    __syncthreads();
    if (warp == 0) {
      rqf_apply<FT, FT>(M, ld, tau2, p, m, 0, n - p, gf, false, lane);  // Q g
      if (!trsv_t<FT, FT>(M, ld, m, n - p, p, gf + (n - p), lane, &iflag[1]) && lane == 0)
        iflag[0] = 3;
    }
    __syncthreads();
    if (iflag[0]) goto finish;
    for (int i = tid; i < p; i += NT) sw[m + i] = sg * double(gf[n - p + i]);
    __syncthreads();
  } else {
    const int kk = n < p ? n : p;
    const int kp = p - n + m;  // column split of T
    FT* c = WF(0);
    FT* rhs = WF(1);
    FT* yv = WF(2);
    FT* g = WF(3);
    FT* zq = WF(4);
    for (int i = tid; i < n; i += NT) c[i] = FT(rinit[i]);
    __syncthreads();
    if (warp == 0) {
      qrf_apply<FT, FT>(M, ld, tau1, m, n, c, true, lane);  // c = Q^T d
      if (!trsv_n<FT, FT>(M, ld, m, m + kp, n - m, c + m, lane, &iflag[1]) && lane == 0)
        iflag[0] = 3;  // T22 s2 = c2
    }
    __syncthreads();
    if (iflag[0]) goto finish;
    gemv_n<FT, FT>(M, ld, 0, m, m + kp, n - m, c + m, rhs, NoMask{}, tid, NT);
    __syncthreads();
    for (int i = tid; i < m; i += NT) rhs[i] = c[i] - rhs[i];
    __syncthreads();
    if (warp == 0) {
      if (!trsv_n<FT, FT>(M, ld, 0, 0, m, rhs, lane, &iflag[1]) && lane == 0) iflag[0] = 3;
    } else if (warp == 1) {
      for (int i = lane; i < p; i += 32) yv[i] = i < kp ? FT(0) : c[m + (i - kp)];
      __syncwarp();
      rqf_apply<FT, FT>(M, ld, tau2, kk, n - kk, m, p - kk, yv, true, lane);  // y = Z^T s
    }
    __syncthreads();
    if (iflag[0]) goto finish;
    if (warp == 0) {  // init_z: g = Z y; T22^T v = g2; z = Q [0; v]
      for (int i = lane; i < p; i += 32) g[i] = yv[i];
      __syncwarp();
      rqf_apply<FT, FT>(M, ld, tau2, kk, n - kk, m, p - kk, g, false, lane);
      if (!trsv_t<FT, FT>(M, ld, m, m + kp, n - m, g + kp, lane, &iflag[1]) && lane == 0)
        iflag[0] = 3;
      __syncwarp();
      for (int i = lane; i < n; i += 32) zq[i] = i < m ? FT(0) : g[kp + (i - m)];
      __syncwarp();
      qrf_apply<FT, FT>(M, ld, tau1, m, n, zq, false, lane);
    }
    __syncthreads();
    if (iflag[0]) goto finish;
    for (int j = tid; j < m; j += NT) su[j] = double(rhs[j]);
    for (int j = tid; j < p; j += NT) su[m + j] = double(yv[j]);
    for (int i = tid; i < n; i += NT) sw[i] = double(zq[i]);
    __syncthreads();
  }
  lap(1);

  // ---------------- refinement loop (lse.hpp:377-421 / gls.hpp:336-380) -------
  {
    const double tol = a.tol;
    const double sA = scal[S_SA], sB = scal[S_SB], c1 = scal[S_CB], c2 = scal[S_CD];
    const double nA = scal[S_NA], nB = scal[S_NBF];
    const double nb = scal[S_NB], nd = scal[S_ND];
    double best = INFINITY;  // divergence detector (thread 0)
    int status = 1;          // max_iterations
    int64_t pass = 0;
    double* hist = a.hist ? a.hist + pid * a.maxit * 3 : nullptr;
    for (pass = 1; pass <= a.maxit; ++pass) {
      // ---- residual (u_r): one fused sweep over the stacked fp64 matrix ----
      // row result  rout[i] = rinit[i] - sum_j M_ij u_j
      // col result  cout[j] = cinit[j] + sum_i M_ij w_i
      // LSE: u = x, w = [-r; v], rinit = [b - r; d], cinit = 0
      // GLS: u = [x; y], w = z, rinit = d, cinit = [0; -y]
      for (int j = tid; j < C; j += NT) {
        const double ci = (KIND == KIND_GLS && j >= m) ? -su[j] : 0.0;
        cacc[j] = ci;
        if (EXT) caccc[j] = 0.0;
      }
      for (int i = tid; i < R; i += NT) {
        if (KIND == KIND_LSE && i < m) {
          if (EXT) two_sum(rinit[i], -sw[i], rout[i], rinitc[i]);
          else rout[i] = rinit[i] - sw[i];
        } else {
          rout[i] = rinit[i];
          if (EXT) rinitc[i] = 0.0;
        }
      }
      __syncthreads();
      for (int rc = 0; rc < R; rc += CH) {
        double racc[RPL];
        dd raccd[RPL];
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          racc[q] = 0.0;
          raccd[q] = dd{0.0, 0.0};
        }
        double wv[RPL];
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          const int i = rc + lane + 32 * q;
          double w = 0.0;
          if (i < R) w = (KIND == KIND_LSE && i < m) ? -sw[i] : sw[i];
          wv[q] = w;
        }
        for (int j = warp; j < C; j += NW) {
          const double uj = su[j];
          double av[RPL];
#pragma unroll
          for (int q = 0; q < RPL; ++q) {
            const int i = rc + lane + 32 * q;
            av[q] = i < R ? sval(i, j) : 0.0;
          }
          if (EXT) {
            dd cs{0.0, 0.0};
#pragma unroll
            for (int q = 0; q < RPL; ++q) {
              dd_fma(raccd[q], -av[q], uj);
              dd_fma(cs, av[q], wv[q]);
            }
            cs = warp_dd_sum(cs);
            if (lane == 0) {
              dd t{cacc[j], caccc[j]};
              dd_merge(t, cs);
              cacc[j] = t.s;
              caccc[j] = t.c;
            }
          } else {
            double cs = 0.0;
#pragma unroll
            for (int q = 0; q < RPL; ++q) {
              racc[q] = fma(av[q], uj, racc[q]);
              cs = fma(av[q], wv[q], cs);
            }
            cs = warp_sum(cs);
            if (lane == 0) cacc[j] += cs;
          }
        }
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          if (EXT) {
            part[(warp * CH + lane + 32 * q) * 2] = raccd[q].s;
            part[(warp * CH + lane + 32 * q) * 2 + 1] = raccd[q].c;
          } else {
            part[warp * CH + lane + 32 * q] = racc[q];
          }
        }
        __syncthreads();
        for (int t = tid; t < CH; t += NT) {
          const int i = rc + t;
          if (i < R) {
            if (EXT) {
              dd s{rout[i], rinitc[i]};
              for (int w2 = 0; w2 < NW; ++w2) dd_merge(s, dd{part[(w2 * CH + t) * 2], part[(w2 * CH + t) * 2 + 1]});
              rout[i] = s.s + s.c;
            } else {
              double s = 0.0;
              for (int w2 = 0; w2 < NW; ++w2) s += part[w2 * CH + t];
              rout[i] = rout[i] - s;
            }
          }
        }
        __syncthreads();
      }
      for (int j = tid; j < C; j += NT) cout[j] = EXT ? cacc[j] + caccc[j] : cacc[j];
      __syncthreads();

      // ---- norms, history, stop test, divergence -------------------------------
      // LSE: f1 = rout[0:m], f2 = rout[m:], f3 = cout;  state r = sw[0:m], v = sw[m:], x = su
      // GLS: f1 = cout[m:], f2 = rout, f3 = cout[0:m]; state x = su[0:m], y = su[m:], z = sw
      {
        double nv[6] = {0, 0, 0, 0, 0, 0};
        double mx[1] = {0.0};
        for (int i = tid; i < R; i += NT) {
          const double f = rout[i], s = sw[i];
          mx[0] = nanskip_max(mx[0], fabs(f));
          if (KIND == KIND_LSE) {
            if (i < m) nv[0] += f * f; else nv[1] += f * f;
            if (i < m) nv[3] += s * s; else nv[4] += s * s;
          } else {
            nv[1] += f * f;
            nv[5] += s * s;
          }
        }
        for (int j = tid; j < C; j += NT) {
          const double f = cout[j], s = su[j];
          mx[0] = nanskip_max(mx[0], fabs(f));
          if (KIND == KIND_LSE) {
            nv[2] += f * f;
            nv[5] += s * s;
          } else {
            if (j < m) nv[2] += f * f; else nv[0] += f * f;
            if (j < m) nv[3] += s * s; else nv[4] += s * s;
          }
        }
        block_sum(nv, red, scal + S_RED0);
        if (LOWS) block_max(mx, red, scal + S_SIG);
      }
      if (tid == 0) {
        const double g1 = sqrt(scal[S_RED0]), g2 = sqrt(scal[S_RED0 + 1]),
                     g3 = sqrt(scal[S_RED0 + 2]);
        const double s3 = sqrt(scal[S_RED0 + 3]), s4 = sqrt(scal[S_RED0 + 4]),
                     s5 = sqrt(scal[S_RED0 + 5]);
        // LSE: s3 = ||r||, s4 = ||v||, s5 = ||x||;  GLS: s3 = ||x||, s4 = ||y||, s5 = ||z||
        double d1, d2, d3;
        if (KIND == KIND_LSE) {
          d1 = nb + s3 + nA * s5;
          d2 = nd + nB * s5;
          d3 = nA * s3 + nB * s4;
          if (hist) {
            hist[(pass - 1) * 3 + 0] = g1 * c1;
            hist[(pass - 1) * 3 + 1] = g2 * c2;
            hist[(pass - 1) * 3 + 2] = g3 * sA * c1;
          }
        } else {
          d1 = s4 + nB * s5;
          d2 = nd + nA * s3 + nB * s4;
          d3 = nA * s5;
          if (hist) {
            hist[(pass - 1) * 3 + 0] = g1 * c2 / sB;
            hist[(pass - 1) * 3 + 1] = g2 * c2;
            hist[(pass - 1) * 3 + 2] = g3 * sA * c2 / (sB * sB);
          }
        }
        int decision = 0;  // 0 continue, 1 converged, 2 diverged
        if (g1 <= tol * d1 && g2 <= tol * d2 && g3 <= tol * d3) {
          decision = 1;
        } else {
          auto ratio = [](double num, double den) {
            if (den > 0.0) return num / den;
            return num == 0.0 ? 0.0 : INFINITY;
          };
          // std::max({r1, r2, r3}) order of lse.hpp:287 / gls.hpp:261
          const double r1 = ratio(g1, d1), r2 = ratio(g2, d2), r3 = ratio(g3, d3);
          const double t12 = r1 < r2 ? r2 : r1;
          const double sm = t12 < r3 ? r3 : t12;
          if (!isfinite(sm)) decision = 2;
          else {
            if (sm < best) best = sm;
            if (sm >= 1e4 * best && best > 0.0) decision = 2;
          }
        }
        iflag[2] = decision;
      }
      __syncthreads();
      lap(2);
      if (iflag[2] == 1) {
        status = 0;
        break;
      }
      if (iflag[2] == 2) {
        status = 2;
        break;
      }

      // ---- correction at u_s --------------------------------------------------
      const double sig = LOWS ? (scal[S_SIG] == 0.0 ? 1.0 : scal[S_SIG]) : 1.0;
      if (KIND == KIND_LSE) {
        const int k = n - p, kz = m < n ? m : n;
        CT* u = WC(0);
        CT* w = WC(1);
        CT* y2 = WC(2);
        CT* q1 = WC(3);
        CT* t4 = WC(4);
        CT* y = WC(5);
        CT* dr = WC(6);
        // demote (refine.hpp:103-119): f / sigma -> u_s
        for (int j = tid; j < n; j += NT) u[j] = CT(cout[j] / sig);
        for (int i = tid; i < m; i += NT) w[i] = CT(rout[i] / sig);
        for (int i = tid; i < p; i += NT) y2[i] = CT(rout[m + i] / sig);
        __syncthreads();
        if (warp == 0) {
          rqf_apply<FT, CT>(M, ld, tau2, p, m, 0, n - p, u, false, lane);  // u = Q f3
        } else if (warp == 1) {
          qrf_apply<FT, CT>(M, ld, tau1, kz, m, w, true, lane);  // w = Z^T f1
        } else if (warp == 2) {
          if (!trsv_n<FT, CT>(M, ld, m, n - p, p, y2, lane, &iflag[1]) && lane == 0) iflag[0] = 3;
        }
        __syncthreads();
        if (iflag[0]) break;
        if (warp == 0) {
          for (int i = lane; i < k; i += 32) q1[i] = u[i];
          __syncwarp();
          if (!trsv_t<FT, CT>(M, ld, 0, 0, k, q1, lane, &iflag[1]) && lane == 0) iflag[0] = 3;
        } else {
          gemv_n<FT, CT>(M, ld, 0, k, k, p, y2, t4, NoMask{}, tid - 32, NT - 32);
          gemv_n<FT, CT>(M, ld, k, m - k, k, p, y2, t4 + k, LowerMask{}, tid - 32, NT - 32);
        }
        __syncthreads();
        if (iflag[0]) break;
        // rhs = w1 - q1 - T12 y2 -> y[0:k]; q = [q1; w2 - T22 y2] -> w; y[k:n] = y2
        for (int i = tid; i < m; i += NT) {
          if (i < k) {
            y[i] = w[i] - q1[i] - t4[i];
            w[i] = q1[i];
          } else {
            w[i] = w[i] - t4[i];
          }
          dr[i] = w[i];
        }
        for (int i = tid; i < p; i += NT) y[k + i] = y2[i];
        __syncthreads();
        if (warp == 0) {
          if (!trsv_n<FT, CT>(M, ld, 0, 0, k, y, lane, &iflag[1]) && lane == 0) iflag[0] = 3;
          __syncwarp();
          rqf_apply<FT, CT>(M, ld, tau2, p, m, 0, n - p, y, true, lane);  // dx = Q^T y
        } else if (warp == 1) {
          qrf_apply<FT, CT>(M, ld, tau1, kz, m, dr, false, lane);  // dr = Z q
        } else {
          // s = T12^T q1 + (T22^T q2 - u2)
          for (int j = tid - 64; j < p; j += NT - 64) {
            CT s1 = CT(0), s2 = CT(0);
            const FT* col = M + size_t(k + j) * ld;
            for (int i = 0; i < k; ++i) s1 += CT(col[i]) * w[i];
            for (int i = k; i < m; ++i)
              if (i <= k + j) s2 += CT(col[i]) * w[i];
            t4[j] = s1 + (s2 - u[k + j]);
          }
        }
        __syncthreads();
        if (iflag[0]) break;
        if (warp == 1) {
          if (!trsv_t<FT, CT>(M, ld, m, n - p, p, t4, lane, &iflag[1]) && lane == 0) iflag[0] = 3;
        }
        __syncthreads();
        if (iflag[0]) break;
        // promote and update (lse.hpp:404-415): r += dr, v += dv, x += dx
        int bad = 0;
        for (int i = tid; i < m; i += NT) {
          sw[i] += sig * double(dr[i]);
          bad |= !isfinite(sw[i]);
        }
        for (int i = tid; i < p; i += NT) {
          sw[m + i] += sig * double(t4[i]);
          bad |= !isfinite(sw[m + i]);
        }
        for (int j = tid; j < n; j += NT) {
          su[j] += sig * double(y[j]);
          bad |= !isfinite(su[j]);
        }
        bad = __syncthreads_or(bad);
        lap(3);
        if (bad) {
          status = 2;
          break;
        }
      } else {
        const int kk = n < p ? n : p;
        const int kp = p - n + m;
        const int nm = n - m;
        CT* u = WC(0);
        CT* w = WC(1);
        CT* h1 = WC(2);
        CT* g2 = WC(3);
        CT* t4 = WC(4);
        CT* r2 = WC(5);
        CT* g = WC(6);
        CT* r1 = WC(7);
        for (int i = tid; i < n; i += NT) u[i] = CT(rout[i] / sig);       // f2
        for (int j = tid; j < p; j += NT) w[j] = CT(cout[m + j] / sig);   // f1
        for (int j = tid; j < m; j += NT) h1[j] = CT(cout[j] / sig);      // f3
        __syncthreads();
        if (warp == 0) {
          qrf_apply<FT, CT>(M, ld, tau1, m, n, u, true, lane);  // u = Q^T f2
        } else if (warp == 1) {
          rqf_apply<FT, CT>(M, ld, tau2, kk, n - kk, m, p - kk, w, false, lane);  // w = Z f1
        } else if (warp == 2) {
          if (!trsv_t<FT, CT>(M, ld, 0, 0, m, h1, lane, &iflag[1]) && lane == 0) iflag[0] = 3;
        }
        __syncthreads();
        if (iflag[0]) break;
        if (warp == 0) {
          for (int i = lane; i < nm; i += 32) g2[i] = u[m + i];
          __syncwarp();
          if (!trsv_n<FT, CT>(M, ld, m, m + kp, nm, g2, lane, &iflag[1]) && lane == 0)
            iflag[0] = 3;
        } else {
          gemv_t<FT, CT>(M, ld, 0, m, m + kp, nm, h1, t4, NoMask{}, tid - 32, NT - 32);
          gemv_t<FT, CT>(M, ld, 0, m, m, kp, h1, t4 + nm, RqMask{n - kk, m, p - kk}, tid - 32,
                         NT - 32);
        }
        __syncthreads();
        if (iflag[0]) break;
        for (int i = tid; i < nm; i += NT) r2[i] = w[kp + i] - g2[i] - t4[i];
        for (int i = tid; i < p; i += NT) g[i] = i < kp ? w[i] - t4[nm + i] : g2[i - kp];
        __syncthreads();
        if (warp == 0) {
          if (!trsv_t<FT, CT>(M, ld, m, m + kp, nm, r2, lane, &iflag[1]) && lane == 0)
            iflag[0] = 3;
        } else if (warp == 1) {
          for (int i = lane; i < p; i += 32) t4[i] = g[i];
          __syncwarp();
          rqf_apply<FT, CT>(M, ld, tau2, kk, n - kk, m, p - kk, t4, true, lane);  // dy = Z^T g
        } else {
          // rhs1 = u1 - (T11 g1 + T12 g2)
          const RqMask mk{n - kk, m, p - kk};
          for (int i = tid - 64; i < m; i += NT - 64) {
            CT s1 = CT(0), s2 = CT(0);
            const FT* rowp = M + i + size_t(m) * ld;
            for (int t = 0; t < kp; ++t)
              if (!mk.zero(i, m + t)) s1 += CT(rowp[size_t(t) * ld]) * g[t];
            for (int t = 0; t < nm; ++t) s2 += CT(rowp[size_t(kp + t) * ld]) * g2[t];
            r1[i] = u[i] - (s1 + s2);
          }
        }
        __syncthreads();
        if (iflag[0]) break;
        if (warp == 0) {  // dz = -Q [h1; h2]
          for (int i = lane; i < n; i += 32) u[i] = i < m ? h1[i] : r2[i - m];
          __syncwarp();
          qrf_apply<FT, CT>(M, ld, tau1, m, n, u, false, lane);
        } else if (warp == 1) {
          if (!trsv_n<FT, CT>(M, ld, 0, 0, m, r1, lane, &iflag[1]) && lane == 0) iflag[0] = 3;
        }
        __syncthreads();
        if (iflag[0]) break;
        int bad = 0;
        for (int j = tid; j < m; j += NT) {
          su[j] += sig * double(r1[j]);
          bad |= !isfinite(su[j]);
        }
        for (int j = tid; j < p; j += NT) {
          su[m + j] += sig * double(t4[j]);
          bad |= !isfinite(su[m + j]);
        }
        for (int i = tid; i < n; i += NT) {
          sw[i] += sig * double(-u[i]);
          bad |= !isfinite(sw[i]);
        }
        bad = __syncthreads_or(bad);
        lap(3);
        if (bad) {
          status = 2;
          break;
        }
      }
    }
    if (pass > a.maxit) pass = a.maxit;
    if (tid == 0 && iflag[0] == 0) {
      if (a.status) a.status[pid] = status;
      if (a.iters) a.iters[pid] = pass;
    }
    // ---------------- unscale and store -------------------------------------
    if (iflag[0] == 0) {
      if (KIND == KIND_LSE) {
        const double fx = c1 / sA, fr = c1, fv = sA * c1 / sB;
        for (int j = tid; j < n; j += NT) a.x[pid * n + j] = fx * su[j];
        for (int i = tid; i < m; i += NT) a.r[pid * m + i] = fr * sw[i];
        for (int i = tid; i < p; i += NT) a.v[pid * p + i] = fv * sw[m + i];
      } else {
        const double fx = c2 / sA, fy = c2 / sB, fz = c2 / (sB * sB);
        for (int j = tid; j < m; j += NT) a.x[pid * m + j] = fx * su[j];
        for (int j = tid; j < p; j += NT) a.r[pid * p + j] = fy * su[m + j];
        for (int i = tid; i < n; i += NT) a.v[pid * n + i] = fz * sw[i];
      }
    }
    lap(5);
  }
finish:
  __syncthreads();
  if (tid == 0) {
    a.err[pid] = iflag[0];
    if (a.sing) a.sing[pid] = iflag[0] == 3 ? iflag[1] : -1;
    if (a.phases)
      for (int k = 0; k < 6; ++k) a.phases[pid * 6 + k] = ph[k];
  }
}

// ============================== host side ===================================
template <int KIND, class FT, class CT, bool EXT, bool MG>
static cudaError_t launch_mg(const TileArgs& a, cudaStream_t st) {
  const Layout L = make_layout(KIND, a.m, a.n, a.p, sizeof(FT), sizeof(CT), EXT, a.gws != nullptr);
  auto kern = tile_solve_kernel<KIND, FT, CT, EXT, MG>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(L.total));
  if (e != cudaSuccess) return e;
  kern<<<dim3(unsigned(a.batch)), dim3(NT), L.total, st>>>(a);
  return cudaGetLastError();
}

template <int KIND, class FT, class CT, bool EXT>
static cudaError_t launch_one(const TileArgs& a, cudaStream_t st) {
  return a.gws ? launch_mg<KIND, FT, CT, EXT, true>(a, st) : launch_mg<KIND, FT, CT, EXT, false>(a, st);
}

template <int KIND>
static cudaError_t launch_kind(const TileArgs& a, cudaStream_t st) {
  const bool ext = a.u_r == 2;
  if (a.u_f == 0 && a.u_s == 0)
    return ext ? launch_one<KIND, float, float, true>(a, st)
               : launch_one<KIND, float, float, false>(a, st);
  if (a.u_f == 0)
    return ext ? launch_one<KIND, float, double, true>(a, st)
               : launch_one<KIND, float, double, false>(a, st);
  return ext ? launch_one<KIND, double, double, true>(a, st)
             : launch_one<KIND, double, double, false>(a, st);
}

cudaError_t launch_tile_solver(const TileArgs& a, cudaStream_t st) {
  if (a.batch <= 0) return cudaSuccess;
  return a.kind == KIND_LSE ? launch_kind<KIND_LSE>(a, st) : launch_kind<KIND_GLS>(a, st);
}

size_t tile_smem_bytes(int kind, int64_t m, int64_t n, int64_t p, int u_f, int u_s, int u_r,
                       bool m_global) {
  const int fsz = u_f == 0 ? 4 : 8, csz = u_s == 0 ? 4 : 8;
  const Layout L = make_layout(kind, m, n, p, fsz, csz, u_r == 2, m_global);
  return L.total + kStaticSmem;
}

size_t tile_gws_bytes(int kind, int64_t m, int64_t n, int64_t p, int u_f) {
  const int fsz = u_f == 0 ? 4 : 8;
  const Layout L = make_layout(kind, m, n, p, fsz, fsz, false, true);
  return size_t(L.ld) * L.C * fsz;
}

size_t device_smem_limit() {
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return 0;
  return size_t(v);
}

}  // namespace mlsb
