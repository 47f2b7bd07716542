// Register-tiled SIMT GEMM for the compact-WY trailing updates of the
// blocked GRQ/GQR (the one dense contraction of the path, at u_f):
//     C = alpha * op(A) * op(B) + beta * C,   op in {N, H (conjugate transpose)}
// column-major operands with arbitrary leading dimensions.  binary32 runs on
// the FFMA pipe (no TF32/BF16 substitution: u_f must stay binary32); complex64
// uses the 4-real-FMA form (no 3M: it changes the rounding).
//
// The WY products are skinny (one dimension = 32 reflectors), so the CTA tile
// is chosen per call: 128x128 square, 256x32 tall (W = M V) or 32x256 wide
// (W = V^H C); 256 threads, thread rows interleaved by the row-thread count so
// a warp touches consecutive rows of C (coalesced epilogue).  Split-K writes
// per-split partial products that a second kernel sums in split order, so the
// result is bitwise deterministic.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "large_common.cuh"
#include "large_internal.h"
#include "../../include/mixedls_b200_tools.h"

namespace mlsb {
namespace lg {

template <int BM_, int BN_, int TM_, int TN_>
struct Tile {
  static constexpr int BM = BM_, BN = BN_, TM = TM_, TN = TN_, BK = 8;
  static constexpr int RT = BM / TM, CTN = BN / TN;  // thread grid
  static_assert(RT * CTN == 256, "256 threads");
};

template <class T, class TL, bool HA, bool HB>
__device__ __forceinline__ void gemm_tile_body(int M, int N, int K, T alpha, const T* __restrict__ A, int64_t lda,
                                               const T* __restrict__ B, int64_t ldb, T beta, T* __restrict__ C,
                                               int64_t ldc, int kchunk, int64_t split_stride, int bx, int by,
                                               int bz) {
  constexpr int BM = TL::BM, BN = TL::BN, BK = TL::BK, TM = TL::TM, TN = TL::TN, RT = TL::RT;
  constexpr int PAD = 4;
  constexpr int LA = BM * BK / 256, LB = BN * BK / 256;  // elements per thread per tile
  __shared__ __align__(16) T As[2][BK][BM + PAD];
  __shared__ __align__(16) T Bs[2][BK][BN + PAD];

  const int tid = threadIdx.x, tr = tid % RT, tc = tid / RT;
  const int i0 = bx * BM, j0 = by * BN;
  const int kbeg = bz * kchunk;
  const int kend = min(K, kbeg + kchunk);
  C += int64_t(bz) * split_stride;

  T ra[LA], rb[LB];
  auto load_tiles = [&](int k0) {
#pragma unroll
    for (int e = 0; e < LA; ++e) {
      const int idx = tid + 256 * e;
      const int i = !HA ? idx % BM : idx / BK, k = !HA ? idx / BM : idx % BK;
      const int gi = i0 + i, gk = k0 + k;
      T v = zero<T>();
      if (gi < M && gk < kend) v = HA ? conj_(A[gk + int64_t(gi) * lda]) : A[gi + int64_t(gk) * lda];
      ra[e] = v;
    }
#pragma unroll
    for (int e = 0; e < LB; ++e) {
      const int idx = tid + 256 * e;
      const int j = !HB ? idx / BK : idx % BN, k = !HB ? idx % BK : idx / BN;
      const int gj = j0 + j, gk = k0 + k;
      T v = zero<T>();
      if (gj < N && gk < kend) v = HB ? conj_(B[gj + int64_t(gk) * ldb]) : B[gk + int64_t(gj) * ldb];
      rb[e] = v;
    }
  };
  auto store_tiles = [&](int buf) {
#pragma unroll
    for (int e = 0; e < LA; ++e) {
      const int idx = tid + 256 * e;
      const int i = !HA ? idx % BM : idx / BK, k = !HA ? idx / BM : idx % BK;
      As[buf][k][i] = ra[e];
    }
#pragma unroll
    for (int e = 0; e < LB; ++e) {
      const int idx = tid + 256 * e;
      const int j = !HB ? idx / BK : idx % BN, k = !HB ? idx % BK : idx / BN;
      Bs[buf][k][j] = rb[e];
    }
  };

  T acc[TM][TN];
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b) acc[a][b] = zero<T>();

  int buf = 0;
  if (kbeg < kend) {
    load_tiles(kbeg);
    store_tiles(0);
  }
  __syncthreads();
  for (int k0 = kbeg; k0 < kend; k0 += BK) {
    const bool more = k0 + BK < kend;
    if (more) load_tiles(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T af[TM], bf[TN];
#pragma unroll
      for (int a = 0; a < TM; ++a) af[a] = As[buf][kk][tr + RT * a];
#pragma unroll
      for (int b = 0; b < TN; ++b) bf[b] = Bs[buf][kk][tc * TN + b];
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b) mac(acc[a][b], af[a], bf[b]);
    }
    if (more) store_tiles(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  // epilogue, one column at a time: all TM loads of C issued before the stores
#pragma unroll
  for (int b = 0; b < TN; ++b) {
    const int gj = j0 + tc * TN + b;
    if (gj >= N) continue;
    T* cj = C + int64_t(gj) * ldc;
    T old[TM];
    if (beta != zero<T>()) {
#pragma unroll
      for (int a = 0; a < TM; ++a) {
        const int gi = i0 + tr + RT * a;
        old[a] = gi < M ? cj[gi] : zero<T>();
      }
    }
#pragma unroll
    for (int a = 0; a < TM; ++a) {
      const int gi = i0 + tr + RT * a;
      if (gi >= M) continue;
      T v = alpha * acc[a][b];
      if (beta != zero<T>()) v = v + beta * old[a];
      cj[gi] = v;
    }
  }
}

// persistent wrapper: CTAs walk the (gm, gn, gz) tiles with a stride, so the
// grid can be capped (g_gemm_cta_cap) to leave SMs to the look-ahead stream
template <class T, class TL, bool HA, bool HB>
__global__ void __launch_bounds__(256) gemm_kernel(int M, int N, int K, T alpha, const T* __restrict__ A,
                                                   int64_t lda, const T* __restrict__ B, int64_t ldb, T beta,
                                                   T* __restrict__ C, int64_t ldc, int kchunk, int64_t split_stride,
                                                   int gm, int gn, int gz) {
  const int ntiles = gm * gn * gz;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    gemm_tile_body<T, TL, HA, HB>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, split_stride, t % gm,
                                  (t / gm) % gn, t / (gm * gn));
    __syncthreads();
  }
}

// binary32 128x128 tile for the rank-NBO trailing updates (K = 128 or K = L):
// BK = 16, 256 threads, 8x8 outputs per thread as 2x2 sub-blocks of 4x4
// (rows tr*4 + {0..3} and 64 + tr*4 + {0..3}; columns likewise), so every
// fragment read is one LDS.128 (4 per kk for 64 FFMA) and a warp's epilogue
// covers 64 consecutive rows of two columns.  Global tiles are read as float4
// along the operand's contiguous dimension when pointer and leading dimension
// allow it (VEC), staged in registers while the previous tile is consumed,
// and transposed into the k-major shared layout on the store.
template <bool HA, bool HB, bool VEC, int BK>
__device__ __forceinline__ void sgemm128_tile(int M, int N, int K, float alpha, const float* __restrict__ A,
                                              int64_t lda, const float* __restrict__ B, int64_t ldb,
                                              float beta, float* __restrict__ C, int64_t ldc, int kchunk,
                                              int64_t split_stride, int bx, int by, int bz,
                                              float (*As)[BK][132], float (*Bs)[BK][132]) {
  constexpr int BM = 128, BN = 128;
  constexpr int KQ = BK / 4;           // float4 slots along k for the k-contiguous operands
  constexpr int NPART = BK / 16;       // staging parts per operand (2 float4 slots each)
  const int tid = threadIdx.x, tr = tid & 15, tc = tid >> 4;
  const int i0 = bx * BM, j0 = by * BN;
  const int kbeg = bz * kchunk;
  const int kend = min(K, kbeg + kchunk);
  C += int64_t(bz) * split_stride;

  // staging: 512 float4 slots per operand tile, two per thread
  float ra[8], rb[8];
  // op(A)(i,k): !HA -> A[i + k lda] (contiguous in i) ; HA -> A[k + i lda] (contiguous in k)
  auto load_a = [&](int k0, int part) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int slot = tid + 256 * (2 * part + s);
      if (!HA) {  // 4 consecutive rows i of one k
        const int i = (slot & 31) * 4, k = slot >> 5;
        const int gi = i0 + i, gk = k0 + k;
        if (VEC) {
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (gk < kend && gi < M) v = *reinterpret_cast<const float4*>(A + gi + int64_t(gk) * lda);
          ra[4 * s] = v.x, ra[4 * s + 1] = v.y, ra[4 * s + 2] = v.z, ra[4 * s + 3] = v.w;
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t)
            ra[4 * s + t] = (gk < kend && gi + t < M) ? A[gi + t + int64_t(gk) * lda] : 0.f;
        }
      } else {  // 4 consecutive k of one row i
        const int k = (slot % KQ) * 4, i = slot / KQ;
        const int gi = i0 + i, gk = k0 + k;
        if (VEC) {
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (gi < M && gk < kend) v = *reinterpret_cast<const float4*>(A + gk + int64_t(gi) * lda);
          ra[4 * s] = v.x, ra[4 * s + 1] = v.y, ra[4 * s + 2] = v.z, ra[4 * s + 3] = v.w;
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t)
            ra[4 * s + t] = (gi < M && gk + t < kend) ? A[gk + t + int64_t(gi) * lda] : 0.f;
        }
      }
    }
  };
  // op(B)(k,j): !HB -> B[k + j ldb] (contiguous in k) ; HB -> B[j + k ldb] (contiguous in j)
  auto load_b = [&](int k0, int part) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int slot = tid + 256 * (2 * part + s);
      if (HB) {
        const int j = (slot & 31) * 4, k = slot >> 5;
        const int gj = j0 + j, gk = k0 + k;
        if (VEC) {
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (gk < kend && gj < N) v = *reinterpret_cast<const float4*>(B + gj + int64_t(gk) * ldb);
          rb[4 * s] = v.x, rb[4 * s + 1] = v.y, rb[4 * s + 2] = v.z, rb[4 * s + 3] = v.w;
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t)
            rb[4 * s + t] = (gk < kend && gj + t < N) ? B[gj + t + int64_t(gk) * ldb] : 0.f;
        }
      } else {
        const int k = (slot % KQ) * 4, j = slot / KQ;
        const int gj = j0 + j, gk = k0 + k;
        if (VEC) {
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (gj < N && gk < kend) v = *reinterpret_cast<const float4*>(B + gk + int64_t(gj) * ldb);
          rb[4 * s] = v.x, rb[4 * s + 1] = v.y, rb[4 * s + 2] = v.z, rb[4 * s + 3] = v.w;
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t)
            rb[4 * s + t] = (gj < N && gk + t < kend) ? B[gk + t + int64_t(gj) * ldb] : 0.f;
        }
      }
    }
  };
  // accumulators as row pairs (rows 2a', 2a'+1 of one column): the inner
  // product is packed FFMA2 (fma.rn.f32x2: two independent binary32 FMAs per
  // instruction, the operands and rounding of the fmaf each replaces), which
  // halves the issue slots of the 64 FMAs of a kk step
  float2 acc2[4][8];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc2[a][b] = make_float2(0.f, 0.f);
#define ACC(a, b) ((((a) & 1) != 0) ? acc2[(a) >> 1][b].y : acc2[(a) >> 1][b].x)
  auto store_a = [&](int buf, int part) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int slot = tid + 256 * (2 * part + s);
      if (!HA) {
        const int i = (slot & 31) * 4, k = slot >> 5;
        *reinterpret_cast<float4*>(&As[buf][k][i]) = make_float4(ra[4 * s], ra[4 * s + 1], ra[4 * s + 2], ra[4 * s + 3]);
      } else {
        const int k = (slot % KQ) * 4, i = slot / KQ;
#pragma unroll
        for (int t = 0; t < 4; ++t) As[buf][k + t][i] = ra[4 * s + t];
      }
    }
  };
  auto store_b = [&](int buf, int part) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int slot = tid + 256 * (2 * part + s);
      if (HB) {
        const int j = (slot & 31) * 4, k = slot >> 5;
        *reinterpret_cast<float4*>(&Bs[buf][k][j]) = make_float4(rb[4 * s], rb[4 * s + 1], rb[4 * s + 2], rb[4 * s + 3]);
      } else {
        const int k = (slot % KQ) * 4, j = slot / KQ;
#pragma unroll
        for (int t = 0; t < 4; ++t) Bs[buf][k + t][j] = rb[4 * s + t];
      }
    }
  };
  // one kk step: 4 LDS.128, 64 FFMA
  auto step = [&](int buf, int kk) {
    const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][tr * 4]);
    const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + tr * 4]);
    const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tc * 4]);
    const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tc * 4]);
    const float2 ap[4] = {make_float2(a0.x, a0.y), make_float2(a0.z, a0.w), make_float2(a1.x, a1.y),
                          make_float2(a1.z, a1.w)};
    const float bf[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) acc2[a][b] = __ffma2_rn(ap[a], make_float2(bf[b], bf[b]), acc2[a][b]);
  };


  int buf = 0;
  if (kbeg < kend) {
#pragma unroll
    for (int pt = 0; pt < NPART; ++pt) {
      load_a(kbeg, pt);
      store_a(0, pt);
      load_b(kbeg, pt);
      store_b(0, pt);
    }
  }
  __syncthreads();
  // the next tile is staged a part at a time (2 float4 slots per thread per
  // window of 8 kk steps: A parts first, then B parts), so only 8 staging
  // registers are live
  for (int k0 = kbeg; k0 < kend; k0 += BK) {
    const bool more = k0 + BK < kend;
#pragma unroll
    for (int win = 0; win < 2 * NPART; ++win) {
      const bool isA = win < NPART;
      const int pt = isA ? win : win - NPART;
      if (more) {
        if (isA) load_a(k0 + BK, pt);
        else load_b(k0 + BK, pt);
      }
#pragma unroll
      for (int kk = 8 * win; kk < 8 * win + 8; ++kk) step(buf, kk);
      if (more) {
        if (isA) store_a(buf ^ 1, pt);
        else store_b(buf ^ 1, pt);
      }
    }
    __syncthreads();
    buf ^= 1;
  }
  // epilogue: column by column, 4-row groups (float4 when aligned).  In the
  // vector path the C reads of a row half are all issued before its first
  // store: C's loads and stores may alias, so interleaved they would each pay
  // a full memory latency.
  const bool cvec = VEC && ((reinterpret_cast<uintptr_t>(C) & 15) == 0) && (ldc & 3) == 0 && (i0 & 3) == 0;
  if (cvec && i0 + 128 <= M && j0 + 128 <= N) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int gi = i0 + h * 64 + tr * 4;
      float4 o[8];
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int gj = j0 + (b < 4 ? tc * 4 + b : 64 + tc * 4 + b - 4);
        o[b] = beta != 0.f ? *reinterpret_cast<const float4*>(C + int64_t(gj) * ldc + gi) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int gj = j0 + (b < 4 ? tc * 4 + b : 64 + tc * 4 + b - 4);
        float4 v = make_float4(alpha * ACC(4 * h, b), alpha * ACC(4 * h + 1, b), alpha * ACC(4 * h + 2, b),
                               alpha * ACC(4 * h + 3, b));
        if (beta != 0.f)
          v.x = fmaf(beta, o[b].x, v.x), v.y = fmaf(beta, o[b].y, v.y), v.z = fmaf(beta, o[b].z, v.z),
          v.w = fmaf(beta, o[b].w, v.w);
        *reinterpret_cast<float4*>(C + int64_t(gj) * ldc + gi) = v;
      }
    }
    return;
  }
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const int gj = j0 + (b < 4 ? tc * 4 + b : 64 + tc * 4 + b - 4);
    if (gj >= N) continue;
    float* cj = C + int64_t(gj) * ldc;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int gi = i0 + h * 64 + tr * 4;
      if (cvec && gi + 3 < M) {
        float4 v = make_float4(alpha * ACC(4 * h, b), alpha * ACC(4 * h + 1, b), alpha * ACC(4 * h + 2, b),
                               alpha * ACC(4 * h + 3, b));
        if (beta != 0.f) {
          const float4 o = *reinterpret_cast<const float4*>(cj + gi);
          v.x = fmaf(beta, o.x, v.x), v.y = fmaf(beta, o.y, v.y), v.z = fmaf(beta, o.z, v.z), v.w = fmaf(beta, o.w, v.w);
        }
        *reinterpret_cast<float4*>(cj + gi) = v;
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (gi + t >= M) continue;
          float v = alpha * ACC(4 * h + t, b);
          if (beta != 0.f) v = fmaf(beta, cj[gi + t], v);
          cj[gi + t] = v;
        }
      }
    }
  }
}
#undef ACC

// Persistent form: the grid may be smaller than the tile count (gm x gn x gz),
// each CTA walking tiles with a stride, so a trailing update can leave SMs
// free for the look-ahead stream's panel cluster and small GEMMs.
template <bool HA, bool HB, bool VEC, int BK>
__global__ void __launch_bounds__(256, 2) sgemm128(int M, int N, int K, float alpha,
                                                   const float* __restrict__ A, int64_t lda,
                                                   const float* __restrict__ B, int64_t ldb, float beta,
                                                   float* __restrict__ C, int64_t ldc, int kchunk,
                                                   int64_t split_stride, int gm, int gn, int gz) {
  extern __shared__ __align__(16) unsigned char gsm_[];
  float(*As)[BK][132] = reinterpret_cast<float(*)[BK][132]>(gsm_);
  float(*Bs)[BK][132] = reinterpret_cast<float(*)[BK][132]>(gsm_ + sizeof(float) * 2 * BK * 132);
  const int ntiles = gm * gn * gz;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int bx = t % gm, by = (t / gm) % gn, bz = t / (gm * gn);
    sgemm128_tile<HA, HB, VEC, BK>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, split_stride, bx, by,
                                   bz, As, Bs);
    __syncthreads();
  }
}

// C[i + j ldc] = sum_z part[z][i + j M] + beta * C   (fixed split order)
template <class T>
__global__ void splitk_reduce(int M, int N, int splits, const T* __restrict__ part, int64_t stride,
                              T beta, T* __restrict__ C, int64_t ldc) {
  const int64_t total = int64_t(M) * N;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(e % M), j = int(e / M);
    T s = part[e];
    for (int z = 1; z < splits; ++z) s = s + part[e + z * stride];
    T* cp = C + i + int64_t(j) * ldc;
    *cp = beta != zero<T>() ? s + beta * (*cp) : s;
  }
}

static thread_local int g_gemm_cta_cap = 0;  // cap on resident CTAs of the trailing GEMMs (0 = none)
void set_gemm_cta_cap(int cap) { g_gemm_cta_cap = cap; }

template <class T, class TL>
static cudaError_t launch(bool ha, bool hb, dim3 tiles, int M, int N, int K, T alpha, const T* A,
                          int64_t lda, const T* B, int64_t ldb, T beta, T* C, int64_t ldc,
                          int kchunk, int64_t sstr, cudaStream_t st) {
  const int gm = int(tiles.x), gn = int(tiles.y), gz = int(tiles.z), nt = gm * gn * gz;
  const int grid = g_gemm_cta_cap > 0 ? std::min(nt, g_gemm_cta_cap) : nt;
  if (!ha && !hb)
    gemm_kernel<T, TL, false, false><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, sstr, gm, gn, gz);
  else if (ha && !hb)
    gemm_kernel<T, TL, true, false><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, sstr, gm, gn, gz);
  else if (!ha && hb)
    gemm_kernel<T, TL, false, true><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, sstr, gm, gn, gz);
  else
    gemm_kernel<T, TL, true, true><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, sstr, gm, gn, gz);
  return cudaGetLastError();
}

template <class T> struct Tiles;
template <> struct Tiles<float> {
  using Sq = Tile<128, 128, 8, 8>;
  using Tall = Tile<256, 32, 8, 4>;
  using Wide = Tile<32, 256, 4, 8>;
};
template <> struct Tiles<double> {  // binary64 (u_f = working): FP64 FMA, 4x4 per thread
  using Sq = Tile<64, 64, 4, 4>;
  using Tall = Tile<128, 32, 4, 4>;
  using Wide = Tile<32, 128, 4, 4>;
};
template <> struct Tiles<cf> {
  using Sq = Tile<64, 64, 4, 4>;
  using Tall = Tile<128, 32, 4, 4>;
  using Wide = Tile<32, 128, 4, 4>;
};

template <class T, class TL>
static cudaError_t gemm_tile(bool ha, bool hb, int M, int N, int K, T alpha, const T* A, int64_t lda,
                             const T* B, int64_t ldb, T beta, T* C, int64_t ldc, T* work,
                             size_t work_elems, cudaStream_t st) {
  const int gm = (M + TL::BM - 1) / TL::BM, gn = (N + TL::BN - 1) / TL::BN;
  // split K when the output tiles cannot fill the machine (148 SMs); only for
  // the plain product C = op(A) op(B) (alpha = 1, beta = 0), whose partial
  // sums are then added in split order
  int splits = 1;
  if (K > 0 && work && alpha == one<T>() && beta == zero<T>()) {
    const int tiles = gm * gn;
    while (tiles * splits < 2 * 148 && splits < 64 && K / (splits * 2) >= 128 &&
           size_t(M) * N * (splits * 2) <= work_elems)
      splits *= 2;
  }
  int kchunk = K > 0 ? (K + splits - 1) / splits : 1;
  kchunk = (kchunk + TL::BK - 1) / TL::BK * TL::BK;
  dim3 grid(gm, gn, splits);
  cudaError_t e;
  if (splits == 1)
    return launch<T, TL>(ha, hb, grid, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, 0, st);
  if ((e = launch<T, TL>(ha, hb, grid, M, N, K, alpha, A, lda, B, ldb, beta, work, M, kchunk,
                         int64_t(M) * N, st)))
    return e;
  const int64_t total = int64_t(M) * N;
  const int blocks = int(std::min<int64_t>((total + 255) / 256, 148 * 8));
  splitk_reduce<T><<<blocks, 256, 0, st>>>(M, N, splits, work, total, zero<T>(), C, ldc);
  return cudaGetLastError();
}


constexpr int GBK = 32;  // k-tile of the binary32 WY GEMM (MLSB_GEMM_BK16=1: 16)
template <bool VEC, int BK>
static void launch128_bk(bool ha, bool hb, int grid, int gm, int gn, int gz, int M, int N, int K, float alpha,
                         const float* A, int64_t lda, const float* B, int64_t ldb, float beta, float* C,
                         int64_t ldc, int kchunk, int64_t sstr, cudaStream_t st) {
  constexpr size_t sm = sizeof(float) * 4 * BK * 132;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sgemm128<false, false, VEC, BK>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    cudaFuncSetAttribute(sgemm128<true, false, VEC, BK>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    cudaFuncSetAttribute(sgemm128<false, true, VEC, BK>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    cudaFuncSetAttribute(sgemm128<true, true, VEC, BK>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    attr = true;
  }
  if (!ha && !hb)
    sgemm128<false, false, VEC, BK><<<grid, 256, sm, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, sstr, gm, gn, gz);
  else if (ha && !hb)
    sgemm128<true, false, VEC, BK><<<grid, 256, sm, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, sstr, gm, gn, gz);
  else if (!ha && hb)
    sgemm128<false, true, VEC, BK><<<grid, 256, sm, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, sstr, gm, gn, gz);
  else
    sgemm128<true, true, VEC, BK><<<grid, 256, sm, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, sstr, gm, gn, gz);
}


template <bool VEC>
static void launch128(bool ha, bool hb, dim3 tiles, int M, int N, int K, float alpha, const float* A,
                      int64_t lda, const float* B, int64_t ldb, float beta, float* C, int64_t ldc,
                      int kchunk, int64_t sstr, cudaStream_t st) {
  const int nt = int(tiles.x * tiles.y * tiles.z);
  const int grid = g_gemm_cta_cap > 0 ? std::min(nt, g_gemm_cta_cap) : nt;
  const int gm = int(tiles.x), gn = int(tiles.y), gz = int(tiles.z);
  // k-tile: 32 for every operand layout since the FFMA2 inner product (the NT
  // form, the RQ trailing update, was faster at 16 before: now 0.583 vs 0.567
  // of the FP32 peak at the C3 shape; MLSB_GEMM_NT16=1 restores it)
  static const bool bk16 = getenv("MLSB_GEMM_BK16") != nullptr;
  static const bool nt16 = getenv("MLSB_GEMM_NT16") != nullptr;
  if (bk16 || (!ha && hb && nt16))
    launch128_bk<VEC, 16>(ha, hb, grid, gm, gn, gz, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, sstr, st);
  else
    launch128_bk<VEC, GBK>(ha, hb, grid, gm, gn, gz, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, sstr, st);
}

static cudaError_t sgemm_sq(bool ha, bool hb, int M, int N, int K, float alpha, const float* A, int64_t lda,
                            const float* B, int64_t ldb, float beta, float* C, int64_t ldc, float* work,
                            size_t work_elems, cudaStream_t st) {
  const int gm = (M + 127) / 128, gn = (N + 127) / 128;
  int splits = 1;
  if (K > 0 && work && alpha == 1.f && beta == 0.f) {
    const int tiles = gm * gn;
    while (tiles * splits < 2 * 148 && splits < 64 && K / (splits * 2) >= 128 &&
           size_t(M) * N * (splits * 2) <= work_elems)
      splits *= 2;
  }
  int kchunk = K > 0 ? (K + splits - 1) / splits : 1;
  kchunk = (kchunk + 31) / 32 * 32;  // a multiple of both k-tiles
  // float4 operand tiles: aligned pointers, leading dimensions and contiguous
  // extents all multiples of 4 (so no vector straddles an edge)
  const bool vec = (reinterpret_cast<uintptr_t>(A) & 15) == 0 && (lda & 3) == 0 &&
                   (reinterpret_cast<uintptr_t>(B) & 15) == 0 && (ldb & 3) == 0 &&
                   ((ha ? K : M) & 3) == 0 && ((hb ? N : K) & 3) == 0;
  dim3 grid(gm, gn, splits);
  float* Cd = splits == 1 ? C : work;
  const int64_t ldd = splits == 1 ? ldc : M, sstr = splits == 1 ? 0 : int64_t(M) * N;
  const float bd = splits == 1 ? beta : 0.f;
  if (vec) launch128<true>(ha, hb, grid, M, N, K, alpha, A, lda, B, ldb, bd, Cd, ldd, kchunk, sstr, st);
  else launch128<false>(ha, hb, grid, M, N, K, alpha, A, lda, B, ldb, bd, Cd, ldd, kchunk, sstr, st);
  cudaError_t e = cudaGetLastError();
  if (e || splits == 1) return e;
  const int64_t total = int64_t(M) * N;
  const int blocks = int(std::min<int64_t>((total + 255) / 256, 148 * 8));
  splitk_reduce<float><<<blocks, 256, 0, st>>>(M, N, splits, work, total, 0.f, C, ldc);
  return cudaGetLastError();
}

template <class T>
cudaError_t gemm_t(bool ha, bool hb, int M, int N, int K, T alpha, const T* A, int64_t lda,
                   const T* B, int64_t ldb, T beta, T* C, int64_t ldc, T* work, size_t work_elems,
                   cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if constexpr (std::is_same<T, float>::value) {
    static const bool old_tiles = getenv("MLSB_GEMM_OLD") != nullptr;  // A/B comparisons
    if (M > 64 && N > 64 && !old_tiles)
      return sgemm_sq(ha, hb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, work, work_elems, st);
  }
  if (N <= 32 && M > 32)
    return gemm_tile<T, typename Tiles<T>::Tall>(ha, hb, M, N, K, alpha, A, lda, B, ldb, beta, C,
                                                 ldc, work, work_elems, st);
  if (M <= 32 && N > 32)
    return gemm_tile<T, typename Tiles<T>::Wide>(ha, hb, M, N, K, alpha, A, lda, B, ldb, beta, C,
                                                 ldc, work, work_elems, st);
  return gemm_tile<T, typename Tiles<T>::Sq>(ha, hb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
                                             work, work_elems, st);
}

// T of an outer WY block from its NB-wide panels: P_0 P_1 ... = I - V T V^H
// with V = [V_0 V_1 ...], so the off-diagonal block column j is
//     T[0:jNB, j] = -T[0:jNB, 0:jNB] * (V_{0:j}^H V_j) * T_jj
// (the block form of xLARFT's forward recursion).  G = V^H V comes from a
// GEMM; one CTA merges the panels' T_jj (stored NB x NB, consecutive) in
// shared memory.
// one CTA of TMT threads: the merge is a chain of small triangular products
// whose outputs are independent dot products, so more threads = more of them
// in flight (round 1 ran 256 threads: ~53 us per outer block at C3)
constexpr int TMT = 1024;
template <class T>
__global__ void __launch_bounds__(TMT) k_tmerge(int nbo, const T* __restrict__ G, int ldg,
                                                const T* __restrict__ Tp, T* __restrict__ Tout,
                                                int ldt) {
  extern __shared__ __align__(16) unsigned char sm_[];
  constexpr int LDS = NBO + 1;
  T* S = reinterpret_cast<T*>(sm_);  // S[r + c LDS], upper triangular
  T* X = S + NBO * LDS;              // X[r + c NBO]
  const int tid = threadIdx.x;
  const int nblk = (nbo + NB - 1) / NB;
  // diagonal blocks: loads issued in batches of 16 from clamped addresses
  for (int e0 = tid; e0 < nbo * nbo; e0 += TMT * 16) {
    T v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = min(e0 + TMT * u, nbo * nbo - 1), r = e % nbo, c = e / nbo, br = r / NB;
      v[u] = Tp[br * NB * NB + (r - br * NB) + (c % NB) * NB];
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = e0 + TMT * u;
      if (e < nbo * nbo) {
        const int r = e % nbo, c = e / nbo;
        S[r + c * LDS] = (r / NB == c / NB) ? v[u] : zero<T>();
      }
    }
  }
  __syncthreads();
  T* GX = X + NBO * NB;  // staged block column G[0:h, c0:c0+w]
  for (int j = 1; j < nblk; ++j) {
    const int c0 = j * NB, w = min(NB, nbo - c0), h = c0;
    for (int e0 = tid; e0 < h * w; e0 += TMT * 12) {
      T v[12];
#pragma unroll
      for (int u = 0; u < 12; ++u) {
        const int e = min(e0 + TMT * u, h * w - 1);
        v[u] = G[e % h + int64_t(c0 + e / h) * ldg];
      }
#pragma unroll
      for (int u = 0; u < 12; ++u) {
        const int e = e0 + TMT * u;
        if (e < h * w) GX[e % h + (e / h) * NBO] = v[u];
      }
    }
    __syncthreads();
    for (int e = tid; e < h * w; e += TMT) {
      const int r = e % h, c = e / h;
      T acc = zero<T>();
      for (int t = 0; t <= c; ++t) mac(acc, GX[r + t * NBO], S[(c0 + t) + (c0 + c) * LDS]);
      X[r + c * NBO] = acc;
    }
    __syncthreads();
    for (int e = tid; e < h * w; e += TMT) {
      const int r = e % h, c = e / h;
      T acc = zero<T>();
      for (int t = r; t < h; ++t) mac(acc, S[r + t * LDS], X[t + c * NBO]);
      S[r + (c0 + c) * LDS] = -acc;
    }
    __syncthreads();
  }
  for (int e = tid; e < nbo * nbo; e += TMT) {
    const int r = e % nbo, c = e / nbo;
    Tout[r + int64_t(c) * ldt] = S[r + c * LDS];
  }
}

template <class T>
static cudaError_t tmerge_t(int nbo, const T* G, int ldg, const T* Tp, T* Tout, int ldt,
                            cudaStream_t st) {
  if (nbo <= 0 || nbo > NBO) return cudaErrorInvalidValue;
  const size_t sm = sizeof(T) * (size_t(NBO) * (NBO + 1) + 2 * size_t(NBO) * NB);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_tmerge<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    if (e) return e;
    attr = true;
  }
  k_tmerge<T><<<1, TMT, sm, st>>>(nbo, G, ldg, Tp, Tout, ldt);
  return cudaGetLastError();
}
cudaError_t tmerge_f32(int nbo, const float* G, int ldg, const float* Tp, float* Tout, int ldt,
                       cudaStream_t st) {
  return tmerge_t<float>(nbo, G, ldg, Tp, Tout, ldt, st);
}
cudaError_t tmerge_c64(int nbo, const cf* G, int ldg, const cf* Tp, cf* Tout, int ldt, cudaStream_t st) {
  return tmerge_t<cf>(nbo, G, ldg, Tp, Tout, ldt, st);
}
cudaError_t tmerge_f64(int nbo, const double* G, int ldg, const double* Tp, double* Tout, int ldt,
                       cudaStream_t st) {
  return tmerge_t<double>(nbo, G, ldg, Tp, Tout, ldt, st);
}

cudaError_t gemm_f32(bool ha, bool hb, int M, int N, int K, float alpha, const float* A,
                     int64_t lda, const float* B, int64_t ldb, float beta, float* C, int64_t ldc,
                     float* work, size_t work_elems, cudaStream_t st) {
  return gemm_t<float>(ha, hb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, work, work_elems, st);
}
cudaError_t gemm_f64(bool ha, bool hb, int M, int N, int K, double alpha, const double* A, int64_t lda,
                     const double* B, int64_t ldb, double beta, double* C, int64_t ldc, double* work,
                     size_t work_elems, cudaStream_t st) {
  return gemm_t<double>(ha, hb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, work, work_elems, st);
}
cudaError_t gemm_c64(bool ha, bool hb, int M, int N, int K, cf alpha, const cf* A, int64_t lda,
                     const cf* B, int64_t ldb, cf beta, cf* C, int64_t ldc, cf* work,
                     size_t work_elems, cudaStream_t st) {
  return gemm_t<cf>(ha, hb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, work, work_elems, st);
}

}  // namespace lg
}  // namespace mlsb

extern "C" int mlsb_wy_gemm_f32(int ta, int tb, int M, int N, int K, float alpha, const float* A,
                                int64_t lda, const float* B, int64_t ldb, float beta, float* C,
                                int64_t ldc, float* work, size_t work_elems, void* stream) {
  return int(mlsb::lg::gemm_f32(ta != 0, tb != 0, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, work,
                                work_elems, static_cast<cudaStream_t>(stream)));
}
