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

#include "large_common.cuh"
#include "large_internal.h"

namespace mlsb {
namespace lg {

template <int BM_, int BN_, int TM_, int TN_>
struct Tile {
  static constexpr int BM = BM_, BN = BN_, TM = TM_, TN = TN_, BK = 8;
  static constexpr int RT = BM / TM, CTN = BN / TN;  // thread grid
  static_assert(RT * CTN == 256, "256 threads");
};

template <class T, class TL, bool HA, bool HB>
__global__ void __launch_bounds__(256) gemm_kernel(int M, int N, int K, T alpha,
                                                   const T* __restrict__ A, int64_t lda,
                                                   const T* __restrict__ B, int64_t ldb, T beta,
                                                   T* __restrict__ C, int64_t ldc, int kchunk,
                                                   int64_t split_stride) {
  constexpr int BM = TL::BM, BN = TL::BN, BK = TL::BK, TM = TL::TM, TN = TL::TN, RT = TL::RT;
  constexpr int PAD = 4;
  constexpr int LA = BM * BK / 256, LB = BN * BK / 256;  // elements per thread per tile
  __shared__ __align__(16) T As[2][BK][BM + PAD];
  __shared__ __align__(16) T Bs[2][BK][BN + PAD];

  const int tid = threadIdx.x, tr = tid % RT, tc = tid / RT;
  const int i0 = blockIdx.x * BM, j0 = blockIdx.y * BN;
  const int kbeg = blockIdx.z * kchunk;
  const int kend = min(K, kbeg + kchunk);
  C += int64_t(blockIdx.z) * split_stride;

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

template <class T, class TL>
static cudaError_t launch(bool ha, bool hb, dim3 grid, int M, int N, int K, T alpha, const T* A,
                          int64_t lda, const T* B, int64_t ldb, T beta, T* C, int64_t ldc,
                          int kchunk, int64_t sstr, cudaStream_t st) {
  if (!ha && !hb)
    gemm_kernel<T, TL, false, false><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, sstr);
  else if (ha && !hb)
    gemm_kernel<T, TL, true, false><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, sstr);
  else if (!ha && hb)
    gemm_kernel<T, TL, false, true><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, sstr);
  else
    gemm_kernel<T, TL, true, true><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, sstr);
  return cudaGetLastError();
}

template <class T> struct Tiles;
template <> struct Tiles<float> {
  using Sq = Tile<128, 128, 8, 8>;
  using Tall = Tile<256, 32, 8, 4>;
  using Wide = Tile<32, 256, 4, 8>;
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

template <class T>
cudaError_t gemm_t(bool ha, bool hb, int M, int N, int K, T alpha, const T* A, int64_t lda,
                   const T* B, int64_t ldb, T beta, T* C, int64_t ldc, T* work, size_t work_elems,
                   cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (N <= 32 && M > 32)
    return gemm_tile<T, typename Tiles<T>::Tall>(ha, hb, M, N, K, alpha, A, lda, B, ldb, beta, C,
                                                 ldc, work, work_elems, st);
  if (M <= 32 && N > 32)
    return gemm_tile<T, typename Tiles<T>::Wide>(ha, hb, M, N, K, alpha, A, lda, B, ldb, beta, C,
                                                 ldc, work, work_elems, st);
  return gemm_tile<T, typename Tiles<T>::Sq>(ha, hb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
                                             work, work_elems, st);
}

cudaError_t gemm_f32(bool ha, bool hb, int M, int N, int K, float alpha, const float* A,
                     int64_t lda, const float* B, int64_t ldb, float beta, float* C, int64_t ldc,
                     float* work, size_t work_elems, cudaStream_t st) {
  return gemm_t<float>(ha, hb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, work, work_elems, st);
}
cudaError_t gemm_c64(bool ha, bool hb, int M, int N, int K, cf alpha, const cf* A, int64_t lda,
                     const cf* B, int64_t ldb, cf beta, cf* C, int64_t ldc, cf* work,
                     size_t work_elems, cudaStream_t st) {
  return gemm_t<cf>(ha, hb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, work, work_elems, st);
}

}  // namespace lg
}  // namespace mlsb
