// Register-tiled SIMT GEMM for the compact-WY trailing updates of the
// blocked GRQ/GQR (the one dense contraction of the path, at u_f):
//     C = alpha * op(A) * op(B) + beta * C,   op in {N, H (conjugate transpose)}
// column-major operands with arbitrary leading dimensions.  binary32 runs on
// the FFMA pipe (no TF32/BF16 substitution: u_f must stay binary32); complex64
// uses the 4-real-FMA form (no 3M: it changes the rounding).  Split-K writes
// per-split partial products that a second kernel sums in split order, so the
// result is bitwise deterministic.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "large_common.cuh"
#include "large_internal.h"

namespace mlsb {
namespace lg {

template <class T> struct Cfg;
template <> struct Cfg<float> {
  static constexpr int BM = 128, BN = 128, BK = 8, TM = 8, TN = 8;
};
template <> struct Cfg<cf> {
  static constexpr int BM = 64, BN = 64, BK = 8, TM = 4, TN = 4;
};

template <class T, bool HA, bool HB>
__global__ void __launch_bounds__(256) gemm_kernel(int M, int N, int K, T alpha,
                                                   const T* __restrict__ A, int64_t lda,
                                                   const T* __restrict__ B, int64_t ldb, T beta,
                                                   T* __restrict__ C, int64_t ldc, int kchunk,
                                                   int64_t split_stride) {
  using CF = Cfg<T>;
  constexpr int BM = CF::BM, BN = CF::BN, BK = CF::BK, TM = CF::TM, TN = CF::TN;
  constexpr int PAD = 4;
  constexpr int LA = BM * BK / 256, LB = BN * BK / 256;  // elements per thread per tile
  __shared__ __align__(16) T As[2][BK][BM + PAD];
  __shared__ __align__(16) T Bs[2][BK][BN + PAD];

  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int i0 = blockIdx.x * BM, j0 = blockIdx.y * BN;
  const int kbeg = blockIdx.z * kchunk;
  const int kend = min(K, kbeg + kchunk);
  C += int64_t(blockIdx.z) * split_stride;

  T ra[LA], rb[LB];
  auto load_tiles = [&](int k0) {
#pragma unroll
    for (int e = 0; e < LA; ++e) {
      const int idx = tid + 256 * e;
      int i, k;
      if (!HA) {  // op(A)(i,k) = A[i + k lda], coalesced along i
        i = idx % BM;
        k = idx / BM;
      } else {  // op(A)(i,k) = conj(A[k + i lda]), coalesced along k
        k = idx % BK;
        i = idx / BK;
      }
      const int gi = i0 + i, gk = k0 + k;
      T v = zero<T>();
      if (gi < M && gk < kend) v = HA ? conj_(A[gk + int64_t(gi) * lda]) : A[gi + int64_t(gk) * lda];
      ra[e] = v;
    }
#pragma unroll
    for (int e = 0; e < LB; ++e) {
      const int idx = tid + 256 * e;
      int j, k;
      if (!HB) {  // op(B)(k,j) = B[k + j ldb], coalesced along k
        k = idx % BK;
        j = idx / BK;
      } else {  // op(B)(k,j) = conj(B[j + k ldb]), coalesced along j
        j = idx % BN;
        k = idx / BN;
      }
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
      for (int a = 0; a < TM / 2; ++a) {
        af[a] = As[buf][kk][ty * (TM / 2) + a];
        af[a + TM / 2] = As[buf][kk][BM / 2 + ty * (TM / 2) + a];
      }
#pragma unroll
      for (int b = 0; b < TN / 2; ++b) {
        bf[b] = Bs[buf][kk][tx * (TN / 2) + b];
        bf[b + TN / 2] = Bs[buf][kk][BN / 2 + tx * (TN / 2) + b];
      }
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b) mac(acc[a][b], af[a], bf[b]);
    }
    if (more) store_tiles(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  // epilogue
#pragma unroll
  for (int a = 0; a < TM; ++a) {
    const int gi = i0 + (a < TM / 2 ? ty * (TM / 2) + a : BM / 2 + ty * (TM / 2) + a - TM / 2);
    if (gi >= M) continue;
#pragma unroll
    for (int b = 0; b < TN; ++b) {
      const int gj = j0 + (b < TN / 2 ? tx * (TN / 2) + b : BN / 2 + tx * (TN / 2) + b - TN / 2);
      if (gj >= N) continue;
      T* cp = C + gi + int64_t(gj) * ldc;
      T v = alpha * acc[a][b];
      if (beta != zero<T>()) v = v + beta * (*cp);
      *cp = v;
    }
  }
}

// C[i + j ldc] = alpha_red * sum_z part[z][i + j M] + beta * C   (fixed split order)
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

template <class T>
cudaError_t gemm_t(bool ha, bool hb, int M, int N, int K, T alpha, const T* A, int64_t lda,
                   const T* B, int64_t ldb, T beta, T* C, int64_t ldc, T* work, size_t work_elems,
                   cudaStream_t st) {
  using CF = Cfg<T>;
  if (M <= 0 || N <= 0) return cudaSuccess;
  const int gm = (M + CF::BM - 1) / CF::BM, gn = (N + CF::BN - 1) / CF::BN;
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
  kchunk = (kchunk + CF::BK - 1) / CF::BK * CF::BK;
  dim3 grid(gm, gn, splits);
  T* out = splits == 1 ? C : work;
  const int64_t ldo = splits == 1 ? ldc : M;
  const int64_t sstr = splits == 1 ? 0 : int64_t(M) * N;
  if (!ha && !hb)
    gemm_kernel<T, false, false><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, out, ldo, kchunk, sstr);
  else if (ha && !hb)
    gemm_kernel<T, true, false><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, out, ldo, kchunk, sstr);
  else if (!ha && hb)
    gemm_kernel<T, false, true><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, out, ldo, kchunk, sstr);
  else
    gemm_kernel<T, true, true><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, out, ldo, kchunk, sstr);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || splits == 1) return e;
  const int64_t total = int64_t(M) * N;
  const int blocks = int(std::min<int64_t>((total + 255) / 256, 148 * 8));
  splitk_reduce<T><<<blocks, 256, 0, st>>>(M, N, splits, work, total, zero<T>(), C, ldc);
  return cudaGetLastError();
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
