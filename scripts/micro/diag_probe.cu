#include <cstdio>
#include "../../paper_2406_16499_b200/csrc/large_kernels.cuh"
using namespace mlsb::lg;
namespace mlsb { namespace lg {
template <class FT, class CT>
__global__ void __launch_bounds__(TRB) k_probe128(const FT* M, int64_t ld, int64_t r0, int64_t c0,
                                                      int i0, int bs, bool herm, CT* x, long long* pr) {
  long long t0 = clock64();
  extern __shared__ __align__(16) unsigned char trsm_[];
  FT* U = reinterpret_cast<FT*>(trsm_);  // U[i + j (TRB + 1)] = M[r0+i0+i, c0+i0+j], j >= i
  CT* xs = reinterpret_cast<CT*>(U + TRB * (TRB + 1));
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  constexpr int LU = TRB + 1;
  {
    // unconditional loads (clamped addresses), 16 in flight per batch
    const FT* mp = M + (r0 + i0 + tid) + (c0 + i0) * ld;
#pragma unroll
    for (int j0 = 0; j0 < TRB; j0 += 32) {
      FT t[32];
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) {
        t[jj] = (tid <= j0 + jj && j0 + jj < bs) ? *mp : FT(0);
        mp += ld;
      }
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) U[tid + (j0 + jj) * LU] = t[jj];
    }
  }
  if (tid < bs) xs[tid] = x[i0 + tid];
  __syncthreads();
  if (threadIdx.x == 0) pr[0] = clock64() - t0;
  const int nsb = (bs + 31) / 32;
  for (int t = 0; t < nsb; ++t) {
    const int sb = herm ? t : nsb - 1 - t;
    const int s0 = sb * 32, sbs = min(32, bs - s0);
    if (w == 0) {
      // lane l owns row l of the sub-block: its off-diagonal entries, its
      // pivot and reciprocal; all loads branch-free from clamped addresses
      const int lr = min(l, sbs - 1);
      const bool lin = l < sbs;
      CT u[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const FT val = !herm ? U[(s0 + lr) + (s0 + j) * LU] : U[(s0 + j) + (s0 + lr) * LU];
        const bool nz = lin && j < sbs && (!herm ? l < j : j < l);
        u[j] = nz ? (herm ? conj_(widen_to<CT>(val)) : widen_to<CT>(val)) : zero<CT>();
      }
      const CT pd = widen_to<CT>(U[(s0 + lr) + (s0 + lr) * LU]);
      const CT pv = lin ? (herm ? conj_(pd) : pd) : one<CT>();
      const CT rp = recip(pv);
      CT xi = lin ? xs[s0 + l] : zero<CT>();
      // chain: lane j's quotient broadcast, every lane updates its row
      if (!herm) {
#pragma unroll
        for (int jj = 31; jj >= 0; --jj) {
          const CT xj = shfl_idx(qdiv(xi, pv, rp), jj);
          if (l == jj) xi = xj;
          xi = xi - u[jj] * xj;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const CT xj = shfl_idx(qdiv(xi, pv, rp), j);
          if (l == j) xi = xj;
          xi = xi - u[j] * xj;
        }
      }
      if (l < sbs) xs[s0 + l] = xi;
      if (l == 0) pr[1 + 2 * t] = clock64() - t0;
    }
    __syncthreads();
    // the block's remaining rows: !herm rows r < s0 ; herm rows r >= s0 + sbs
    const int r = tid;
    if (!herm ? (r < s0) : (r >= s0 + sbs && r < bs)) {
      CT acc = zero<CT>();
      for (int q = 0; q < sbs; ++q) {
        const CT uv = !herm ? widen_to<CT>(U[r + (s0 + q) * LU]) : conj_(widen_to<CT>(U[(s0 + q) + r * LU]));
        mac(acc, uv, xs[s0 + q]);
      }
      xs[r] = xs[r] - acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) pr[2 + 2 * t] = clock64() - t0;
  }
  if (tid < bs) x[i0 + tid] = xs[tid];
}

}}
int main() {
  const int n = 1024; float *M, *x; long long* pr;
  cudaMalloc(&M, 4 * n * n); cudaMalloc(&x, 4 * n); cudaMalloc(&pr, 8 * 16);
  cudaMemset(M, 0, 4 * n * n); cudaMemset(x, 0, 4 * n);
  float one = 1.f; for (int i = 0; i < n; ++i) cudaMemcpy(M + i + size_t(i) * n, &one, 4, cudaMemcpyHostToDevice);
  const size_t sm = sizeof(float) * TRB * (TRB + 1) + sizeof(float) * TRB;
  cudaFuncSetAttribute(k_probe128<float, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
  for (int it = 0; it < 3; ++it) k_probe128<float, float><<<1, TRB, sm>>>(M, n, 0, 0, 0, 128, false, x, pr);
  cudaDeviceSynchronize();
  long long h[16]; cudaMemcpy(h, pr, 8 * 16, cudaMemcpyDeviceToHost);
  printf("load %lld | ", h[0]);
  for (int t = 0; t < 4; ++t) printf("chain%d %lld upd%d %lld | ", t, h[1 + 2 * t], t, h[2 + 2 * t]);
  printf("\n");
  return 0;
}
