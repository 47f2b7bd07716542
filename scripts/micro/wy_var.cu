#include <cstdio>
#include "../../paper_2406_16499_b200/csrc/large_kernels.cuh"
using namespace mlsb::lg;
// variant: MODE 0 partials only; 1 + fence/atomic; 2 full (tail) ; 3 tail alone (1 CTA, pretend last)
template <int MODE>
__global__ void __launch_bounds__(KT) dotv(const float* V, int64_t ldv, int L, int nbk, const float* x, int rpc,
                                           float* ypart, const float* Tm, int ldt, unsigned* ticket, float* zout, int nparts_tail) {
  __shared__ float red[2][WYB];
  __shared__ float ys[WYB];
  __shared__ bool last;
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  if (MODE != 3) {
    const int r0 = blockIdx.x * rpc, r1 = min(L, r0 + rpc);
    float a[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = 0.f;
    for (int b = r0; b < r1; b += WYR) {
      const int ra = b + l, rb2 = b + 32 + l;
      const float x0 = ra < r1 ? x[ra] : 0.f, x1 = rb2 < r1 ? x[rb2] : 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int q = w * 16 + j;
        if (q < nbk) {
          const float* vq = V + int64_t(q) * ldv;
          if (ra < r1) a[j] = fmaf(vq[ra], x0, a[j]);
          if (rb2 < r1) a[j] = fmaf(vq[rb2], x1, a[j]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = wsum(a[j]);
    if (l == 0)
#pragma unroll
      for (int j = 0; j < 16; ++j) ypart[int64_t(blockIdx.x) * WYB + w * 16 + j] = a[j];
    if (MODE == 0) return;
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (MODE == 1) { if (last && tid == 0) *ticket = 0; return; }
    if (!last) return;
    __threadfence();
  }
  const int nparts = MODE == 3 ? nparts_tail : gridDim.x, q = tid & (WYB - 1), h = tid / WYB;
  {
    float s = 0.f;
#pragma unroll 16
    for (int c = h; c < nparts; c += 2) s += ypart[int64_t(c) * WYB + q];
    red[h][q] = s;
  }
  __syncthreads();
  if (tid < WYB) ys[tid] = red[0][tid] + red[1][tid];
  __syncthreads();
  {
    float z = 0.f;
    const int ka = h == 0 ? 0 : nbk / 2, kb = h == 0 ? nbk / 2 : nbk;
#pragma unroll 16
    for (int k = max(ka, q); k < kb; ++k) z = fmaf(Tm[q + int64_t(ldt) * k], ys[k], z);
    red[h][q] = z;
  }
  __syncthreads();
  if (tid < nbk) zout[tid] = red[0][tid] + red[1][tid];
  if (tid == 0) *ticket = 0u;
}
int main() {
  const int L = 8192, nbk = 128;
  float *V, *T, *x, *yp;
  cudaMalloc(&V, sizeof(float) * L * nbk); cudaMalloc(&T, sizeof(float) * 128 * 128);
  cudaMalloc(&x, sizeof(float) * L); cudaMalloc(&yp, sizeof(float) * (WYB * 256 + WYB + 4));
  cudaMemset(V, 0, sizeof(float) * L * nbk); cudaMemset(T, 0, 65536); cudaMemset(x, 0, 4 * L);
  cudaMemset(yp, 0, sizeof(float) * (WYB * 256 + WYB + 4));
  float* z = yp + WYB * 256; unsigned* ticket = reinterpret_cast<unsigned*>(z + WYB);
  const int rpc = WYR, ncta = L / rpc;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    for (int r = 0; r < 3; ++r) launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 64; ++r) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float a; cudaEventElapsedTime(&a, e0, e1);
    printf("%-28s %.2f us\n", name, 1e3 * a / 64);
  };
  run("partials only", [&] { dotv<0><<<ncta, KT>>>(V, L, L, nbk, x, rpc, yp, T, 128, ticket, z, 0); });
  run("+ fence/atomic", [&] { dotv<1><<<ncta, KT>>>(V, L, L, nbk, x, rpc, yp, T, 128, ticket, z, 0); });
  run("full (last-CTA tail)", [&] { dotv<2><<<ncta, KT>>>(V, L, L, nbk, x, rpc, yp, T, 128, ticket, z, 0); });
  run("tail alone (1 CTA)", [&] { dotv<3><<<1, KT>>>(V, L, L, nbk, x, rpc, yp, T, 128, ticket, z, ncta); });
  run("empty kernel", [&] { dotv<3><<<1, KT>>>(V, L, L, 0, x, rpc, yp, T, 128, ticket, z, 0); });
  run("upd", [&] { k_wy_upd<float, float><<<ncta, KT>>>(V, L, L, nbk, z, rpc, x); });
  return 0;
}
