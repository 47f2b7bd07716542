// Latency probes (1 warp / 4 warps per SM): SHFL chain, DADD chain, FFMA chain,
// 32-value transposed warp reduction.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* out, long long* t, int reps) {
  const int l = threadIdx.x & 31;
  float d[32];
  for (int k = 0; k < 32; ++k) d[k] = l * 0.01f + k;
  float s = l;
  double dd = l;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) s = __shfl_xor_sync(0xffffffffu, s, 1 + (r & 15));
  long long t1 = clock64();
  for (int r = 0; r < reps; ++r) dd = dd + dd * 1e-9;
  long long t2 = clock64();
  for (int r = 0; r < reps; ++r) s = fmaf(s, 1.0001f, 1e-5f);
  long long t3 = clock64();
  for (int r = 0; r < reps / 16; ++r) {
#pragma unroll
    for (int st = 16; st >= 1; st >>= 1) {
      const bool up = (l & st) != 0;
#pragma unroll
      for (int j = 0; j < st; ++j) {
        const float send = up ? d[j] : d[j + st];
        const float keep = up ? d[j + st] : d[j];
        d[j] = keep + __shfl_xor_sync(0xffffffffu, send, st);
      }
    }
#pragma unroll
    for (int k = 1; k < 32; ++k) d[k] = d[0] * k;
  }
  long long t4 = clock64();
  double x = l;
  for (int r = 0; r < reps; ++r) x = __shfl_xor_sync(0xffffffffu, x, 1 + (r & 15)) + 1.0;
  long long t5 = clock64();
  if (threadIdx.x == 0) {
    t[blockIdx.x * 8 + 0] = t1 - t0; t[blockIdx.x * 8 + 1] = t2 - t1; t[blockIdx.x * 8 + 2] = t3 - t2;
    t[blockIdx.x * 8 + 3] = t4 - t3; t[blockIdx.x * 8 + 4] = t5 - t4;
  }
  out[threadIdx.x] = s + d[5] + float(dd) + float(x);
}
int main() {
  float* o; long long* t; cudaMalloc(&o, 4096 * 4); cudaMalloc(&t, 64 * 8);
  const int reps = 1024;
  for (int nt : {32, 128, 512}) {
    k<<<1, nt>>>(o, t, reps); cudaDeviceSynchronize();
    k<<<1, nt>>>(o, t, reps); cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, t, 64, cudaMemcpyDeviceToHost);
    printf("threads %d: SHFL chain %.1f cyc, DADD/DFMA chain %.1f, FFMA chain %.1f, transposed-reduce32 %.1f cyc each, SHFL.f64+DADD %.1f\n",
           nt, h[0] / double(reps), h[1] / double(reps), h[2] / double(reps), h[3] / double(reps / 16),
           h[4] / double(reps));
  }
  return 0;
}
