// microbenchmark: FFMA vs FFMA2 issue throughput on one SM and full chip
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void burn(float* out, int iters, float s) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  if (MODE == 0) {
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], s, 0.5f);
  } else {
    float2* b = reinterpret_cast<float2*>(a);
    const float2 ss = make_float2(s, s), h = make_float2(0.5f, 0.5f);
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) b[i] = __ffma2_rn(b[i], ss, h);
  }
  float t = 0;
  for (int i = 0; i < 16; ++i) t += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
  float* o;
  cudaMalloc(&o, 148 * 8 * 512 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int mode = 0; mode < 2; ++mode)
    for (int blocks : {1, 148 * 4}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) burn<0><<<blocks, 512>>>(o, iters, 0.999f);
        else burn<1><<<blocks, 512>>>(o, iters, 0.999f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 16 * iters * 512.0 * blocks;
        if (rep) printf("mode %s blocks %d: %.3f ms, %.1f TFLOP/s, %.2f flop/clk/SM-eq\n", mode ? "FFMA2" : "FFMA ", blocks, ms, flops / ms / 1e9, flops / (ms * 1e-3) / 1.965e9 / (blocks < 148 ? 1 : 148));
      }
    }
  return 0;
}
