// microbenchmark: FP32 FMA issue forms on B200 -- FFMA with an immediate
// addend, FFMA with three register operands (the GEMM / rank-1 update form),
// and the packed FFMA2 (fma.rn.f32x2) in three-register form.  Full chip,
// 4 CTAs x 512 threads per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void burn(float* out, int iters, float s, float c) {
  float a[16], b[16];
  const float sv = s + threadIdx.x * 1e-9f;  // per-thread register operand
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i, b[i] = c + i * 1e-3f;
  if (MODE == 0) {
#pragma unroll 4
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], s, 0.5f);
  } else if (MODE == 1) {
#pragma unroll 4
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fmaf(b[i], sv, a[i]);  // acc += b * s (3 registers)
  } else {
    float2* a2 = reinterpret_cast<float2*>(a);
    const float2* b2 = reinterpret_cast<const float2*>(b);
    const float2 ss = make_float2(sv, sv);
#pragma unroll 4
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) a2[i] = __ffma2_rn(b2[i], ss, a2[i]);
  }
  float t = 0;
  for (int i = 0; i < 16; ++i) t += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int MODE>
static double run(float* o, int blocks, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    burn<MODE><<<blocks, 512>>>(o, iters, 0.999f, 1e-3f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  return 2.0 * 16 * iters * 512.0 * blocks / (ms * 1e-3) / 1e12;
}
int main() {
  float* o;
  cudaMalloc(&o, 148 * 4 * 512 * 4);
  const int iters = 20000, blocks = 148 * 4;
  printf("FFMA imm-form   : %.1f TFLOP/s\n", run<0>(o, blocks, iters));
  printf("FFMA 3-register : %.1f TFLOP/s\n", run<1>(o, blocks, iters));
  printf("FFMA2 3-register: %.1f TFLOP/s\n", run<2>(o, blocks, iters));
  return 0;
}
