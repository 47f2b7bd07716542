// SIMT FMA-throughput microbenchmarks: the FP32 / FP64 roofline denominators
// the tensor-core-centric MEASURED_PEAKS.json does not carry.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mixedls_b200_tools.h"

namespace {

template <class T>
__global__ void __launch_bounds__(256) fma_burn(T* out, int iters, T seed) {
  // 8 independent chains per thread hide the 4-cycle FMA latency
  T a0 = seed + threadIdx.x, a1 = a0 + T(1), a2 = a0 + T(2), a3 = a0 + T(3);
  T a4 = a0 + T(4), a5 = a0 + T(5), a6 = a0 + T(6), a7 = a0 + T(7);
  const T b = T(0.999999), c = T(1e-7);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  const T s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == T(-1234.5)) out[blockIdx.x] = s;  // keep the chains alive
}

template <class T>
double run_peak(int device, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (device >= 0) cudaSetDevice(device);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  T* out = nullptr;
  const int blocks = sms * 8;
  if (cudaMallocAsync(&out, sizeof(T) * blocks, st) != cudaSuccess) return -1.0;
  const int iters = sizeof(T) == 4 ? 4096 : 1024;
  fma_burn<T><<<blocks, 256, 0, st>>>(out, iters, T(1));  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0, st);
    fma_burn<T><<<blocks, 256, 0, st>>>(out, iters, T(1));
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(out, st);
  cudaStreamSynchronize(st);
  if (cudaGetLastError() != cudaSuccess) return -1.0;
  const double flops = 2.0 * 8 * 16 * double(iters) * 256.0 * blocks;
  return flops / (best * 1e-3) / 1e12;
}

}  // namespace

extern "C" {
double mlsb_fp32_fma_peak_tflops(int device, void* stream) { return run_peak<float>(device, stream); }
double mlsb_fp64_fma_peak_tflops(int device, void* stream) { return run_peak<double>(device, stream); }
}
