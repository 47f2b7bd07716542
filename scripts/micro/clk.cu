#include <cstdio>
__global__ void spin(long long cyc, long long* out) {
  long long t0 = clock64();
  while (clock64() - t0 < cyc) {}
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}
__global__ void empty() {}
int main() {
  long long* o; cudaMalloc(&o, 8 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int it = 0; it < 3; ++it) {
    for (int nb : {1, 148}) {
      cudaEventRecord(a); spin<<<nb, 32>>>(2000000, o); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("spin 2e6 cycles on %d CTA(s): %.3f ms -> %.0f MHz\n", nb, ms, 2e6 / (ms * 1e3));
    }
  }
  cudaEventRecord(a);
  for (int i = 0; i < 1000; ++i) empty<<<1, 32>>>();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("empty kernel back-to-back: %.2f us\n", ms);
  cudaGraph_t g; cudaGraphExec_t ge; cudaStream_t s; cudaStreamCreate(&s);
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 1000; ++i) empty<<<1, 32, 0, s>>>();
  cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
  cudaEventRecord(a, s); cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("empty kernel in a graph: %.2f us\n", ms);
  return 0;
}
