#include <cstdio>
#include "../../paper_2406_16499_b200/csrc/large_kernels.cuh"
using namespace mlsb::lg;
__global__ void __launch_bounds__(256) empty256(const float* V, int64_t ldv, int L, int nbk, const float* x, int rpc, float* yp) {
  if (threadIdx.x == 999) yp[0] = V[0];
}
int main() {
  const int L = 8192, nbk = 128;
  float *V, *x, *yp;
  cudaMalloc(&V, sizeof(float) * L * nbk); cudaMalloc(&x, sizeof(float) * L); cudaMalloc(&yp, sizeof(float) * (WYB * 256));
  cudaMemset(V, 0, sizeof(float) * L * nbk); cudaMemset(x, 0, 4 * L);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    for (int r = 0; r < 3; ++r) launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 64; ++r) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float a; cudaEventElapsedTime(&a, e0, e1);
    printf("%-40s %.2f us\n", name, 1e3 * a / 64);
  };
  for (int g : {1, 8, 64, 148, 296}) {
    char nm[64]; snprintf(nm, 64, "empty256 grid %d", g);
    run(nm, [&] { empty256<<<g, 256>>>(V, L, L, nbk, x, WYD, yp); });
    snprintf(nm, 64, "k_wy_dot grid %d (rows %d)", g, g * WYD);
    run(nm, [&] { k_wy_dot<float, float><<<g, KT>>>(V, L, std::min(L, g * WYD), nbk, x, WYD, yp); });
  }
  // same, inside a CUDA graph of 64 launches
  cudaStream_t s; cudaStreamCreate(&s);
  cudaGraph_t gr; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int r = 0; r < 64; ++r) k_wy_dot<float, float><<<64, KT, 0, s>>>(V, L, L, nbk, x, WYD, yp);
  cudaStreamEndCapture(s, &gr); cudaGraphInstantiate(&ge, gr, 0);
  cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
  cudaEventRecord(e0, s); cudaGraphLaunch(ge, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
  float a; cudaEventElapsedTime(&a, e0, e1);
  printf("k_wy_dot grid 64 in a graph: %.2f us\n", 1e3 * a / 64);
  return 0;
}
