// Back-to-back timing of the cascade building blocks at the C3 shapes:
// one 128-wide WY block apply (k_wy_dot + k_wy_upd) and one 128-row TRSV block
// (k_trsv_diag128 + k_trsv_off).
#include <cstdio>
#include "../../paper_2406_16499_b200/csrc/large_kernels.cuh"
using namespace mlsb::lg;
int main() {
  const int L = 8192, nbk = 128;
  float *V, *T, *x, *yp, *M;
  cudaMalloc(&V, sizeof(float) * L * nbk); cudaMalloc(&T, sizeof(float) * 128 * 128);
  cudaMalloc(&x, sizeof(float) * L); cudaMalloc(&yp, sizeof(float) * (WYB * 256));
  const int n = 3072;
  cudaMalloc(&M, sizeof(float) * size_t(n) * n);
  cudaMemset(V, 0, sizeof(float) * L * nbk); cudaMemset(T, 0, 65536); cudaMemset(x, 0, 4 * L);
  cudaMemset(M, 0, sizeof(float) * size_t(n) * n);
  // unit diagonal so the solves stay finite
  float one = 1.f;
  for (int i = 0; i < n; ++i) cudaMemcpy(M + i + size_t(i) * n, &one, 4, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, int per, auto launch) {
    for (int r = 0; r < 3; ++r) launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 32; ++r) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float a; cudaEventElapsedTime(&a, e0, e1);
    printf("%-34s %.2f us\n", name, 1e3 * a / 32 / per);
  };
  const int nd = L / WYD, nu = L / WYR;
  run("apply (dot + upd)", 1, [&] {
    k_wy_dot<float, float><<<nd, KT>>>(V, L, L, nbk, x, WYD, yp);
    k_wy_upd<float, float><<<nu, KT>>>(V, L, L, nbk, yp, nd, T, 128, false, WYR, x);
  });
  run("  dot", 1, [&] { k_wy_dot<float, float><<<nd, KT>>>(V, L, L, nbk, x, WYD, yp); });
  run("  upd", 1, [&] { k_wy_upd<float, float><<<nu, KT>>>(V, L, L, nbk, yp, nd, T, 128, false, WYR, x); });
  const size_t sm = sizeof(float) * TRB * (TRB + 1) + sizeof(float) * TRB;
  cudaFuncSetAttribute(k_trsv_diag128<float, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
  run("trsv block (diag128 + off), N", 1, [&] {
    k_trsv_diag128<float, float><<<1, TRB, sm>>>(M, n, 0, 0, n - 128, 128, false, x);
    k_trsv_off<float, float><<<(n - 128 + 63) / 64, KT>>>(M, n, 0, 0, n - 128, 128, n, false, x);
  });
  run("  diag128 N", 1, [&] { k_trsv_diag128<float, float><<<1, TRB, sm>>>(M, n, 0, 0, n - 128, 128, false, x); });
  run("  diag128 H", 1, [&] { k_trsv_diag128<float, float><<<1, TRB, sm>>>(M, n, 0, 0, 0, 128, true, x); });
  run("  off N", 1, [&] { k_trsv_off<float, float><<<(n - 128 + 63) / 64, KT>>>(M, n, 0, 0, n - 128, 128, n, false, x); });
  run("  off H", 1, [&] { k_trsv_off<float, float><<<(n - 128 + 7) / 8, KT>>>(M, n, 0, 0, 0, 128, n, true, x); });
  return 0;
}
