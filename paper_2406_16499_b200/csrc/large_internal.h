// Internal interfaces of the large-problem path (blocked GRQ/GQR + host-driven IR).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "large_common.cuh"

namespace mlsb {
namespace lg {

// C = alpha op(A) op(B) + beta C (column-major; ha/hb: conjugate-transpose A/B).
// `work` (>= M*N*splits elements) enables split-K for the alpha = 1, beta = 0 case.
cudaError_t gemm_f32(bool ha, bool hb, int M, int N, int K, float alpha, const float* A,
                     int64_t lda, const float* B, int64_t ldb, float beta, float* C, int64_t ldc,
                     float* work, size_t work_elems, cudaStream_t st);
cudaError_t gemm_f64(bool ha, bool hb, int M, int N, int K, double alpha, const double* A, int64_t lda,
                     const double* B, int64_t ldb, double beta, double* C, int64_t ldc, double* work,
                     size_t work_elems, cudaStream_t st);
cudaError_t gemm_c64(bool ha, bool hb, int M, int N, int K, cf alpha, const cf* A, int64_t lda,
                     const cf* B, int64_t ldb, cf beta, cf* C, int64_t ldc, cf* work,
                     size_t work_elems, cudaStream_t st);

// cap on the resident CTAs of the binary32 WY GEMMs issued by this host thread
// (0 = none): the trailing updates leave SMs to the look-ahead stream
void set_gemm_cta_cap(int cap);

constexpr int NB = 32;       // reflectors per panel / WY block
constexpr int NBO = 128;     // reflectors per outer block (one trailing update)
constexpr int PCL = 16;      // CTAs per panel cluster

// Tout (nbo x nbo, ld ldt) = T of the outer block whose NB-wide panels have
// T_j at Tp + j NB NB (ld NB) and Gram matrix G = V^H V (ld ldg).
cudaError_t tmerge_f32(int nbo, const float* G, int ldg, const float* Tp, float* Tout, int ldt,
                       cudaStream_t st);
cudaError_t tmerge_c64(int nbo, const cf* G, int ldg, const cf* Tp, cf* Tout, int ldt, cudaStream_t st);
cudaError_t tmerge_f64(int nbo, const double* G, int ldg, const double* Tp, double* Tout, int ldt,
                       cudaStream_t st);

// One panel of NB Householder reflectors, factored by a PCL-CTA cluster.
// QR view P (L x nb): P[r][q] = M[r0 + r, c0 + q]           (rq = false)
//                     P[r][q] = conj(M[r0 - q, c0 - r])     (rq = true: row panel,
//                                                            rows bottom-up, pivots from the right)
// Outputs: the factored panel written back through the same map (R / beta on
// and above the diagonal, v below it), tau[q], the dense reflector block
// V[idx(r) + q ldv] with explicit unit and zeros (idx(r) = r for QR,
// ...  L-1-r for RQ, i.e. M-column order), and T (nb x nb, column-major) with
// P_block = H_0 ... H_{nb-1} = I - V T V^H.
// vbase: (RQ) M column stored in V row 0.
template <class T>
cudaError_t panel_factor(T* M, int64_t ld, int64_t r0, int64_t c0, int L, int nb, bool rq, T* tau,
                         T* V, int64_t ldv, T* Tm, int64_t vbase, cudaStream_t st,
                         long long* probe = nullptr);

// One problem on the whole GPU (device pointers, column-major; WT = binary64 or
// complex128 interleaved).  LSE: A m x n, B p x n, b, d -> x, r, v.
// GLS: A = W n x m, B = V n x p, d -> x, r = y, v = z.
struct LargeProblem {
  int kind;
  int64_t m, n, p;
  const void* A;
  int64_t lda;
  const void* B;
  int64_t ldb;
  const void* b;
  const void* d;
  void* x;
  void* r;
  void* v;
  double tol;
  int64_t maxit;
  int u_f, u_s, u_r;
  bool cplx;
  // GMRES-IR (krylov.hpp:545-689): 0 = classical IR, 1 = left preconditioner,
  // 2 = block-diagonal split preconditioner; alpha = alpha_scale * ||r0||
  int gmres = 0;
  double alpha_scale = 1.0;
};
struct LargeOut {
  int status = 1;
  int64_t iters = 0;
  int err = 0;
  int64_t sing = -1;
  int64_t inner = 0;  // GMRES iterations summed over the passes
  std::vector<double> hist;
  double phases[6] = {0, 0, 0, 0, 0, 0};
};
// returns an mlsb_error code (argument/launch failures); solver errors in out->err
int large_solve(const LargeProblem& P, cudaStream_t st, LargeOut* out);

}  // namespace lg
}  // namespace mlsb
