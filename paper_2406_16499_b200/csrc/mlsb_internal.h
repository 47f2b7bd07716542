// Internal interfaces between the C-ABI layer (capi.cu) and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mlsb {

enum Kind : int { KIND_LSE = 0, KIND_GLS = 1 };

// One launch of the fused tile solver: `batch` independent problems of one
// shape, one CTA per problem.  All pointers are device pointers.
//   LSE:  A = A (m x n), B = B (p x n), b, d;   outputs x (n), r (m), v (p)
//   GLS:  A = W (n x m), B = V (n x p), d;      outputs x (m), r = y (p), v = z (n)
struct TileArgs {
  int kind;
  int64_t m, n, p;
  int64_t batch;
  const double* A;
  int64_t lda, sA;
  const double* B;
  int64_t ldb, sB;
  const double* b;
  int64_t sb;
  const double* d;
  int64_t sd;
  double* x;
  double* r;
  double* v;
  int32_t* status;   // [batch] or null
  int64_t* iters;    // [batch] or null
  int32_t* err;      // [batch] (required)
  int64_t* sing;     // [batch] or null
  double* hist;      // [batch * maxit * 3] or null
  double* phases;    // [batch * 6] or null (ns -> s converted on host)
  double tol;
  int64_t maxit;
  int u_f, u_s, u_r;
  void* gws;         // per-problem factor workspace in global memory, or null (shared memory)
  unsigned long long* stamps;  // debug: globaltimer stamps of problem 0 (MLSB_DEBUG_STAMPS), or null
  int opts = 0;                // kernel variant bits (A/B switches), 0 = product configuration
  int opts2 = 0;               // second A/B parameter
};

// shared-memory bytes the tile solver needs for this shape/precision
// (0 if the shape cannot be handled by one CTA)
size_t tile_smem_bytes(int kind, int64_t m, int64_t n, int64_t p, int u_f, int u_s, int u_r,
                       bool m_global);
// bytes of the per-problem global factor workspace (M in global memory)
size_t tile_gws_bytes(int kind, int64_t m, int64_t n, int64_t p, int u_f);
// max dynamic shared memory per block on the current device
size_t device_smem_limit();
cudaError_t launch_tile_solver(const TileArgs& a, cudaStream_t stream);

// register-resident LSE tile solver (m + p <= 288, n <= 128, u_f = binary32,
// u_r = binary64): BASELINE configs 1 and 4
void* probe_buffer();  // debug (MLSB_PROBE builds): clock64 probe slots, or nullptr
bool lse_reg_supported(int64_t m, int64_t n, int64_t p, int u_f, int u_s, int u_r,
                       size_t smem_limit);
cudaError_t launch_lse_reg(const TileArgs& a, cudaStream_t stream);

}  // namespace mlsb
