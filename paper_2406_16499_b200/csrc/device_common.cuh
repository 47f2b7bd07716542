// Device helpers shared by the B200 kernels: warp/block reductions,
// double-double error-free transformations, timers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mlsb {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// max that skips NaN (the reference's std::max(m, |x|) never selects a NaN)
__device__ __forceinline__ double nanskip_max(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---- double-double (precision.hpp:131-175 semantics) ----------------------
struct dd {
  double s, c;
};
// Knuth TwoSum: s + e = a + b exactly
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double z = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, z)), __dsub_rn(b, z));
}
// acc += a*b with the product and the sum error carried in acc.c (Dot2)
__device__ __forceinline__ void dd_fma(dd& acc, double a, double b) {
  const double p = __dmul_rn(a, b);
  const double pe = fma(a, b, -p);
  double s, se;
  two_sum(acc.s, p, s, se);
  acc.s = s;
  acc.c = __dadd_rn(acc.c, __dadd_rn(se, pe));
}
__device__ __forceinline__ void dd_merge(dd& a, const dd& b) {
  double s, e;
  two_sum(a.s, b.s, s, e);
  a.s = s;
  a.c = __dadd_rn(__dadd_rn(a.c, b.c), e);
}
__device__ __forceinline__ dd warp_dd_sum(dd v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    dd w;
    w.s = __shfl_xor_sync(0xffffffffu, v.s, o);
    w.c = __shfl_xor_sync(0xffffffffu, v.c, o);
    // merge in a lane-symmetric order so every lane ends with the same value
    const int lane = threadIdx.x & 31;
    if (lane & o) {
      dd t = w;
      dd_merge(t, v);
      v = t;
    } else {
      dd_merge(v, w);
    }
  }
  return v;
}

// mbarrier (shared::cta) helpers: arrive = release, try_wait = acquire, CTA scope
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ---- block reductions (fixed order, deterministic); results in out[], all threads synced
template <int N, int NW = 16>
__device__ __forceinline__ void block_sum(double (&v)[N], double* red, double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < N; ++k) red[warp * 8 + k] = v[k];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double t = lane < NW ? red[lane * 8 + k] : 0.0;
      t = warp_sum(t);
      if (lane == 0) out[k] = t;
    }
  }
  __syncthreads();
}
template <int N, int NW = 16>
__device__ __forceinline__ void block_max(double (&v)[N], double* red, double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = warp_max(v[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < N; ++k) red[warp * 8 + k] = v[k];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double t = lane < NW ? red[lane * 8 + k] : 0.0;
      t = warp_max(t);
      if (lane == 0) out[k] = t;
    }
  }
  __syncthreads();
}

}  // namespace mlsb
