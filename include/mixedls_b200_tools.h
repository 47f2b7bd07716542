/*
 * mixedls_b200_tools.h -- measurement helpers exported by libmixedls_b200.so
 * next to the reference-facing API (mixedls_b200.h).  They have no reference
 * counterpart: they measure the SIMT roofline denominators on the running
 * B200 (FP32/FP64 peaks are not in MEASURED_PEAKS.json).
 */
#ifndef MIXEDLS_B200_TOOLS_H
#define MIXEDLS_B200_TOOLS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* best-of-5 FMA throughput of a full-occupancy register-only kernel, TFLOP/s
 * (2 flops per FMA); device -1 = current; stream may be NULL; -1 on error */
double mlsb_fp32_fma_peak_tflops(int device, void* stream);
double mlsb_fp64_fma_peak_tflops(int device, void* stream);

/* The large path's building blocks, exported so bench.py can time them on
 * their own against the roofline (device pointers, column-major):
 *   mlsb_wy_gemm_f32: C = alpha op(A) op(B) + beta C, op = N or T (ta/tb != 0),
 *     the binary32 SIMT GEMM of the compact-WY trailing updates; `work`
 *     (>= M*N*64 floats, may be NULL) enables split-K for alpha=1, beta=0.
 *   mlsb_panel_f32: one NB=32-reflector Householder panel (QR view, rows
 *     r0.., columns c0..c0+nb) of the L x nb block of M, factored by one
 *     thread-block cluster; V (L x nb at ldv), tau (nb), T (32 x 32).
 * Return 0 or a CUDA error code. */
int mlsb_wy_gemm_f32(int ta, int tb, int M, int N, int K, float alpha, const float* A, int64_t lda,
                     const float* B, int64_t ldb, float beta, float* C, int64_t ldc, float* work,
                     size_t work_elems, void* stream);
int mlsb_panel_f32(float* M, int64_t ld, int64_t r0, int64_t c0, int L, int nb, float* tau, float* V,
                   int64_t ldv, float* T, void* stream);
/* the complex64 panel (interleaved re, im; ld, ldv in complex elements) */
int mlsb_panel_c64(float* M, int64_t ld, int64_t r0, int64_t c0, int L, int nb, float* tau, float* V,
                   int64_t ldv, float* T, void* stream);
/* the same panel (r0 = c0 = 0, ldv = L) with clock64 stamps of CTA 0 /
 * thread 0 written to probe[8 q + phase] for each reflector q */
int mlsb_panel_probe_f32(float* M, int64_t ld, int L, int nb, float* tau, float* V, float* T,
                         long long* probe, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MIXEDLS_B200_TOOLS_H */
