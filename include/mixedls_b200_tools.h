/*
 * mixedls_b200_tools.h -- measurement helpers exported by libmixedls_b200.so
 * next to the reference-facing API (mixedls_b200.h).  They have no reference
 * counterpart: they measure the SIMT roofline denominators on the running
 * B200 (FP32/FP64 peaks are not in MEASURED_PEAKS.json).
 */
#ifndef MIXEDLS_B200_TOOLS_H
#define MIXEDLS_B200_TOOLS_H

#ifdef __cplusplus
extern "C" {
#endif

/* best-of-5 FMA throughput of a full-occupancy register-only kernel, TFLOP/s
 * (2 flops per FMA); device -1 = current; stream may be NULL; -1 on error */
double mlsb_fp32_fma_peak_tflops(int device, void* stream);
double mlsb_fp64_fma_peak_tflops(int device, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MIXEDLS_B200_TOOLS_H */
