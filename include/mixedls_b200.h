/*
 * mixedls_b200.h -- C ABI of libmixedls_b200.so, the B200 (sm_100a) drop-in
 * for the classical mixed-precision iterative-refinement path of the
 * reference library `mixedls` (arXiv 2406.16499).
 *
 * Reference interface each entry point replaces (paths relative to
 * /root/reference/proj/include/mixedls):
 *
 *   mlsb_mplse          mplse(const lse_problem&, const refinement_config&)
 *                       -> mplse_result                        lse.hpp:303-429
 *   mlsb_mpgls          mpgls(const gls_problem&, const refinement_config&)
 *                       -> mpgls_result                        gls.hpp:276-387
 *   mlsb_mplse_batched  independent mplse calls, the run_sweep pattern of
 *                       run_experiment                         experiment.hpp:191-217
 *   mlsb_mpgls_batched  idem for mpgls
 *   mlsb_mpgls_z        complex128 GLS with complex64 factors (BASELINE config 5);
 *                       no reference counterpart (the reference is real-only)
 *   mlsb_config         refinement_config {tol, maxit, precision_config}
 *                                                               refine.hpp:28-38,
 *                                                               precision.hpp:57-90
 *   mlsb_trace          refinement_trace {status, iterations, residual_history,
 *                       inner_iterations, timing}               refine.hpp:46-61
 *   return codes        the exception types of errors.hpp:14-49 (dimension_error,
 *                       invalid_input, singular_triangular{index}); non-convergence
 *                       is NOT an error, it is trace.status (as in the reference).
 *
 * Storage is column-major float64 exactly as dense_matrix<double>
 * (matrix.hpp:21-50), with explicit leading dimensions.  Outputs are the
 * UNSCALED state, as the reference returns it (lse.hpp:424-426, gls.hpp:382-384).
 *
 * Every entry point runs on the GPU; there is no CPU fallback.  If no CUDA
 * device is usable the call returns MLSB_ERR_CUDA.
 */
#ifndef MIXEDLS_B200_H
#define MIXEDLS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* precision_level (precision.hpp:23-52) */
enum mlsb_precision { MLSB_LOW = 0, MLSB_WORKING = 1, MLSB_EXTENDED = 2 };

/* refine_status (refine.hpp:17) */
enum mlsb_status { MLSB_CONVERGED = 0, MLSB_MAX_ITERATIONS = 1, MLSB_DIVERGED = 2 };

/* return codes (errors.hpp:14-49) */
enum mlsb_error {
  MLSB_OK = 0,
  MLSB_ERR_DIMENSION = 1,      /* dimension_error */
  MLSB_ERR_INVALID_INPUT = 2,  /* invalid_input */
  MLSB_ERR_SINGULAR = 3,       /* singular_triangular; pivot index in *singular_index */
  MLSB_ERR_CUDA = 4,           /* no device / launch failure / out of memory */
  MLSB_ERR_UNSUPPORTED = 5,    /* shape or precision combination not built */
  MLSB_ERR_OTHER = 9
};

/* where the caller's arrays live */
enum mlsb_pointer_kind { MLSB_HOST = 0, MLSB_DEVICE = 1 };

/* refinement_config: tol > 0, maxit >= 1, u_f >= u_s >= u >= u_r with u = working.
 * Rejected exactly where precision_config::validate() / refinement_config::validate()
 * throw invalid_input (precision.hpp:63-70, refine.hpp:33-37). */
typedef struct mlsb_config {
  double tol;     /* default 1e-13 */
  int64_t maxit;  /* default 40 */
  int32_t u_f;    /* factorization precision, default MLSB_LOW */
  int32_t u_s;    /* correction-solve precision, default MLSB_LOW */
  int32_t u;      /* working precision, must be MLSB_WORKING */
  int32_t u_r;    /* residual precision, default MLSB_WORKING */
} mlsb_config;

/* refinement_trace.  residual_history is caller-owned (>= 3*maxit doubles,
 * row i = unscaled (||f1||, ||f2||, ||f3||) of pass i+1) or NULL.
 * phase_seconds = {factorization, init, residual, correction, gmres, other},
 * measured on the device. */
typedef struct mlsb_trace {
  int32_t status;
  int32_t reserved;
  int64_t iterations;       /* loop passes, the final residual-only pass included */
  int64_t inner_iterations; /* always 0 for classical IR */
  double* residual_history;
  double phase_seconds[6];
} mlsb_trace;

/* execution context; NULL means {MLSB_HOST, current device, default stream} */
typedef struct mlsb_exec {
  int32_t pointer_kind; /* MLSB_HOST or MLSB_DEVICE for every array argument */
  int32_t device;       /* CUDA ordinal, -1 = current */
  void* stream;         /* cudaStream_t or NULL (legacy default stream) */
} mlsb_exec;

mlsb_config mlsb_default_config(void);
const char* mlsb_last_error(void); /* thread-local message of the last non-OK return */
int mlsb_version(void);

/* LSE: min ||A x - b|| s.t. B x = d.  A m x n (lda >= m), B p x n (ldb >= p),
 * requires p <= n <= m + p.  Outputs x (n), r = b - A x (m), v (p). */
int mlsb_mplse(const double* A, int64_t lda, const double* B, int64_t ldb, const double* b,
               const double* d, int64_t m, int64_t n, int64_t p, const mlsb_config* cfg,
               double* x, double* r, double* v, mlsb_trace* trace, int64_t* singular_index,
               const mlsb_exec* exec);

/* GLS: min ||y|| s.t. W x + V y = d.  W n x m (ldw >= n), V n x p (ldv >= n),
 * requires m <= n <= m + p.  Outputs x (m), y (p), z (n). */
int mlsb_mpgls(const double* W, int64_t ldw, const double* V, int64_t ldv, const double* d,
               int64_t n, int64_t m, int64_t p, const mlsb_config* cfg, double* x, double* y,
               double* z, mlsb_trace* trace, int64_t* singular_index, const mlsb_exec* exec);

/* binary64 direct solvers: the err-2 / er-2 reference of the experiment
 * harness (detail::lse_direct_reference / gls_direct_reference,
 * inc/experiment.hpp:50-73, over lse_direct inc/lse.hpp:132-152 and
 * gls_direct inc/gls.hpp:85-91).  GRQ / GQR and the null-space solve at
 * binary64 (no pre-scaling, no refinement); LSE r = b - A x and v from
 * R^T v = (Q A^T r)(n-p:n), GLS z = Q [0; T22^-T (Z y)(k:p)] -- the same
 * quantities the reference forms through the factors.  Zero pivots give
 * MLSB_ERR_SINGULAR with the reference's index. */
int mlsb_lse_direct(const double* A, int64_t lda, const double* B, int64_t ldb, const double* b,
                    const double* d, int64_t m, int64_t n, int64_t p, double* x, double* r,
                    double* v, int64_t* singular_index, const mlsb_exec* exec);
int mlsb_gls_direct(const double* W, int64_t ldw, const double* V, int64_t ldv, const double* d,
                    int64_t n, int64_t m, int64_t p, double* x, double* y, double* z,
                    int64_t* singular_index, const mlsb_exec* exec);

/* GMRES-IR for LSE (gmres_refine_lse, inc/krylov.hpp:545-689): the outer
 * loop of mplse with each correction system solved by full MGS-GMRES
 * (binary64, rel_tol 1e-6) on the alpha-scaled augmented operator, alpha =
 * alpha_scale * ||r0||, preconditioned by the binary32 GRQ factors widened to
 * binary64.  precond: MLSB_PRECOND_LEFT (krylov.hpp:209-230, with the
 * triangular cascade as initial guess) or MLSB_PRECOND_BD_SPLIT (two-sided,
 * krylov.hpp:253-287, both the m >= n and the n > m case).  Built for
 * u_f = low; other factor precisions return MLSB_ERR_UNSUPPORTED.
 * trace->inner_iterations = total GMRES iterations. */
enum { MLSB_PRECOND_LEFT = 0, MLSB_PRECOND_BD_SPLIT = 1 };
int mlsb_gmres_lse(const double* A, int64_t lda, const double* B, int64_t ldb, const double* b,
                   const double* d, int64_t m, int64_t n, int64_t p, const mlsb_config* cfg,
                   int precond, double alpha_scale, double* x, double* r, double* v,
                   mlsb_trace* trace, int64_t* singular_index, const mlsb_exec* exec);

/* GMRES-IR for GLS (gmres_refine_gls, inc/krylov.hpp:673-784): the outer
 * loop of mpgls with each correction solved by full MGS-GMRES on the alpha-
 * scaled GLS augmented operator [a I_p V^T 0; V 0 W; 0 W^T 0] (krylov.hpp:
 * 24-26), alpha = alpha_scale * ||y0||, pre-scaling s_W = s_V ||W||_F/||V||_F.
 * precond: MLSB_PRECOND_LEFT (left_gls_apply, krylov.hpp:232-250, cascade
 * initial guess) or MLSB_PRECOND_BD_SPLIT (bd_gls_apply, krylov.hpp:288-321,
 * both the n <= p and the n > p case).  Built for u_f = low. */
int mlsb_gmres_gls(const double* W, int64_t ldw, const double* V, int64_t ldv, const double* d,
                   int64_t n, int64_t m, int64_t p, const mlsb_config* cfg, int precond,
                   double alpha_scale, double* x, double* y, double* z, mlsb_trace* trace,
                   int64_t* singular_index, const mlsb_exec* exec);

/* Complex128 problems (interleaved re, im; same shapes and semantics with
 * Hermitian transposes), solved with complex64 factors at u_f = low.  The
 * reference is real-only; these serve BASELINE config 5. */
int mlsb_mplse_z(const double* A, int64_t lda, const double* B, int64_t ldb, const double* b,
                 const double* d, int64_t m, int64_t n, int64_t p, const mlsb_config* cfg,
                 double* x, double* r, double* v, mlsb_trace* trace, int64_t* singular_index,
                 const mlsb_exec* exec);
int mlsb_mpgls_z(const double* W, int64_t ldw, const double* V, int64_t ldv, const double* d,
                 int64_t n, int64_t m, int64_t p, const mlsb_config* cfg, double* x, double* y,
                 double* z, mlsb_trace* trace, int64_t* singular_index, const mlsb_exec* exec);

/* Batched LSE over `batch` independent problems of one shape.  Problem i reads
 * A + i*strideA, B + i*strideB, b + i*strideb, d + i*strided and writes
 * x + i*n, r + i*m, v + i*p.  Per-problem status, iterations and error code
 * (MLSB_OK / _SINGULAR / _INVALID_INPUT) go to the optional arrays; history
 * (batch*maxit*3) and singular_index (batch) are optional too.  The return
 * value reports argument / launch errors only. */
int mlsb_mplse_batched(int64_t batch, const double* A, int64_t lda, int64_t strideA,
                       const double* B, int64_t ldb, int64_t strideB, const double* b,
                       int64_t strideb, const double* d, int64_t strided, int64_t m, int64_t n,
                       int64_t p, const mlsb_config* cfg, double* x, double* r, double* v,
                       int32_t* status, int64_t* iterations, int32_t* errcode,
                       int64_t* singular_index, double* history, const mlsb_exec* exec);

int mlsb_mpgls_batched(int64_t batch, const double* W, int64_t ldw, int64_t strideW,
                       const double* V, int64_t ldv, int64_t strideV, const double* d,
                       int64_t strided, int64_t n, int64_t m, int64_t p, const mlsb_config* cfg,
                       double* x, double* y, double* z, int32_t* status, int64_t* iterations,
                       int32_t* errcode, int64_t* singular_index, double* history,
                       const mlsb_exec* exec);

#ifdef __cplusplus
}
#endif

#endif /* MIXEDLS_B200_H */
