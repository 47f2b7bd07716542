/*
 * oracle/orc_api.h -- TEST INFRASTRUCTURE ONLY.
 *
 * The C surface shared by the two CPU checkers of this repository:
 *   oracle/_ref/libmixedls_ref.so   the UNMODIFIED reference headers
 *                                   (/root/reference/proj/include/mixedls)
 *                                   compiled behind this ABI by oracle/ref_shim.cpp
 *   oracle/_build/libmixedls_port.so  oracle/port/mixedls_port.cpp, a restatement
 *                                   of the same algorithms (real + complex)
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg load
 * these libraries, and only as the checker / the CPU arm.  The product
 * (paper_2406_16499_b200/, libmixedls_b200.so) never links or calls them.
 *
 * Conventions: column-major float64, leading dimension == rows.
 * Return codes mirror the reference exception types (inc/errors.hpp:14-49):
 *   0 ok, 1 dimension_error, 2 invalid_input, 3 singular_triangular
 *   (pivot index in *sing), 9 any other exception.
 * Precision codes: 0 = low (binary32), 1 = working (binary64), 2 = extended.
 * status codes: 0 converged, 1 max_iterations, 2 diverged (inc/refine.hpp:17).
 * hist receives iterations*3 unscaled residual norms (room for maxit*3).
 * phases receives the six phase_times fields (inc/refine.hpp:46-53).
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int orc_mplse(int64_t m, int64_t n, int64_t p, const double* A, const double* B,
              const double* b, const double* d, double tol, int64_t maxit, int uf, int us,
              int ur, double* x, double* r, double* v, int32_t* status, int64_t* iters,
              double* hist, double* phases, int64_t* sing);

int orc_mpgls(int64_t n, int64_t m, int64_t p, const double* W, const double* V,
              const double* d, double tol, int64_t maxit, int uf, int us, int ur, double* x,
              double* y, double* z, int32_t* status, int64_t* iters, double* hist,
              double* phases, int64_t* sing);

/* independent solves over a std::thread pool (the run_sweep pattern,
 * inc/experiment.hpp:191-217).  Problem i's arrays start at i*m*n etc. */
int orc_mplse_batch(int64_t batch, int64_t m, int64_t n, int64_t p, const double* A,
                    const double* B, const double* b, const double* d, double tol,
                    int64_t maxit, int uf, int us, int ur, double* x, double* r, double* v,
                    int32_t* status, int64_t* iters, int32_t* err, int nthreads);

/* the reference's own seeded generator (inc/generate.hpp:60-106), dist 0 = geometric */
int orc_gen_lse(int64_t m, int64_t n, int64_t p, double cond, uint64_t seed, int dist,
                double* A, double* B, double* b, double* d);
int orc_gen_gls(int64_t n, int64_t m, int64_t p, double cond, uint64_t seed, int dist,
                double* W, double* V, double* d);

/* components */
int orc_lse_residuals(int64_t m, int64_t n, int64_t p, const double* A, const double* B,
                      const double* b, const double* d, const double* x, const double* r,
                      const double* v, int ur, double* f1, double* f2, double* f3);
int orc_gls_residuals(int64_t n, int64_t m, int64_t p, const double* W, const double* V,
                      const double* d, const double* x, const double* y, const double* z,
                      int ur, double* f1, double* f2, double* f3);
/* factor (B, A) at uf, then one correction solve at uf's precision on (f1,f2,f3)
 * (demoted by a plain cast when uf = low, as in proj/tests/acceptance_tests.cpp:184-189) */
int orc_lse_correction(int64_t m, int64_t n, int64_t p, const double* A, const double* B,
                       const double* f1, const double* f2, const double* f3, int uf,
                       double* dr, double* dv, double* dx, int64_t* sing);
int orc_gls_correction(int64_t n, int64_t m, int64_t p, const double* W, const double* V,
                       const double* f1, const double* f2, const double* f3, int uf,
                       double* dy, double* dz, double* dx, int64_t* sing);
/* GMRES-IR (inc/krylov.hpp:545 gmres_refine_lse), reference build only:
 * precond 0 = left, 1 = bd_split; inner = total GMRES iterations */
int orc_gmres_lse(int64_t m, int64_t n, int64_t p, const double* A, const double* B,
                  const double* b, const double* d, double tol, int64_t maxit, int uf, int us,
                  int ur, int precond, double alpha_scale, double* x, double* r, double* v,
                  int32_t* status, int64_t* iters, int64_t* inner, double* hist, int64_t* sing);

/* GMRES-IR for GLS (inc/krylov.hpp:673 gmres_refine_gls), reference build only */
int orc_gmres_gls(int64_t n, int64_t m, int64_t p, const double* W, const double* V,
                  const double* d, double tol, int64_t maxit, int uf, int us, int ur, int precond,
                  double alpha_scale, double* x, double* y, double* z, int32_t* status,
                  int64_t* iters, int64_t* inner, double* hist, int64_t* sing);

/* binary64 direct solves (the err-2 / er-2 denominators, inc/experiment.hpp:50-73) */
int orc_lse_direct(int64_t m, int64_t n, int64_t p, const double* A, const double* B,
                   const double* b, const double* d, double* x, double* r, double* v,
                   int64_t* sing);
int orc_gls_direct(int64_t n, int64_t m, int64_t p, const double* W, const double* V,
                   const double* d, double* x, double* y, double* z, int64_t* sing);
double orc_extended_dot(int64_t n, const double* x, const double* y);
/* upper-triangular solve of the n x n column-major T (transpose: 0/1) */
int orc_trsv(int64_t n, const double* T, const double* rhs, int transpose, double* x,
             int64_t* sing);

#ifdef __cplusplus
}
#endif
