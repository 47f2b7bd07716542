// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (see oracle/orc_api.h).
//
// Exposes the UNMODIFIED reference library (header-only C++20, included by
// path from /root/reference/proj/include) behind the C surface in
// orc_api.h.  Built by oracle/Makefile into oracle/_ref/libmixedls_ref.so
// with the reference's own Release flags (-O3 -DNDEBUG -std=c++20, no -march;
// proj/CMakeLists.txt:1-8).  Nothing here re-implements an algorithm: each
// entry point marshals arrays into the reference's types and calls
//   mplse  inc/lse.hpp:303      mpgls  inc/gls.hpp:276
//   lse_residuals inc/lse.hpp:181, gls_residuals inc/gls.hpp:161
//   lse_correction_solve inc/lse.hpp:84, gls_correction_solve inc/gls.hpp:107
//   lse_direct inc/lse.hpp:132, gls_direct inc/gls.hpp:85
//   gen_lse_problem / gen_gls_problem inc/generate.hpp:60-106
//   gmres_refine_lse inc/krylov.hpp:545, gmres_refine_gls inc/krylov.hpp:673
#include <algorithm>
#include <atomic>
#include <cstring>
#include <thread>
#include <vector>

#include "mixedls/errors.hpp"
#include "mixedls/generate.hpp"
#include "mixedls/gls.hpp"
#include "mixedls/krylov.hpp"
#include "mixedls/lse.hpp"

#include "orc_api.h"

using namespace mixedls;

namespace {

dense_matrix<double> to_mat(const double* p, int64_t r, int64_t c) {
    dense_matrix<double> M(r, c);
    std::memcpy(M.data().data(), p, sizeof(double) * r * c);
    return M;
}
std::vector<double> to_vec(const double* p, int64_t n) { return std::vector<double>(p, p + n); }
void put(const std::vector<double>& v, double* out) {
    if (out) std::copy(v.begin(), v.end(), out);
}

precision_level lvl(int c) {
    if (c == 0) return precision_level::low();
    if (c == 2) return precision_level::extended();
    return precision_level::working();
}

refinement_config make_cfg(double tol, int64_t maxit, int uf, int us, int ur) {
    refinement_config cfg;
    cfg.tol = tol;
    cfg.maxit = static_cast<std::size_t>(maxit < 0 ? 0 : maxit);
    cfg.precisions.factor = lvl(uf);
    cfg.precisions.solve = lvl(us);
    cfg.precisions.residual = lvl(ur);
    return cfg;
}

template <typename F>
int guarded(F&& fn, int64_t* sing) {
    try {
        fn();
        return 0;
    } catch (const singular_triangular& e) {
        if (sing) *sing = static_cast<int64_t>(e.index);
        return 3;
    } catch (const dimension_error&) {
        return 1;
    } catch (const invalid_input&) {
        return 2;
    } catch (...) {
        return 9;
    }
}

void put_trace(const refinement_trace& t, int32_t* status, int64_t* iters, double* hist,
               double* phases) {
    if (status) *status = static_cast<int32_t>(t.status);
    if (iters) *iters = static_cast<int64_t>(t.iterations);
    if (hist)
        for (std::size_t i = 0; i < t.residual_history.size(); ++i) {
            hist[3 * i + 0] = t.residual_history[i].f1;
            hist[3 * i + 1] = t.residual_history[i].f2;
            hist[3 * i + 2] = t.residual_history[i].f3;
        }
    if (phases) {
        phases[0] = t.timing.factorization;
        phases[1] = t.timing.init;
        phases[2] = t.timing.residual;
        phases[3] = t.timing.correction;
        phases[4] = t.timing.gmres;
        phases[5] = t.timing.other;
    }
}

lse_problem make_lse(int64_t m, int64_t n, int64_t p, const double* A, const double* B,
                     const double* b, const double* d) {
    lse_problem pb;
    pb.A = to_mat(A, m, n);
    pb.B = to_mat(B, p, n);
    pb.b = to_vec(b, m);
    pb.d = to_vec(d, p);
    return pb;
}

gls_problem make_gls(int64_t n, int64_t m, int64_t p, const double* W, const double* V,
                     const double* d) {
    gls_problem pb;
    pb.W = to_mat(W, n, m);
    pb.V = to_mat(V, n, p);
    pb.d = to_vec(d, n);
    return pb;
}

}  // namespace

extern "C" {

int orc_mplse(int64_t m, int64_t n, int64_t p, const double* A, const double* B,
              const double* b, const double* d, double tol, int64_t maxit, int uf, int us,
              int ur, double* x, double* r, double* v, int32_t* status, int64_t* iters,
              double* hist, double* phases, int64_t* sing) {
    return guarded(
        [&] {
            auto pb = make_lse(m, n, p, A, B, b, d);
            auto res = mplse(pb, make_cfg(tol, maxit, uf, us, ur));
            put(res.state.x, x);
            put(res.state.r, r);
            put(res.state.v, v);
            put_trace(res.trace, status, iters, hist, phases);
        },
        sing);
}

int orc_gmres_lse(int64_t m, int64_t n, int64_t p, const double* A, const double* B,
                  const double* b, const double* d, double tol, int64_t maxit, int uf, int us,
                  int ur, int precond, double alpha_scale, double* x, double* r, double* v,
                  int32_t* status, int64_t* iters, int64_t* inner, double* hist, int64_t* sing) {
    return guarded(
        [&] {
            auto pb = make_lse(m, n, p, A, B, b, d);
            auto res = gmres_refine_lse(pb, make_cfg(tol, maxit, uf, us, ur),
                                        precond == 0 ? precond_choice::left : precond_choice::bd_split,
                                        alpha_scale);
            put(res.state.x, x);
            put(res.state.r, r);
            put(res.state.v, v);
            put_trace(res.trace, status, iters, hist, nullptr);
            if (inner) *inner = static_cast<int64_t>(res.trace.inner_iterations);
        },
        sing);
}

int orc_gmres_gls(int64_t n, int64_t m, int64_t p, const double* W, const double* V,
                  const double* d, double tol, int64_t maxit, int uf, int us, int ur, int precond,
                  double alpha_scale, double* x, double* y, double* z, int32_t* status,
                  int64_t* iters, int64_t* inner, double* hist, int64_t* sing) {
    return guarded(
        [&] {
            auto pb = make_gls(n, m, p, W, V, d);
            auto res = gmres_refine_gls(pb, make_cfg(tol, maxit, uf, us, ur),
                                        precond == 0 ? precond_choice::left : precond_choice::bd_split,
                                        alpha_scale);
            put(res.state.x, x);
            put(res.state.y, y);
            put(res.state.z, z);
            put_trace(res.trace, status, iters, hist, nullptr);
            if (inner) *inner = static_cast<int64_t>(res.trace.inner_iterations);
        },
        sing);
}

int orc_mpgls(int64_t n, int64_t m, int64_t p, const double* W, const double* V,
              const double* d, double tol, int64_t maxit, int uf, int us, int ur, double* x,
              double* y, double* z, int32_t* status, int64_t* iters, double* hist,
              double* phases, int64_t* sing) {
    return guarded(
        [&] {
            auto pb = make_gls(n, m, p, W, V, d);
            auto res = mpgls(pb, make_cfg(tol, maxit, uf, us, ur));
            put(res.state.x, x);
            put(res.state.y, y);
            put(res.state.z, z);
            put_trace(res.trace, status, iters, hist, phases);
        },
        sing);
}

int orc_mplse_batch(int64_t batch, int64_t m, int64_t n, int64_t p, const double* A,
                    const double* B, const double* b, const double* d, double tol,
                    int64_t maxit, int uf, int us, int ur, double* x, double* r, double* v,
                    int32_t* status, int64_t* iters, int32_t* err, int nthreads) {
    const int T = std::max(1, nthreads);
    std::atomic<int64_t> next{0};
    auto worker = [&] {
        for (;;) {
            const int64_t i = next.fetch_add(1);
            if (i >= batch) return;
            int64_t sing = -1;
            const int rc = orc_mplse(m, n, p, A + i * m * n, B + i * p * n, b + i * m, d + i * p,
                                     tol, maxit, uf, us, ur, x ? x + i * n : nullptr,
                                     r ? r + i * m : nullptr, v ? v + i * p : nullptr,
                                     status ? status + i : nullptr, iters ? iters + i : nullptr,
                                     nullptr, nullptr, &sing);
            if (err) err[i] = rc;
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    return 0;
}

int orc_gen_lse(int64_t m, int64_t n, int64_t p, double cond, uint64_t seed, int dist,
                double* A, double* B, double* b, double* d) {
    return guarded(
        [&] {
            generator_spec gs;
            gs.kind = problem_kind::lse;
            gs.m = m;
            gs.n = n;
            gs.p = p;
            gs.cond = cond;
            gs.seed = seed;
            gs.distribution = dist ? sv_distribution::arithmetic : sv_distribution::geometric;
            auto pb = gen_lse_problem(gs);
            put(pb.A.data(), A);
            put(pb.B.data(), B);
            put(pb.b, b);
            put(pb.d, d);
        },
        nullptr);
}

int orc_gen_gls(int64_t n, int64_t m, int64_t p, double cond, uint64_t seed, int dist,
                double* W, double* V, double* d) {
    return guarded(
        [&] {
            generator_spec gs;
            gs.kind = problem_kind::gls;
            gs.m = m;
            gs.n = n;
            gs.p = p;
            gs.cond = cond;
            gs.seed = seed;
            gs.distribution = dist ? sv_distribution::arithmetic : sv_distribution::geometric;
            auto pb = gen_gls_problem(gs);
            put(pb.W.data(), W);
            put(pb.V.data(), V);
            put(pb.d, d);
        },
        nullptr);
}

int orc_lse_residuals(int64_t m, int64_t n, int64_t p, const double* A, const double* B,
                      const double* b, const double* d, const double* x, const double* r,
                      const double* v, int ur, double* f1, double* f2, double* f3) {
    return guarded(
        [&] {
            auto pb = make_lse(m, n, p, A, B, b, d);
            lse_state st{to_vec(x, n), to_vec(r, m), to_vec(v, p)};
            auto f = lse_residuals(pb, st, lvl(ur));
            put(f.f1, f1);
            put(f.f2, f2);
            put(f.f3, f3);
        },
        nullptr);
}

int orc_gls_residuals(int64_t n, int64_t m, int64_t p, const double* W, const double* V,
                      const double* d, const double* x, const double* y, const double* z,
                      int ur, double* f1, double* f2, double* f3) {
    return guarded(
        [&] {
            auto pb = make_gls(n, m, p, W, V, d);
            gls_state st{to_vec(x, m), to_vec(y, p), to_vec(z, n)};
            auto f = gls_residuals(pb, st, lvl(ur));
            put(f.f1, f1);
            put(f.f2, f2);
            put(f.f3, f3);
        },
        nullptr);
}

int orc_lse_correction(int64_t m, int64_t n, int64_t p, const double* A, const double* B,
                       const double* f1, const double* f2, const double* f3, int uf,
                       double* dr, double* dv, double* dx, int64_t* sing) {
    return guarded(
        [&] {
            auto Am = to_mat(A, m, n), Bm = to_mat(B, p, n);
            auto g1 = to_vec(f1, m), g2 = to_vec(f2, p), g3 = to_vec(f3, n);
            if (uf == 0) {
                auto F = grq(cast_matrix<float>(Bm), cast_matrix<float>(Am));
                auto c = lse_correction_solve(F, cast_vector<float>(g1), cast_vector<float>(g2),
                                              cast_vector<float>(g3));
                put(cast_vector<double>(c.dr), dr);
                put(cast_vector<double>(c.dv), dv);
                put(cast_vector<double>(c.dx), dx);
            } else {
                auto F = grq(Bm, Am);
                auto c = lse_correction_solve(F, g1, g2, g3);
                put(c.dr, dr);
                put(c.dv, dv);
                put(c.dx, dx);
            }
        },
        sing);
}

int orc_gls_correction(int64_t n, int64_t m, int64_t p, const double* W, const double* V,
                       const double* f1, const double* f2, const double* f3, int uf,
                       double* dy, double* dz, double* dx, int64_t* sing) {
    return guarded(
        [&] {
            auto Wm = to_mat(W, n, m), Vm = to_mat(V, n, p);
            auto g1 = to_vec(f1, p), g2 = to_vec(f2, n), g3 = to_vec(f3, m);
            if (uf == 0) {
                auto F = gqr(cast_matrix<float>(Wm), cast_matrix<float>(Vm));
                auto c = gls_correction_solve(F, cast_vector<float>(g1), cast_vector<float>(g2),
                                              cast_vector<float>(g3));
                put(cast_vector<double>(c.dy), dy);
                put(cast_vector<double>(c.dz), dz);
                put(cast_vector<double>(c.dx), dx);
            } else {
                auto F = gqr(Wm, Vm);
                auto c = gls_correction_solve(F, g1, g2, g3);
                put(c.dy, dy);
                put(c.dz, dz);
                put(c.dx, dx);
            }
        },
        sing);
}

int orc_lse_direct(int64_t m, int64_t n, int64_t p, const double* A, const double* B,
                   const double* b, const double* d, double* x, double* r, double* v,
                   int64_t* sing) {
    return guarded(
        [&] {
            auto pb = make_lse(m, n, p, A, B, b, d);
            auto F = grq(pb.B, pb.A);
            auto st = lse_direct(F, pb.b, pb.d);
            put(st.x, x);
            put(st.r, r);
            put(st.v, v);
        },
        sing);
}

int orc_gls_direct(int64_t n, int64_t m, int64_t p, const double* W, const double* V,
                   const double* d, double* x, double* y, double* z, int64_t* sing) {
    return guarded(
        [&] {
            auto pb = make_gls(n, m, p, W, V, d);
            auto F = gqr(pb.W, pb.V);
            auto st = gls_direct(F, pb.d);
            put(st.x, x);
            put(st.y, y);
            put(st.z, z);
        },
        sing);
}

double orc_extended_dot(int64_t n, const double* x, const double* y) {
    return extended_dot(x, y, static_cast<std::size_t>(n));
}

int orc_trsv(int64_t n, const double* T, const double* rhs, int transpose, double* x,
             int64_t* sing) {
    return guarded(
        [&] {
            auto M = to_mat(T, n, n);
            put(trsv(M, to_vec(rhs, n), transpose != 0), x);
        },
        sing);
}

}  // extern "C"
