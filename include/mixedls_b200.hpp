// mixedls_b200.hpp -- header-only C++ shim that makes libmixedls_b200.so a
// drop-in for the reference's classical-IR entry points:
//
//   #include <mixedls/lse.hpp>        // the reference (inc/lse.hpp, inc/gls.hpp)
//   #include <mixedls/gls.hpp>
//   #include "mixedls_b200.hpp"       // this shim (include order matters)
//
//   auto res = mixedls::b200::mplse(pb, cfg);   // instead of mixedls::mplse(pb, cfg)
//   auto res = mixedls::b200::mpgls(pb, cfg);   // instead of mixedls::mpgls(pb, cfg)
//   (with MIXEDLS_B200_KRYLOV and <mixedls/krylov.hpp>: gmres_refine_lse / _gls too)
//
// Same argument and result types (lse_problem / gls_problem /
// refinement_config -> mplse_result / mpgls_result, inc/lse.hpp:294-303,
// inc/gls.hpp:268-276) and the same exception types for the same conditions
// (inc/errors.hpp:14-49): dimension_error, invalid_input, singular_triangular
// carrying the pivot index.  trace.timing holds device-measured phases.
// Link with -lmixedls_b200 (paper_2406_16499_b200/lib).
#pragma once

#include <cstring>
#include <string>
#include <vector>

#include "mixedls_b200.h"

namespace mixedls {
namespace b200 {

namespace detail {

inline int32_t level(precision_level p) {
  if (p == precision_level::low()) return MLSB_LOW;
  if (p == precision_level::extended()) return MLSB_EXTENDED;
  return MLSB_WORKING;
}

inline mlsb_config to_c(const refinement_config& cfg) {
  mlsb_config c = mlsb_default_config();
  c.tol = cfg.tol;
  c.maxit = static_cast<int64_t>(cfg.maxit);
  c.u_f = level(cfg.precisions.factor);
  c.u_s = level(cfg.precisions.solve);
  c.u = level(cfg.precisions.working);
  c.u_r = level(cfg.precisions.residual);
  return c;
}

inline void throw_for(int rc, int64_t sing) {
  if (rc == MLSB_OK) return;
  const std::string msg = mlsb_last_error();
  if (rc == MLSB_ERR_DIMENSION) throw dimension_error(msg);
  if (rc == MLSB_ERR_INVALID_INPUT) throw invalid_input(msg);
  if (rc == MLSB_ERR_SINGULAR) throw singular_triangular("trsv: zero pivot", static_cast<std::size_t>(sing));
  throw error(msg);
}

inline void fill_trace(refinement_trace& t, const mlsb_trace& c, const std::vector<double>& hist) {
  t.status = c.status == MLSB_CONVERGED   ? refine_status::converged
             : c.status == MLSB_DIVERGED ? refine_status::diverged
                                         : refine_status::max_iterations;
  t.iterations = static_cast<std::size_t>(c.iterations);
  t.inner_iterations = 0;
  t.residual_history.clear();
  for (int64_t i = 0; i < c.iterations; ++i)
    t.residual_history.push_back(residual_norms{hist[3 * i], hist[3 * i + 1], hist[3 * i + 2]});
  t.timing.factorization = c.phase_seconds[0];
  t.timing.init = c.phase_seconds[1];
  t.timing.residual = c.phase_seconds[2];
  t.timing.correction = c.phase_seconds[3];
  t.timing.gmres = c.phase_seconds[4];
  t.timing.other = c.phase_seconds[5];
}

}  // namespace detail

// GPU drop-in for mixedls::mplse (inc/lse.hpp:303)
inline mplse_result mplse(const lse_problem& pb, const refinement_config& cfg) {
  pb.validate();  // the reference's own checks, same exceptions, same order
  cfg.validate();
  const auto m = static_cast<int64_t>(pb.m()), n = static_cast<int64_t>(pb.n()),
             p = static_cast<int64_t>(pb.p());
  mplse_result out;
  out.state.x.assign(n, 0.0);
  out.state.r.assign(m, 0.0);
  out.state.v.assign(p, 0.0);
  std::vector<double> hist(3 * cfg.maxit);
  mlsb_trace tr{};
  tr.residual_history = hist.data();
  int64_t sing = -1;
  const mlsb_config c = detail::to_c(cfg);
  const int rc = mlsb_mplse(pb.A.data().data(), m, pb.B.data().data(), p, pb.b.data(), pb.d.data(), m,
                            n, p, &c, out.state.x.data(), out.state.r.data(), out.state.v.data(), &tr,
                            &sing, nullptr);
  detail::throw_for(rc, sing);
  detail::fill_trace(out.trace, tr, hist);
  return out;
}

// GPU drop-in for mixedls::mpgls (inc/gls.hpp:276)
inline mpgls_result mpgls(const gls_problem& pb, const refinement_config& cfg) {
  pb.validate();
  cfg.validate();
  const auto n = static_cast<int64_t>(pb.n()), m = static_cast<int64_t>(pb.m()),
             p = static_cast<int64_t>(pb.p());
  mpgls_result out;
  out.state.x.assign(m, 0.0);
  out.state.y.assign(p, 0.0);
  out.state.z.assign(n, 0.0);
  std::vector<double> hist(3 * cfg.maxit);
  mlsb_trace tr{};
  tr.residual_history = hist.data();
  int64_t sing = -1;
  const mlsb_config c = detail::to_c(cfg);
  const int rc = mlsb_mpgls(pb.W.data().data(), n, pb.V.data().data(), n, pb.d.data(), n, m, p, &c,
                            out.state.x.data(), out.state.y.data(), out.state.z.data(), &tr, &sing,
                            nullptr);
  detail::throw_for(rc, sing);
  detail::fill_trace(out.trace, tr, hist);
  return out;
}

// GPU drop-in for detail::lse_direct_reference (inc/experiment.hpp:50-59):
// binary64 factorization + direct solve, the err-2 reference
inline lse_state lse_direct_reference(const lse_problem& pb) {
  pb.validate();
  const auto m = static_cast<int64_t>(pb.m()), n = static_cast<int64_t>(pb.n()),
             p = static_cast<int64_t>(pb.p());
  lse_state st;
  st.x.assign(n, 0.0);
  st.r.assign(m, 0.0);
  st.v.assign(p, 0.0);
  int64_t sing = -1;
  const int rc = mlsb_lse_direct(pb.A.data().data(), m, pb.B.data().data(), p, pb.b.data(),
                                 pb.d.data(), m, n, p, st.x.data(), st.r.data(), st.v.data(), &sing,
                                 nullptr);
  detail::throw_for(rc, sing);
  return st;
}

// GPU drop-in for detail::gls_direct_reference (inc/experiment.hpp:65-73)
inline gls_state gls_direct_reference(const gls_problem& pb) {
  pb.validate();
  const auto n = static_cast<int64_t>(pb.n()), m = static_cast<int64_t>(pb.m()),
             p = static_cast<int64_t>(pb.p());
  gls_state st;
  st.x.assign(m, 0.0);
  st.y.assign(p, 0.0);
  st.z.assign(n, 0.0);
  int64_t sing = -1;
  const int rc = mlsb_gls_direct(pb.W.data().data(), n, pb.V.data().data(), n, pb.d.data(), n, m,
                                 p, st.x.data(), st.y.data(), st.z.data(), &sing, nullptr);
  detail::throw_for(rc, sing);
  return st;
}

#ifdef MIXEDLS_B200_KRYLOV
// GPU drop-ins for mixedls::gmres_refine_lse / gmres_refine_gls
// (inc/krylov.hpp:545, :673).  Define MIXEDLS_B200_KRYLOV and include
// <mixedls/krylov.hpp> before this header.
inline mplse_result gmres_refine_lse(const lse_problem& pb, const refinement_config& cfg,
                                     precond_choice choice = precond_choice::bd_split,
                                     double alpha_scale = 1.0) {
  pb.validate();
  cfg.validate();
  const auto m = static_cast<int64_t>(pb.m()), n = static_cast<int64_t>(pb.n()),
             p = static_cast<int64_t>(pb.p());
  mplse_result out;
  out.state.x.assign(n, 0.0);
  out.state.r.assign(m, 0.0);
  out.state.v.assign(p, 0.0);
  std::vector<double> hist(3 * cfg.maxit);
  mlsb_trace tr{};
  tr.residual_history = hist.data();
  int64_t sing = -1;
  const mlsb_config c = detail::to_c(cfg);
  const int rc = mlsb_gmres_lse(pb.A.data().data(), m, pb.B.data().data(), p, pb.b.data(), pb.d.data(),
                                m, n, p, &c,
                                choice == precond_choice::left ? MLSB_PRECOND_LEFT : MLSB_PRECOND_BD_SPLIT,
                                alpha_scale, out.state.x.data(), out.state.r.data(), out.state.v.data(), &tr,
                                &sing, nullptr);
  detail::throw_for(rc, sing);
  detail::fill_trace(out.trace, tr, hist);
  out.trace.inner_iterations = static_cast<std::size_t>(tr.inner_iterations);
  return out;
}

inline mpgls_result gmres_refine_gls(const gls_problem& pb, const refinement_config& cfg,
                                     precond_choice choice = precond_choice::bd_split,
                                     double alpha_scale = 1.0) {
  pb.validate();
  cfg.validate();
  const auto n = static_cast<int64_t>(pb.n()), m = static_cast<int64_t>(pb.m()),
             p = static_cast<int64_t>(pb.p());
  mpgls_result out;
  out.state.x.assign(m, 0.0);
  out.state.y.assign(p, 0.0);
  out.state.z.assign(n, 0.0);
  std::vector<double> hist(3 * cfg.maxit);
  mlsb_trace tr{};
  tr.residual_history = hist.data();
  int64_t sing = -1;
  const mlsb_config c = detail::to_c(cfg);
  const int rc = mlsb_gmres_gls(pb.W.data().data(), n, pb.V.data().data(), n, pb.d.data(), n, m, p, &c,
                                choice == precond_choice::left ? MLSB_PRECOND_LEFT : MLSB_PRECOND_BD_SPLIT,
                                alpha_scale, out.state.x.data(), out.state.y.data(), out.state.z.data(), &tr,
                                &sing, nullptr);
  detail::throw_for(rc, sing);
  detail::fill_trace(out.trace, tr, hist);
  out.trace.inner_iterations = static_cast<std::size_t>(tr.inner_iterations);
  return out;
}
#endif  // MIXEDLS_B200_KRYLOV

}  // namespace b200
}  // namespace mixedls
