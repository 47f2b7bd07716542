// The reference's own experiment harness -- the UNMODIFIED inc/experiment.hpp
// (run_experiment :80-160, run_sweep :132-159, paper_sweep_cells :161-198) --
// with its classical-IR and GMRES-IR calls routed to the B200 library by the
// compile-time switch of INTEGRATION.md ("Patch a maintainer would add"),
// applied here at the include site instead of inside the header:
//
//   every header experiment.hpp needs is included first (unaffected), then
//   mplse / mpgls / gmres_refine_lse / gmres_refine_gls are #defined to the
//   mixedls::b200 drop-ins for the one remaining header, experiment.hpp.
//
// Built twice by oracle/Makefile (target `harness`): with -DROUTE_B200 and
// linked to libmixedls_b200.so (oracle/_ref/b200_harness), and without (the
// plain reference, oracle/_ref/ref_harness).  tests/test_gpu_dropin.py runs
// both on the reference's desk-scale LSE and GLS sweeps and compares them.
#include <cstdio>
#include <cstring>
#include <string>

#include "mixedls/errors.hpp"
#include "mixedls/generate.hpp"
#include "mixedls/gls.hpp"
#include "mixedls/krylov.hpp"
#include "mixedls/lse.hpp"
#include "mixedls/metrics.hpp"

#ifdef ROUTE_B200
#define MIXEDLS_B200_KRYLOV
#include "mixedls_b200.hpp"
#define mplse ::mixedls::b200::mplse
#define mpgls ::mixedls::b200::mpgls
#define gmres_refine_lse ::mixedls::b200::gmres_refine_lse
#define gmres_refine_gls ::mixedls::b200::gmres_refine_gls
#endif
#include "mixedls/experiment.hpp"
#ifdef ROUTE_B200
#undef mplse
#undef mpgls
#undef gmres_refine_lse
#undef gmres_refine_gls
#endif

static const char* status_name(mixedls::refine_status s) {
  switch (s) {
    case mixedls::refine_status::converged: return "converged";
    case mixedls::refine_status::max_iterations: return "max_iterations";
    case mixedls::refine_status::diverged: return "diverged";
  }
  return "unknown";
}

int main(int argc, char** argv) {
  using namespace mixedls;
  const bool gls = argc > 1 && std::strcmp(argv[1], "gls") == 0;
  const auto cells = paper_sweep_cells(gls ? problem_kind::gls : problem_kind::lse, false);
  refinement_config cfg;  // reference defaults
  const auto reps = run_sweep(cells, cfg);
  for (std::size_t i = 0; i < reps.size(); ++i) {
    const auto& r = reps[i];
    std::printf("CELL %zu kind %s cond %.0e method %s status %s iters %zu inner %zu m1 %.6e m2 %.6e\n", i,
                gls ? "gls" : "lse", r.spec.cond, to_string(r.method), status_name(r.status), r.iterations,
                r.inner_iterations, r.metric1, r.metric2);
  }
  return 0;
}
