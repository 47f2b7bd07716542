// Drop-in demonstration: the SAME reference problem solved by the reference
// (mixedls::mplse / mpgls, CPU) and by the B200 library through the shim
// (mixedls::b200::mplse / mpgls).  Built by `make -C oracle demo` against the
// unmodified reference headers; run by tests/test_gpu_dropin.py.
#include <cmath>
#include <cstdio>

#include "mixedls/experiment.hpp"
#include "mixedls/generate.hpp"
#include "mixedls/gls.hpp"
#include "mixedls/krylov.hpp"
#include "mixedls/lse.hpp"
#define MIXEDLS_B200_KRYLOV
#include "mixedls_b200.hpp"

using namespace mixedls;

static double reldiff(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return std::sqrt(num / den);
}

int main() {
  generator_spec gs;
  gs.kind = problem_kind::lse;
  gs.m = 200;
  gs.n = 100;
  gs.p = 50;
  gs.cond = 1e3;
  gs.seed = 7;
  auto pb = gen_lse_problem(gs);
  refinement_config cfg;
  auto ref = mplse(pb, cfg);
  auto gpu = b200::mplse(pb, cfg);
  std::printf("LSE ref_iters %zu gpu_iters %zu ref_status %s gpu_status %s relx %.3e\n",
              ref.trace.iterations, gpu.trace.iterations, to_string(ref.trace.status),
              to_string(gpu.trace.status), reldiff(gpu.state.x, ref.state.x));
  generator_spec gg;
  gg.kind = problem_kind::gls;
  gg.n = 200;
  gg.m = 100;
  gg.p = 150;
  gg.cond = 1e3;
  gg.seed = 2;
  auto pg = gen_gls_problem(gg);
  auto refg = mpgls(pg, cfg);
  auto gpug = b200::mpgls(pg, cfg);
  std::printf("GLS ref_iters %zu gpu_iters %zu ref_status %s gpu_status %s relx %.3e rely %.3e\n",
              refg.trace.iterations, gpug.trace.iterations, to_string(refg.trace.status),
              to_string(gpug.trace.status), reldiff(gpug.state.x, refg.state.x),
              reldiff(gpug.state.y, refg.state.y));
  // binary64 direct reference (experiment harness err-2 denominator)
  auto dref = detail::lse_direct_reference(pb).state;
  auto dgpu = b200::lse_direct_reference(pb);
  std::printf("DIRECT relx %.3e relr %.3e\n", reldiff(dgpu.x, dref.x), reldiff(dgpu.r, dref.r));
  // GMRES-IR drop-ins (krylov.hpp:545, :673), both preconditioners
  for (precond_choice pc : {precond_choice::bd_split, precond_choice::left}) {
    auto rg = gmres_refine_lse(pb, cfg, pc);
    auto gg2 = b200::gmres_refine_lse(pb, cfg, pc);
    std::printf("GMRES-LSE %d ref_iters %zu gpu_iters %zu ref_status %s gpu_status %s relx %.3e\n", int(pc),
                rg.trace.iterations, gg2.trace.iterations, to_string(rg.trace.status),
                to_string(gg2.trace.status), reldiff(gg2.state.x, rg.state.x));
    auto rgl = gmres_refine_gls(pg, cfg, pc);
    auto ggl = b200::gmres_refine_gls(pg, cfg, pc);
    std::printf("GMRES-GLS %d ref_iters %zu gpu_iters %zu ref_status %s gpu_status %s relx %.3e\n", int(pc),
                rgl.trace.iterations, ggl.trace.iterations, to_string(rgl.trace.status),
                to_string(ggl.trace.status), reldiff(ggl.state.x, rgl.state.x));
  }
  // exception parity: the reference's validation is reused verbatim
  lse_problem bad = pb;
  bad.d.pop_back();
  try {
    b200::mplse(bad, cfg);
    std::printf("EXC none\n");
  } catch (const dimension_error&) {
    std::printf("EXC dimension_error\n");
  }
  return 0;
}
