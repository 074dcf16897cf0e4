// si_dispatch.cu — picks the (K, NT) instantiation of K1/K2 for a launch.
#include <cstdlib>

#include "si_kernels.cuh"

using namespace snop_si;

namespace snop_si {
SNOP_DECL_SI(8, 32) SNOP_DECL_SI(8, 64) SNOP_DECL_SI(8, 128) SNOP_DECL_SI(8, 256) SNOP_DECL_SI(8, 512)
SNOP_DECL_SI(16, 32) SNOP_DECL_SI(16, 64) SNOP_DECL_SI(16, 128) SNOP_DECL_SI(16, 256)
SNOP_DECL_PI(8, 32) SNOP_DECL_PI(8, 64) SNOP_DECL_PI(8, 128) SNOP_DECL_PI(8, 256) SNOP_DECL_PI(8, 512)
SNOP_DECL_PI(16, 32) SNOP_DECL_PI(16, 64) SNOP_DECL_PI(16, 128) SNOP_DECL_PI(16, 256)
}  // namespace snop_si

namespace {

// Block shape: K cells per thread (compile-time, register arrays), NT = smallest power of two
// >= ceil(Nc/K), NT >= 32. K = 8 by default (measured fastest on C2-C5); SNOP_CELLS_PER_THREAD=16 selects K = 16.
int pick_k() {
  static const int k = [] {
    const char* e = std::getenv("SNOP_CELLS_PER_THREAD");
    return (e && std::atoi(e) == 16) ? 16 : 8;
  }();
  return k;
}

int pick_nt(int n_cells, int K) {
  const int need = (n_cells + K - 1) / K;
  int nt = 32;
  while (nt < need) nt <<= 1;
  return nt;
}

SolveConfig inner_cfg(const snop_solver_config& c) {
  SolveConfig s;
  s.tol = c.tolerance;
  s.max_it = c.max_inner;
  s.bc_left = c.bc_left;
  s.bc_right = c.bc_right;
  s.norm = c.norm;
  return s;
}

}  // namespace

namespace snop_impl {

snop_status launch_source_iteration(Ctx& ctx, const snop_grid& g, int order, int batch, const double* st,
                                    const double* ss0, const double* ss1, const double* src,
                                    const snop_solver_config& cfg, const double* phi0, double* phi, double* cur,
                                    int32_t* iters, uint8_t* conv) {
  if (batch == 0) return SNOP_OK;
  const SweepConsts sc = make_consts(g, order);
  const SolveConfig c = inner_cfg(cfg);
  const int K = pick_k();
#define SNOP_SI(KK, NN) \
  if (K == KK && pick_nt(g.n_cells, KK) == NN) \
    return launch_si_t<KK, NN>(ctx, sc, c, batch, st, ss0, ss1, src, phi0, phi, cur, iters, conv);
  SNOP_SI(8, 32) SNOP_SI(8, 64) SNOP_SI(8, 128) SNOP_SI(8, 256) SNOP_SI(8, 512)
  SNOP_SI(16, 32) SNOP_SI(16, 64) SNOP_SI(16, 128) SNOP_SI(16, 256)

#undef SNOP_SI
  {
      set_error("n_cells exceeds the per-CTA register-resident sweep limit (4096)");
      return SNOP_INVALID_ARGUMENT;
  }
}

snop_status launch_power_iteration(Ctx& ctx, const snop_grid& g, int order, int batch, int G, const double* st,
                                   const double* ss0, const double* ss1, const double* nsf, const double* chi,
                                   const snop_solver_config& cfg, const double* k0, const double* phi0, double* k,
                                   double* phi, double* old, int32_t* outer, int64_t* inner, uint8_t* conv) {
  if (batch == 0) return SNOP_OK;
  const SweepConsts sc = make_consts(g, order);
  const SolveConfig ic = inner_cfg(cfg);
  EigenParams ep;
  ep.G = G;
  ep.tol_k = cfg.tolerance_k;
  ep.tol_phi = cfg.tolerance_phi;
  ep.max_outer = cfg.max_outer;
  ep.norm = cfg.norm;
  const int K = pick_k();
#define SNOP_PI(KK, NN) \
  if (K == KK && pick_nt(g.n_cells, KK) == NN) \
    return launch_pi_t<KK, NN>(ctx, sc, ic, ep, batch, st, ss0, ss1, nsf, chi, k0, phi0, k, phi, old, outer, inner, conv);
  SNOP_PI(8, 32) SNOP_PI(8, 64) SNOP_PI(8, 128) SNOP_PI(8, 256) SNOP_PI(8, 512)
  SNOP_PI(16, 32) SNOP_PI(16, 64) SNOP_PI(16, 128) SNOP_PI(16, 256)

#undef SNOP_PI
  {
      set_error("n_cells exceeds the per-CTA register-resident sweep limit (4096)");
      return SNOP_INVALID_ARGUMENT;
  }
}

}  // namespace snop_impl
