// si_dispatch.cu — picks the block shape (K cells per thread, NT threads per CTA) and the cluster
// size (CS CTAs per instance) of K1/K2 for a launch.
#include <algorithm>
#include <cstdlib>

#define SNOP_PHASE_SYM g_phase_cycles_disp
#include "si_kernels.cuh"

namespace snop_si {
SNOP_DECL_SI(SNOP_K, 32, false) SNOP_DECL_SI(SNOP_K, 64, false) SNOP_DECL_SI(SNOP_K, 128, false) SNOP_DECL_SI(SNOP_K, 256, false)
SNOP_DECL_SI(SNOP_K, 512, false)
SNOP_DECL_SI(SNOP_K, 32, true) SNOP_DECL_SI(SNOP_K, 64, true) SNOP_DECL_SI(SNOP_K, 128, true) SNOP_DECL_SI(SNOP_K, 256, true)
SNOP_DECL_PI(SNOP_K, 32, false) SNOP_DECL_PI(SNOP_K, 64, false) SNOP_DECL_PI(SNOP_K, 128, false) SNOP_DECL_PI(SNOP_K, 256, false)
SNOP_DECL_PI(SNOP_K, 512, false)
SNOP_DECL_PI(SNOP_K, 32, true) SNOP_DECL_PI(SNOP_K, 64, true) SNOP_DECL_PI(SNOP_K, 128, true) SNOP_DECL_PI(SNOP_K, 256, true)
SNOP_DECL_PS(SNOP_K, 32) SNOP_DECL_PS(SNOP_K, 64) SNOP_DECL_PS(SNOP_K, 128) SNOP_DECL_PS(SNOP_K, 256) SNOP_DECL_PS(SNOP_K, 512)
extern template snop_status launch_tiled_t<SNOP_K, 256>(snop_impl::Ctx&, const SweepConsts&, const SolveConfig&, int,
                                                        const double*, const double*, const double*, const double*,
                                                        const double*, double*, double*, int32_t*, uint8_t*, double*,
                                                        const uint8_t*);
}  // namespace snop_si

using namespace snop_si;

namespace {

constexpr int K = SNOP_K;  // cells per thread (experiments: -DSNOP_K=4)

int pow2_at_least(int v, int lo) {
  int p = lo;
  while (p < v) p <<= 1;
  return p;
}

struct Shape {
  int cs, nt;
};

// Cluster size: one CTA per instance whenever the slab fits one CTA (<= 4096 cells). Spreading an
// instance over a thread-block cluster (cells split across SMs, joined through DSMEM) is correct
// but measured slower on every BASELINE config (C2-C5, DESIGN.md §K1 "clusters"): the
// per-pair-group cluster barrier costs more than the split saves. Above 4096 cells the smallest
// cluster that holds the slab is used (up to 8 CTAs x 256 threads x K cells = 16384 cells).
// ctx.opt.cell_cluster = 1 / 2 / 4 / 8 forces a size (1 = never split). Beyond the cluster limit,
// or with ctx.opt.cell_cluster = -1, the streaming kernel (si_tiled.cu) sweeps the slab in tiles.
Shape pick_shape(const snop_impl::Ctx& ctx, int n_cells) {
  int cs = 1;
  const int force = ctx.opt.cell_cluster;
  if (force == 2 || force == 4 || force == 8) cs = force;
  int nt = pow2_at_least(((n_cells + cs - 1) / cs + K - 1) / K, 32);
  if (force != 1 && (nt > 512 || (cs > 1 && nt > 256))) {  // clusters are instantiated up to NT = 256
    if (cs == 1) cs = 2;
    nt = pow2_at_least(((n_cells + cs - 1) / cs + K - 1) / K, 32);
    while (cs < 8 && nt > 256) {
      cs <<= 1;
      nt = pow2_at_least(((n_cells + cs - 1) / cs + K - 1) / K, 32);
    }
  }
  return {cs, nt};
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
                                    int32_t* iters, uint8_t* conv, double* leak, double* stage,
                                    const uint8_t* active) {
  if (batch == 0) return SNOP_OK;
  const SweepConsts sc = make_consts(g, order);
  const SolveConfig c = inner_cfg(cfg);
  if (ctx.opt.cell_cluster == -1 || g.n_cells > kMaxCells) {
    if (stage) {
      set_error("host-resident inputs need the one-CTA-per-instance kernel");
      return SNOP_INVALID_ARGUMENT;
    }
    return launch_tiled_t<K, 256>(ctx, sc, c, batch, st, ss0, ss1, src, phi0, phi, cur, iters, conv, leak, active);
  }
  const Shape s = pick_shape(ctx, g.n_cells);
  if (stage && s.cs > 1) {
    set_error("host-resident inputs need the one-CTA-per-instance kernel");
    return SNOP_INVALID_ARGUMENT;
  }
#define SNOP_SI(NN, CC)                       \
  if (s.nt == NN && (s.cs > 1) == CC)         \
    return launch_si_t<K, NN, CC>(ctx, sc, c, batch, s.cs, st, ss0, ss1, src, phi0, phi, cur, iters, conv, leak, \
                                  stage, active);
  SNOP_SI(32, false) SNOP_SI(64, false) SNOP_SI(128, false) SNOP_SI(256, false) SNOP_SI(512, false)
  SNOP_SI(32, true) SNOP_SI(64, true) SNOP_SI(128, true) SNOP_SI(256, true)
#undef SNOP_SI
  set_error("n_cells exceeds the cluster sweep limit (16384 per instance)");
  return SNOP_INVALID_ARGUMENT;
}

snop_status launch_power_iteration(Ctx& ctx, const snop_grid& g, int order, int batch, int G, const double* st,
                                   const double* ss0, const double* ss1, const double* nsf, const double* chi,
                                   const snop_solver_config& cfg, const double* k0, const double* phi0, double* k,
                                   double* phi, double* old, int32_t* outer, int64_t* inner, uint8_t* conv) {
  if (batch == 0) return SNOP_OK;
  if (ctx.opt.cell_cluster == -1 || g.n_cells > kMaxCells)  // streaming inner solves, device outer loop
    return launch_power_iteration_big(ctx, g, order, batch, G, st, ss0, ss1, nsf, chi, cfg, k0, phi0, k, phi, outer,
                                      inner, conv);
  const SweepConsts sc = make_consts(g, order);
  const SolveConfig ic = inner_cfg(cfg);
  EigenParams ep;
  ep.G = G;
  ep.tol_k = cfg.tolerance_k;
  ep.tol_phi = cfg.tolerance_phi;
  ep.max_outer = cfg.max_outer;
  ep.norm = cfg.norm;
  const Shape s = pick_shape(ctx, g.n_cells);
  // Pair-split clusters (si_solve PS): a single-group eigen solve is one long chain of dependent
  // sweeps and a batch finishes with its slowest instance, so the sweep of one instance is spread
  // over cs CTAs (measured on C3, slowest instance alone: 320 ms on one CTA, 153 ms at cs = 4,
  // 125 ms at cs = 8). cs = 8 for the tail phase below; without it the whole batch runs at cs = 4
  // (361 -> 275 ms; at cs = 8 the batch becomes throughput-bound). Multigroup solves spend their time in the outer
  // loop, which every CTA of a cluster repeats, so they stay on one CTA (C4: 37 vs 49 ms). The
  // rule depends on (G, order) only, never on the batch, so an instance's result does not depend
  // on what it is batched with. ctx.opt.pair_split = -1 disables it, n sets the cluster size (<= 8).
  const int cap = ctx.opt.pi_tail_cap == 0 ? 12 : (ctx.opt.pi_tail_cap < 0 ? 0 : ctx.opt.pi_tail_cap);  // tail split
  int ps = 0;
  if (!ss1 && s.cs == 1) {
    int want = G == 1 ? (cap > 0 ? 8 : 4) : 0;
    if (ctx.opt.pair_split != 0) want = ctx.opt.pair_split < 0 ? 0 : ctx.opt.pair_split;
    ps = std::min(std::min(want, 8), (order / 2) / 2);
    if (ps < 2 || (s.nt % ps) != 0) ps = 0;
  }
  // Tail split (single-group, pair-split eligible): a batch of eigen solves ends with its few
  // longest instances (C3: outer counts 17 ... 1303), and the batch time is the slowest instance's
  // chain of sweeps. Phase 1 runs every instance on one CTA for `cap` outers and predicts each
  // one's remaining outers from its own convergence rate (gap ratio over its last 4 outers). Then,
  // concurrently: the predicted-long instances (> kLongOuters) continue on pair-split clusters to
  // the end (main stream, longest first); the others continue on single CTAs for up to kMidOuters
  // outers (aux stream) and whatever is still iterating after that finishes on clusters. Routing
  // depends on an instance's own data only (constant cap and threshold), so results never depend on
  // the batch. ctx.opt.pi_tail_cap sets the phase-1 cap (default 12; -1 disables the split).
  constexpr float kLongOuters = 256.f;
  constexpr int kMidOuters = 32;
  if (ps && cap > 0 && cfg.max_outer > cap) {
    EigenParams e1 = ep, e2 = ep, em = ep, e3 = ep;
    e1.max_outer = cap;
    e2.max_outer = cfg.max_outer - cap;
    em.max_outer = std::min(kMidOuters, cfg.max_outer - cap);
    e3.max_outer = cfg.max_outer - cap - em.max_outer;
    int* lst = static_cast<int*>(ctx.slot(25, (3 * (size_t)batch + 4) * sizeof(int)));
    float* key = static_cast<float*>(ctx.slot(26, (size_t)batch * sizeof(float)));
    if (!lst || !key) {
      set_error("cudaMalloc (tail list) failed");
      return SNOP_CUDA_ERROR;
    }
    if (!ctx.aux) {
      if (cudaStreamCreateWithFlags(&ctx.aux, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&ctx.ev_fork, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&ctx.ev_join, cudaEventDisableTiming) != cudaSuccess) {
        set_error("tail split: stream / event creation failed");
        return SNOP_CUDA_ERROR;
      }
    }
    int *lA = lst, *lB = lst + batch, *lC = lst + 2 * (size_t)batch, *cnt = lst + 3 * (size_t)batch;
    snop_status st1 = SNOP_INVALID_ARGUMENT, st2 = SNOP_OK, stm = SNOP_OK, st3 = SNOP_OK;
#define SNOP_P1(NN) \
  if (s.nt == NN) st1 = launch_pi_t<K, NN, false>(ctx, sc, ic, e1, batch, 1, st, ss0, ss1, nsf, chi, k0, phi0, k, phi, old, outer, inner, conv, nullptr, nullptr, 0, key);
#define SNOP_PSR(NN, EP, L, C, ST) \
  if (s.nt == NN) ST = launch_pi_t<K, NN, false, true>(ctx, sc, ic, EP, batch, ps, st, ss0, ss1, nsf, chi, k, phi, k, phi, old, outer, inner, conv, L, C, 1);
#define SNOP_MID(NN) \
  if (s.nt == NN) stm = launch_pi_t<K, NN, false>(ctx, sc, ic, em, batch, 1, st, ss0, ss1, nsf, chi, k, phi, k, phi, old, outer, inner, conv, lB, cnt + 1, 1, key);
    SNOP_P1(32) SNOP_P1(64) SNOP_P1(128) SNOP_P1(256) SNOP_P1(512)
    if (st1 != SNOP_OK) return st1;
    cudaMemsetAsync(cnt, 0, 4 * sizeof(int), ctx.stream);
    pi_tail_list_kernel<<<(batch + 255) / 256, 256, 0, ctx.stream>>>(batch, cap, outer, conv, key, kLongOuters, lA,
                                                                     cnt, lB, cnt + 1);
    ctx.launches++;
    cudaEventRecord(ctx.ev_fork, ctx.stream);
    // main stream: the predicted-long instances on clusters, launched first so their clusters are
    // placed before the single-CTA work of the aux stream fills the SMs
    SNOP_PSR(32, e2, lA, cnt, st2) SNOP_PSR(64, e2, lA, cnt, st2) SNOP_PSR(128, e2, lA, cnt, st2)
    SNOP_PSR(256, e2, lA, cnt, st2) SNOP_PSR(512, e2, lA, cnt, st2)
    // aux stream: the rest on single CTAs, then the still-iterating ones on clusters
    const cudaStream_t main_stream = ctx.stream;
    cudaStreamWaitEvent(ctx.aux, ctx.ev_fork, 0);
    ctx.stream = ctx.aux;
    SNOP_MID(32) SNOP_MID(64) SNOP_MID(128) SNOP_MID(256) SNOP_MID(512)
    if (stm == SNOP_OK && e3.max_outer > 0) {
      pi_tail_list_kernel<<<(batch + 255) / 256, 256, 0, ctx.stream>>>(batch, cap + em.max_outer, outer, conv, key,
                                                                       0.f, lC, cnt + 2, nullptr, nullptr, lB,
                                                                       cnt + 1);
      ctx.launches++;
      SNOP_PSR(32, e3, lC, cnt + 2, st3) SNOP_PSR(64, e3, lC, cnt + 2, st3) SNOP_PSR(128, e3, lC, cnt + 2, st3)
      SNOP_PSR(256, e3, lC, cnt + 2, st3) SNOP_PSR(512, e3, lC, cnt + 2, st3)
    }
    cudaEventRecord(ctx.ev_join, ctx.stream);
    ctx.stream = main_stream;
    cudaStreamWaitEvent(ctx.stream, ctx.ev_join, 0);
#undef SNOP_P1
#undef SNOP_PSR
#undef SNOP_MID
    if (st2 != SNOP_OK) return st2;
    if (stm != SNOP_OK) return stm;
    return st3;
  }
  if (ps) {
#define SNOP_PS(NN) \
  if (s.nt == NN)   \
    return launch_pi_t<K, NN, false, true>(ctx, sc, ic, ep, batch, ps, st, ss0, ss1, nsf, chi, k0, phi0, k, phi, old, outer, inner, conv);
    SNOP_PS(32) SNOP_PS(64) SNOP_PS(128) SNOP_PS(256) SNOP_PS(512)
#undef SNOP_PS
  }
#define SNOP_PI(NN, CC)               \
  if (s.nt == NN && (s.cs > 1) == CC) \
    return launch_pi_t<K, NN, CC>(ctx, sc, ic, ep, batch, s.cs, st, ss0, ss1, nsf, chi, k0, phi0, k, phi, old, outer, inner, conv);
  SNOP_PI(32, false) SNOP_PI(64, false) SNOP_PI(128, false) SNOP_PI(256, false) SNOP_PI(512, false)
  SNOP_PI(32, true) SNOP_PI(64, true) SNOP_PI(128, true) SNOP_PI(256, true)
#undef SNOP_PI
  set_error("n_cells exceeds the cluster sweep limit (16384 per instance)");
  return SNOP_INVALID_ARGUMENT;
}

}  // namespace snop_impl


#ifdef SNOP_PHASE_TIMING
// nvcc also emits the kernel templates referenced from this TU; the runtime may launch that copy
extern "C" int snop_internal_phase_cycles_disp(unsigned long long* out /* [2][10] */, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, snop_dev::g_phase_cycles_disp, sizeof(unsigned long long) * 20);
  if (reset) {
    unsigned long long z[20] = {};
    cudaMemcpyToSymbol(snop_dev::g_phase_cycles_disp, z, sizeof(z));
  }
  return (int)e;
}
#endif

