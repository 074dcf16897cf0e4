// si_tiled.cu — K1 for slabs of any length (the "streaming" path): one CTA per instance sweeps the
// slab tile by tile (a tile = NT threads x K cells), with the per-cell state (emission, scalar
// flux, edge accumulators) in a global workspace instead of shared memory. It is selected when an
// instance does not fit the shared-memory-resident kernels (more than 16384 cells, the largest
// thread-block cluster path) or when ctx.opt.cell_cluster = -1 forces it (tests).
//
// Per source iteration and pair group (SPEC.md:115-128 arithmetic, the same maps / scan / replay
// device code as the resident kernel, snop_device.cuh):
//   pass A  tile by tile: affine maps of the tile's cells, chunk compositions, the CTA scan ->
//           the tile's composed maps (forward and backward) into a small table;
//   join    one thread per pair composes the tile maps across the slab: boundary inflows
//           (vacuum / reflective, SURVEY §9 #2 ordering, both-reflective right face lagged) and
//           the inflow entering every tile in both directions;
//   pass B  tile by tile: maps and scan again, replay from the tile's inflows, edge scalar fluxes
//           (and currents for P1) added into the workspace rows (each element owned by one thread).
// Then the flux update phi_i = (Phi_{i-1/2} + Phi_{i+1/2}) / 2, the next emission and the
// convergence norm over all tiles. Results equal the resident kernel's to rounding.
#include "si_kernels.cuh"

namespace snop_si {

// Workspace doubles per instance for n_cells cells in tiles of NT*K: emission q2, edge scalar flux
// of every cell's left edge FL, right edge of every thread chunk FR, tile map table [T][NP][4],
// tile inflows [T][NP][2]; P1 adds the edge currents JL, JR.
template <int K, int NT>
__host__ __device__ inline size_t tiled_ws_doubles(int n_cells, bool aniso) {
  const size_t TC = (size_t)NT * K, T = ((size_t)n_cells + TC - 1) / TC, Np = T * TC, nch = T * NT;
  return 2 * Np + nch + T * kNP * 6 + (aniso ? Np + nch : 0);
}

// replay of one tile from given inflows (psi+ entering the tile's left edge, psi- entering its
// right edge, per pair) instead of the resident kernel's domain boundary logic
template <int K, int NT, int NP, bool WJ>
__device__ __forceinline__ void replay_tile(const SweepConsts& sc, SweepSmem<K, NT>& sm, int p0, int t,
                                            const double (&al)[NP][K], const double (&bp)[NP][K],
                                            const double (&bm)[NP][K], const double* ein, EdgeAcc<K, WJ>& acc) {
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    const int p = p0 + q;
    const double wq = sc.w[p], wm = sc.wmu[p];
    const int pt = SweepSmem<K, NT>::spos(t);
    double psi = fma(sm.xmap[q][0][pt], ein[2 * q], sm.agg[q][1][pt]);
    double psib = fma(sm.xmap[q][1][pt], ein[2 * q + 1], sm.agg[q][2][pt]);
    const double psib_in = psib;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      acc.Fl[j] = fma(wq, psi, acc.Fl[j]);
      if constexpr (WJ) acc.Jl[j] = fma(wm, psi, acc.Jl[j]);
      psi = fma(al[q][j], psi, bp[q][j]);
      psib = fma(al[q][K - 1 - j], psib, bm[q][K - 1 - j]);
      acc.Fl[K - 1 - j] = fma(wq, psib, acc.Fl[K - 1 - j]);
      if constexpr (WJ) acc.Jl[K - 1 - j] = fma(-wm, psib, acc.Jl[K - 1 - j]);
    }
    acc.Fr = fma(wq, psi + psib_in, acc.Fr);
    if constexpr (WJ) acc.Jr = fma(wm, psi - psib_in, acc.Jr);
  }
}

// One pair group (NP pairs starting at p0) of one source iteration over all tiles.
template <int K, int NT, bool ANISO, bool WJ, int NP>
__device__ void tiled_pair_group(const SweepConsts& sc, SweepSmem<K, NT>& sm, const CellIO& io, SweepCtl& w,
                                 int p0, int T, const double* __restrict__ st, const double* __restrict__ q2,
                                 double* __restrict__ FL, double* __restrict__ FR, double* __restrict__ JL,
                                 double* __restrict__ JR, double* __restrict__ tt, double* __restrict__ ein) {
  constexpr int TC = NT * K;
  const int t = w.t, Nc = sc.n_cells;
  double al[NP][K], bp[NP][K], bm[NP][K];
  auto stage = [&](int tau) {  // the tile's Sigma_t and emission into the resident layout
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int i = tau * TC + t * K + j;
      sm.st[j * NT + t] = i < Nc ? st[i] : 0.0;  // padding: identity map (see maps_phase)
      sm.q2[j * NT + t] = i < Nc ? q2[i] : 0.0;
    }
  };
  // pass A: composed maps of every tile
  for (int tau = 0; tau < T; ++tau) {
    w.cbase = tau * TC;
    stage(tau);
    maps_phase<K, NT, ANISO, NP>(sc, sm, io, p0, w, al, bp, bm);
    __syncthreads();
    scan_phase<K, NT, NP, false>(sm, w.lane, w.warp, 0);
    __syncthreads();
    if (t < NP)
#pragma unroll
      for (int r = 0; r < 4; ++r) tt[((size_t)tau * kNP + t) * 4 + r] = sm.total[t][r];
    __syncthreads();
  }
  // join: inflows at the slab faces and at every tile boundary, one thread per pair
  if (t < NP) {
    const int q = t, p = p0 + q;
    double TAf = 1.0, TBf = 0.0, TAb = 1.0, TBb = 0.0;
    for (int tau = 0; tau < T; ++tau) {  // forward: left to right
      const double* m = tt + ((size_t)tau * kNP + q) * 4;
      TBf = fma(m[0], TBf, m[1]);
      TAf *= m[0];
    }
    for (int tau = T - 1; tau >= 0; --tau) {  // backward: right to left
      const double* m = tt + ((size_t)tau * kNP + q) * 4;
      TBb = fma(m[2], TBb, m[3]);
      TAb *= m[2];
    }
    double psi_right_in = 0.0, psi_left_in = 0.0;
    if (w.rr || w.rl) {
      if (w.rr && !w.rl) {
        psi_right_in = TBf;
      } else {
        if (w.rr) psi_right_in = sm.lag[w.it & 1][p];
        if (w.rl) psi_left_in = fma(TAb, psi_right_in, TBb);
        if (w.rr && w.rl) sm.lag[(w.it + 1) & 1][p] = fma(TAf, psi_left_in, TBf);
      }
    }
    double e = psi_left_in;
    for (int tau = 0; tau < T; ++tau) {
      const double* m = tt + ((size_t)tau * kNP + q) * 4;
      ein[((size_t)tau * kNP + q) * 2] = e;
      e = fma(m[0], e, m[1]);
    }
    e = psi_right_in;
    for (int tau = T - 1; tau >= 0; --tau) {
      const double* m = tt + ((size_t)tau * kNP + q) * 4;
      ein[((size_t)tau * kNP + q) * 2 + 1] = e;
      e = fma(m[2], e, m[3]);
    }
  }
  __syncthreads();
  // pass B: replay every tile from its inflows, edge accumulators into the workspace rows
  for (int tau = 0; tau < T; ++tau) {
    w.cbase = tau * TC;
    stage(tau);
    maps_phase<K, NT, ANISO, NP>(sc, sm, io, p0, w, al, bp, bm);
    __syncthreads();
    scan_phase<K, NT, NP, false>(sm, w.lane, w.warp, 0);
    __syncthreads();
    double e[2 * NP];
#pragma unroll
    for (int r = 0; r < 2 * NP; ++r) e[r] = ein[(size_t)tau * kNP * 2 + r];
    EdgeAcc<K, WJ> acc;
    acc.zero();
    replay_tile<K, NT, NP, WJ>(sc, sm, p0, t, al, bp, bm, e, acc);
    const size_t c0 = (size_t)tau * TC + (size_t)t * K;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      FL[c0 + j] += acc.Fl[j];
      if constexpr (WJ) JL[c0 + j] += acc.Jl[j];
    }
    FR[(size_t)tau * NT + t] += acc.Fr;
    if constexpr (WJ) JR[(size_t)tau * NT + t] += acc.Jr;
    __syncthreads();  // (sm.agg / xmap are rewritten by the next tile)
  }
}

// WJ: edge currents wanted (P1 emission, current output, face leakages)
template <int K, int NT, bool ANISO, bool WJ>
__global__ void __launch_bounds__(NT, 1)
si_tiled_kernel(const __grid_constant__ SweepConsts sc, const SolveConfig cfg, const double* __restrict__ st_g,
                const double* __restrict__ ss0_g, const double* __restrict__ ss1_g, const double* __restrict__ src_g,
                const double* __restrict__ phi0_g, double* __restrict__ phi_g, double* __restrict__ jc_g,
                int32_t* __restrict__ iters, uint8_t* __restrict__ conv, int* __restrict__ flags,
                double* __restrict__ ws_g, double* __restrict__ leak_g, const uint8_t* __restrict__ active) {
  extern __shared__ __align__(32) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<SweepSmem<K, NT>*>(smem_raw);
  constexpr int TC = NT * K;
  const int b = blockIdx.x, t = threadIdx.x, Nc = sc.n_cells, P = sc.n_pairs;
  if (active && !active[b]) return;
  const int T = (Nc + TC - 1) / TC;
  const size_t Np = (size_t)T * TC, nch = (size_t)T * NT, base = (size_t)b * Nc;
  double* ws = ws_g + (size_t)b * tiled_ws_doubles<K, NT>(Nc, WJ);
  double *q2 = ws, *FL = ws + Np, *FR = FL + Np, *tt = FR + nch, *ein = tt + (size_t)T * kNP * 4;
  double* JL = WJ ? ein + (size_t)T * kNP * 2 : nullptr;
  double* JR = WJ ? JL + Np : nullptr;
  const double *st = st_g + base, *ss = ss0_g + base, *src = src_g + base;
  double* phi = phi_g + base;
  CellIO io;
  io.ss0 = ss;
  io.src = src;
  io.ss1 = ANISO ? ss1_g + base : nullptr;
  io.jc = (WJ && jc_g) ? jc_g + base : nullptr;
  SweepCtl w;
  w.t = t;
  w.lane = t & 31;
  w.warp = t >> 5;
  w.crank = 0;
  w.csz = 1;
  w.gslot = 0;
  w.cbase = 0;
  w.owns_last = false;
  w.rl = cfg.bc_left == 1;
  w.rr = cfg.bc_right == 1;
  // validation, initial flux (zero guess unless phi0), emission, P1 current
  bool bad = false;
  for (int i = t; i < Nc; i += NT) {
    bad |= !(st[i] > 0.0);
    const double p0 = phi0_g ? phi0_g[base + i] : 0.0;
    phi[i] = p0;
    q2[i] = fma(ss[i], p0, src[i]);
    if constexpr (ANISO) io.jc[i] = 0.0;
  }
  (void)ANISO;
  for (int i = t; i < kMaxPairs; i += NT) {
    sm.lag[0][i] = 0.0;
    sm.lag[1][i] = 0.0;
  }
  if (__syncthreads_or(bad)) {
    if (t == 0) {
      atomicOr(flags, snop_impl::FLAG_BAD_SIGMA_T);
      iters[b] = 0;
      conv[b] = 0;
    }
    return;
  }
  int it = 0, rphase = 0;
  bool converged = false;
  while (it < cfg.max_it) {
    ++it;
    w.it = it;
    for (size_t i = t; i < Np; i += NT) {
      FL[i] = 0.0;
      if constexpr (WJ) JL[i] = 0.0;
    }
    for (size_t i = t; i < nch; i += NT) {
      FR[i] = 0.0;
      if constexpr (WJ) JR[i] = 0.0;
    }
    __syncthreads();
    int p = 0;
    for (; p + 1 < P; p += 2)
      tiled_pair_group<K, NT, ANISO, WJ, 2>(sc, sm, io, w, p, T, st, q2, FL, FR, JL, JR, tt, ein);
    for (; p < P; ++p) tiled_pair_group<K, NT, ANISO, WJ, 1>(sc, sm, io, w, p, T, st, q2, FL, FR, JL, JR, tt, ein);
    // flux update, next emission, convergence norm
    double num = 0.0, den = 0.0;
    for (int tau = 0; tau < T; ++tau) {
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const size_t i = (size_t)tau * TC + (size_t)t * K + j;
        if (i < (size_t)Nc) {
          const double FRi = (j + 1 < K) ? FL[i + 1] : FR[(size_t)tau * NT + t];
          const double pn = 0.5 * (FL[i] + FRi);
          if constexpr (WJ) {
            const double JRi = (j + 1 < K) ? JL[i + 1] : JR[(size_t)tau * NT + t];
            if (io.jc) io.jc[i] = 0.5 * (JL[i] + JRi);
            if (leak_g && i == 0) leak_g[2 * (size_t)b] = -JL[0];              // J(0) = in - out
            if (leak_g && i == (size_t)Nc - 1) leak_g[2 * (size_t)b + 1] = JRi;  // J(L) = out - in
          }
          const double d = pn - phi[i];
          if (cfg.norm == 0) {
            num = fmax(num, fabs(d));
            den = fmax(den, fabs(pn));
          } else {
            num = fma(d, d, num);
            den = fma(pn, pn, den);
          }
          phi[i] = pn;
          q2[i] = fma(ss[i], pn, src[i]);
        }
      }
    }
    reduce2<NT, false>(num, den, cfg.norm == 0, sm.red, sm.cred, rphase++, sm);
    const double rel = rel_change(num, den, cfg.norm);
    if (!(rel == rel)) break;  // NaN: stop, reported non-converged
    if (rel < cfg.tol) {
      converged = true;
      break;
    }
  }
  if (t == 0) {
    iters[b] = it;
    conv[b] = converged ? 1 : 0;
  }
}

template <int K, int NT>
snop_status launch_tiled_t(snop_impl::Ctx& ctx, const SweepConsts& sc, const SolveConfig& cfg, int batch,
                           const double* st, const double* ss0, const double* ss1, const double* src,
                           const double* phi0, double* phi, double* cur, int32_t* iters, uint8_t* conv,
                           double* leak, const uint8_t* active) {
  const bool aniso = ss1 != nullptr, wj = aniso || cur || leak;
  const size_t per = tiled_ws_doubles<K, NT>(sc.n_cells, wj);
  double* ws = static_cast<double*>(ctx.slot(30, (size_t)batch * per * sizeof(double)));
  double* jc = cur;
  if (aniso && !jc) jc = static_cast<double*>(ctx.slot(21, (size_t)batch * sc.n_cells * sizeof(double)));
  if (!ws || (aniso && !jc)) {
    snop_impl::set_error("cudaMalloc (streaming sweep workspace) failed");
    return SNOP_CUDA_ERROR;
  }
  const size_t smem = smem_bytes<K, NT>();
  auto kern = aniso ? si_tiled_kernel<K, NT, true, true>
                    : (wj ? si_tiled_kernel<K, NT, false, true> : si_tiled_kernel<K, NT, false, false>);
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<batch, NT, smem, ctx.stream>>>(sc, cfg, st, ss0, ss1, src, phi0, phi, jc, iters, conv, ctx.d_flags, ws,
                                        leak, active);
  ctx.launches++;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snop_impl::set_error(std::string("si_tiled_kernel launch: ") + cudaGetErrorString(e));
    return SNOP_CUDA_ERROR;
  }
  return SNOP_OK;
}

template snop_status launch_tiled_t<SNOP_K, 256>(snop_impl::Ctx&, const SweepConsts&, const SolveConfig&, int,
                                                 const double*, const double*, const double*, const double*,
                                                 const double*, double*, double*, int32_t*, uint8_t*, double*,
                                                 const uint8_t*);

}  // namespace snop_si
