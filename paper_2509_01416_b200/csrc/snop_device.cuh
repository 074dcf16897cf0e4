// snop_device.cuh — device-side building blocks of the fused S_N source-iteration kernels
// (sm_100a). See DESIGN.md §K1 for the derivation; summary:
//
//   * One CTA owns one transport instance for the WHOLE solve (all source iterations, and for
//     eigenproblems all outer/group/inner iterations): its per-cell state lives in registers
//     (sigma_t, phi, Q, edge currents) and shared memory (sigma_s0, external source), so the
//     iteration loop never round-trips HBM. Instances with different iteration counts simply
//     retire their CTA early; the block scheduler back-fills the SM (no lock-step batch).
//   * Thread t owns K contiguous cells. For each +/-mu pair p the diamond-difference cell
//     recurrence psi_out = alpha_i psi_in + beta_i (alpha = (c-St)/(c+St) = 2c r - 1,
//     beta = 2q r, r = 1/(St+c), c = 2|mu|/dx) is an affine map. Both directions of the pair
//     share alpha_i and r_i (and beta_i for isotropic emission), so one reciprocal serves two
//     updates. Maps are composed per thread (K cells), scanned across the warp with shuffles
//     (prefix for mu>0, suffix for mu<0), then across warps through shared memory, and replayed.
//   * The scalar flux is not summed from psi_avg: the DD balance  mu (psi_R - psi_L)/dx +
//     St psi_avg = q  summed with the quadrature weights gives
//        phi_i = (Ss0_i phi_i^old + S_i - (J_{i+1/2} - J_{i-1/2}) / dx) / St_i,
//     J_e = sum_n w_n mu_n psi_n(e), so each update accumulates one edge current (1 FMA) instead
//     of two cell-average terms. Exact in exact arithmetic; ~1e-14 relative in fp64.
//   * The convergence norm (relative L-inf or L2 of successive scalar fluxes) is
//     a block reduction fused in the same kernel; max is order-independent (bit-deterministic),
//     the L2 sums use a fixed lane/warp order.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace snop_dev {

constexpr int kMaxPairs = 64;  // order <= 128

// Quadrature/mesh constants for one launch (kernel parameter => constant bank, uniform loads).
struct SweepConsts {
  int n_cells;
  int n_pairs;
  double dx;
  double inv_dx;
  double c[kMaxPairs];     // 2 mu_p / dx  (mu_p > 0, ascending p)
  double wmu[kMaxPairs];   // w_p mu_p
  double mu3[kMaxPairs];   // 3 mu_p (P1 emission term)
};

struct SolveConfig {
  double tol;
  int max_it;
  int bc_left;   // 0 vacuum, 1 reflective
  int bc_right;
  int norm;      // 0 rel-Linf, 1 rel-L2
};

__device__ __forceinline__ double rcp_fast(double t) {
  // MUFU.RCP64H seed + one cubic Newton step: rel. error ~ e0^3 (< 1e-18 for a ~2^-22 seed).
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(t));
  double e = fma(-t, r, 1.0);
  e = fma(e, e, e);
  return fma(r, e, r);
}

__device__ __forceinline__ double shfl_up_d(double v, int off) { return __shfl_up_sync(0xffffffffu, v, off); }
__device__ __forceinline__ double shfl_down_d(double v, int off) { return __shfl_down_sync(0xffffffffu, v, off); }
__device__ __forceinline__ double shfl_xor_d(double v, int off) { return __shfl_xor_sync(0xffffffffu, v, off); }
__device__ __forceinline__ double shfl_d(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

// Block-wide reductions (result broadcast to all threads). `scratch` holds >= 2*NW doubles and
// is double-buffered by `phase` so back-to-back reductions need only one barrier each.
template <int NT>
__device__ __forceinline__ double block_max(double v, double* scratch, int phase) {
  constexpr int NW = NT / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, shfl_xor_d(v, o));
  double* s = scratch + (phase & 1) * NW;
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = s[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) r = fmax(r, s[w]);
  return r;
}

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* scratch, int phase) {
  constexpr int NW = NT / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += shfl_xor_d(v, o);
  double* s = scratch + (phase & 1) * NW;
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = s[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) r += s[w];
  return r;
}

// Two independent block maxima with a single barrier.
template <int NT>
__device__ __forceinline__ void block_max2(double& a, double& b, double* scratch, int phase) {
  constexpr int NW = NT / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a = fmax(a, shfl_xor_d(a, o));
    b = fmax(b, shfl_xor_d(b, o));
  }
  double* s = scratch + (phase & 1) * 2 * NW;
  if ((threadIdx.x & 31) == 0) {
    s[threadIdx.x >> 5] = a;
    s[NW + (threadIdx.x >> 5)] = b;
  }
  __syncthreads();
  double ra = s[0], rb = s[NW];
#pragma unroll
  for (int w = 1; w < NW; ++w) {
    ra = fmax(ra, s[w]);
    rb = fmax(rb, s[NW + w]);
  }
  a = ra;
  b = rb;
}

template <int NT>
__device__ __forceinline__ void block_sum2(double& a, double& b, double* scratch, int phase) {
  constexpr int NW = NT / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += shfl_xor_d(a, o);
    b += shfl_xor_d(b, o);
  }
  double* s = scratch + (phase & 1) * 2 * NW;
  if ((threadIdx.x & 31) == 0) {
    s[threadIdx.x >> 5] = a;
    s[NW + (threadIdx.x >> 5)] = b;
  }
  __syncthreads();
  double ra = s[0], rb = s[NW];
#pragma unroll
  for (int w = 1; w < NW; ++w) {
    ra += s[w];
    rb += s[NW + w];
  }
  a = ra;
  b = rb;
}

// relative change from the two reduced quantities (zero rule pinned in oracle)
__device__ __forceinline__ double rel_change(double num, double den, int norm) {
  if (norm == 1) {
    num = sqrt(num);
    den = sqrt(den);
  }
  if (den > 0.0) return num / den;
  return num > 0.0 ? __longlong_as_double(0x7ff0000000000000ll) : 0.0;
}

// Shared-memory workspace of one CTA solver (the P1 moment array, when present, is a separate
// dynamic-smem region passed as a pointer so isotropic launches do not pay for it).
template <int K, int NT>
struct SweepSmem {
  static constexpr int NW = NT / 32;
  double ss0[K * NT];          // within-group Sigma_s0 of own cells, [j][t] (conflict-free)
  double src[K * NT];          // external isotropic source S (or q_ext), [j][t]
  double phi[K * NT];          // scalar flux of own cells, [j][t]
  double jc[K * NT];           // cell-average current (P1 emission / optional output), [j][t]
  double tot[2][NW][4];        // per-warp scan totals {Afwd, Bfwd, Abwd, Bbwd}, double-buffered
  double jfirst[NT + 1];       // J at each thread's first edge (+ J at the last edge, slot NT)
  double red[4 * NW];          // reductions inside si_solve
  double red2[4 * NW];         // reductions of the enclosing (eigen) kernel
  double lag[2][kMaxPairs];    // both-reflective: lagged mu>0 outflow at x=L, by iteration parity
};

// One CTA solves one within-group fixed-source problem by source iteration.
// On entry: st[] own sigma_t (>0; 1 on padding cells); sm.phi initial flux, sm.jc initial cell
// current (read only when ANISO), sm.ss0/src (and ss1s when ANISO) filled for own cells.
// On exit: sm.phi final flux, sm.jc cell-average current of the last sweep (written when
// ANISO || CUR). Returns sweeps performed; *converged is uniform across the CTA.
template <int K, int NT, bool ANISO, bool CUR>
__device__ int si_solve(const SweepConsts& sc, const SolveConfig& cfg, SweepSmem<K, NT>& sm,
                        const double* __restrict__ ss1s, const double (&st)[K], bool* converged) {
  constexpr int NW = NT / 32;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int c0 = t * K;
  const int Nc = sc.n_cells, P = sc.n_pairs;
  const bool owns_last = (c0 <= Nc - 1) && (Nc - 1 < c0 + K);
  const int jlast = Nc - 1 - c0;
  const bool rl = cfg.bc_left == 1, rr = cfg.bc_right == 1;

  if (t < kMaxPairs) {
    sm.lag[0][t] = 0.0;
    sm.lag[1][t] = 0.0;
  }
  __syncthreads();

  double Q[K];
  int it = 0;
  bool conv = false;
  int rphase = 0;
  while (it < cfg.max_it) {
    ++it;
    // emission (x2): Q = Ss0 phi + S ; angular q_n = Q/2 + 3/2 Ss1 mu_n J
#pragma unroll
    for (int j = 0; j < K; ++j) Q[j] = fma(sm.ss0[j * NT + t], sm.phi[j * NT + t], sm.src[j * NT + t]);
    double Jl[K];
#pragma unroll
    for (int j = 0; j < K; ++j) Jl[j] = 0.0;
    double Jend = 0.0;

    for (int p = 0; p < P; ++p) {
      const double c = sc.c[p], c2 = 2.0 * c, wm = sc.wmu[p];
      double al[K], bp[K], bm[K];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (c0 + j < Nc) {
          const double r = rcp_fast(st[j] + c);
          al[j] = fma(c2, r, -1.0);
          if constexpr (ANISO) {
            const double a3 = sc.mu3[p] * ss1s[j * NT + t] * sm.jc[j * NT + t];
            bp[j] = (Q[j] + a3) * r;
            bm[j] = (Q[j] - a3) * r;
          } else {
            bp[j] = Q[j] * r;
            bm[j] = bp[j];
          }
        } else {  // padding cell: identity map
          al[j] = 1.0;
          bp[j] = 0.0;
          bm[j] = 0.0;
        }
      }
      // compose own chunk: forward (cells ascending) and backward (descending)
      double Af = al[0], Bf = bp[0];
#pragma unroll
      for (int j = 1; j < K; ++j) {
        Bf = fma(al[j], Bf, bp[j]);
        Af *= al[j];
      }
      double Bb = bm[K - 1];
#pragma unroll
      for (int j = K - 2; j >= 0; --j) Bb = fma(al[j], Bb, bm[j]);
      double Ab = Af;
      // warp scans: forward inclusive prefix, backward inclusive suffix (Kogge-Stone)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double ap = shfl_up_d(Af, o), bpv = shfl_up_d(Bf, o);
        const double an = shfl_down_d(Ab, o), bnv = shfl_down_d(Bb, o);
        if (lane >= o) {
          Bf = fma(Af, bpv, Bf);
          Af *= ap;
        }
        if (lane + o < 32) {
          Bb = fma(Ab, bnv, Bb);
          Ab *= an;
        }
      }
      double* tot = &sm.tot[p & 1][0][0];
      if (lane == 31) { tot[warp * 4 + 0] = Af; tot[warp * 4 + 1] = Bf; }
      if (lane == 0) { tot[warp * 4 + 2] = Ab; tot[warp * 4 + 3] = Bb; }
      __syncthreads();
      // boundary values (SURVEY §9 #2 ordering) and the psi entering this warp, composed
      // serially from broadcast smem reads of the warp totals (warp-uniform work).
      double psi_right_in = 0.0, psi_left_in = 0.0;
      if (rr && !rl) {
        double v = 0.0;
        for (int w = 0; w < NW; ++w) v = fma(tot[w * 4 + 0], v, tot[w * 4 + 1]);
        psi_right_in = v;
      } else {
        if (rr) psi_right_in = sm.lag[it & 1][p];
        if (rl) {
          double v = psi_right_in;
          for (int w = NW - 1; w >= 0; --w) v = fma(tot[w * 4 + 2], v, tot[w * 4 + 3]);
          psi_left_in = v;
        }
        if (rr && rl && t == 0) {
          double v = psi_left_in;
          for (int w = 0; w < NW; ++w) v = fma(tot[w * 4 + 0], v, tot[w * 4 + 1]);
          sm.lag[(it + 1) & 1][p] = v;
        }
      }
      double wf_in = psi_left_in;
      for (int w = 0; w < warp; ++w) wf_in = fma(tot[w * 4 + 0], wf_in, tot[w * 4 + 1]);
      double wb_in = psi_right_in;
      for (int w = NW - 1; w > warp; --w) wb_in = fma(tot[w * 4 + 2], wb_in, tot[w * 4 + 3]);
      // psi entering this lane's chunk = psi leaving the neighbour lane's chunk
      double psi = shfl_up_d(fma(Af, wf_in, Bf), 1);
      if (lane == 0) psi = wf_in;
      double psib = shfl_down_d(fma(Ab, wb_in, Bb), 1);
      if (lane == 31) psib = wb_in;
      // replay: accumulate the edge currents J_e += w mu (psi+ - psi-)
#pragma unroll
      for (int j = 0; j < K; ++j) {
        Jl[j] = fma(wm, psi, Jl[j]);
        psi = fma(al[j], psi, bp[j]);
      }
      if (owns_last) Jend = fma(wm, psi - psib, Jend);
#pragma unroll
      for (int j = K - 1; j >= 0; --j) {
        psib = fma(al[j], psib, bm[j]);
        Jl[j] = fma(-wm, psib, Jl[j]);
      }
    }
    // edge-current exchange: J at the right edge of own last cell = next thread's first edge
    sm.jfirst[t] = Jl[0];
    if (owns_last) sm.jfirst[NT] = Jend;
    __syncthreads();
    const double Jnext = sm.jfirst[t + 1 < NT ? t + 1 : NT];
    const double Jlastv = sm.jfirst[NT];
    double num = 0.0, den = 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (c0 + j < Nc) {
        double JR = (j + 1 < K) ? Jl[j + 1] : Jnext;
        if (owns_last && j == jlast) JR = Jlastv;
        // balance form of phi = sum_n w_n psi_avg,n
        const double pn = (Q[j] - (JR - Jl[j]) * sc.inv_dx) / st[j];
        if constexpr (ANISO || CUR) sm.jc[j * NT + t] = 0.5 * (Jl[j] + JR);
        const double d = pn - sm.phi[j * NT + t];
        if (cfg.norm == 0) {
          num = fmax(num, fabs(d));
          den = fmax(den, fabs(pn));
        } else {
          num = fma(d, d, num);
          den = fma(pn, pn, den);
        }
        sm.phi[j * NT + t] = pn;
      }
    }
    if (cfg.norm == 0) block_max2<NT>(num, den, sm.red, rphase++);
    else block_sum2<NT>(num, den, sm.red, rphase++);
    const double rel = rel_change(num, den, cfg.norm);
    if (!(rel == rel)) break;  // NaN: stop, reported non-converged
    if (rel < cfg.tol) {
      conv = true;
      break;
    }
  }
  *converged = conv;
  return it;
}

}  // namespace snop_dev
