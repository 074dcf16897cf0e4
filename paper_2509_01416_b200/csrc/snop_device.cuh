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

// Predicated FP64 ops (no select instructions in the scan; the predicate is lane-constant).
__device__ __forceinline__ void pfma(double& d, double a, double b, double c, bool p) {
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %4, 0;\n\t@q fma.rn.f64 %0, %1, %2, %3;\n\t}"
      : "+d"(d) : "d"(a), "d"(b), "d"(c), "r"((unsigned)p));
}
__device__ __forceinline__ void pmul(double& d, double a, double b, bool p) {
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q mul.rn.f64 %0, %1, %2;\n\t}"
      : "+d"(d) : "d"(a), "d"(b), "r"((unsigned)p));
}

// Shared-memory workspace of one CTA solver (the P1 moment array, when present, is a separate
// dynamic-smem region passed as a pointer so isotropic launches do not pay for it). Per-cell
// arrays use the [j][t] layout: thread t's cell j sits at j*NT + t (conflict-free, private).
template <int K, int NT>
struct SweepSmem {
  static constexpr int NW = NT / 32;
  double st[K * NT];           // Sigma_t (0 on padding cells)
  double q2[K * NT];           // 2 x isotropic emission: Ss0 phi + S (rebuilt every iteration)
  double phi[K * NT];          // scalar flux
  alignas(32) double tot[2][2][NW][4];  // scan totals [slot][pair-in-group][warp] {Af,Bf,Ab,Bb}
  double jfirst[NT + 1];       // J at each thread's first edge (+ J at the last edge, slot NT)
  double red[4 * NW];          // reductions inside si_solve
  double red2[4 * NW];         // reductions of the enclosing (eigen) kernel
  double lag[2][kMaxPairs];    // both-reflective: lagged mu>0 outflow at x=L, by iteration parity
};

// Per-cell inputs that are touched once per iteration stay in global memory (L2-resident for
// the active instances), natural layout, already offset to the instance: g[c0 + j] for thread
// t's cell j (c0 = t*K). Padding cells (c0 + j >= Nc) are never read.
struct CellIO {
  const double* __restrict__ ss0;  // within-group Sigma_s0
  const double* __restrict__ src;  // external isotropic source
  const double* __restrict__ ss1;  // P1 moment (ANISO only)
  double* __restrict__ jc;         // cell-average current (ANISO / CUR)
};

struct SweepCtl {
  int t, lane, warp, it, slot;
  bool rl, rr, owns_last;
};

// Sweeps NP (1 or 2) +/-mu pairs starting at p0 and accumulates their edge currents into Jl /
// Jend. The NP pairs are independent chains the scheduler interleaves (ILP); one barrier per
// group. Padding cells carry St = q2 = 0, so alpha = 2c/c - 1 = 1 (to 1 ulp) and beta = 0.
template <int K, int NT, bool ANISO, int NP>
__device__ __forceinline__ void sweep_pair_group(const SweepConsts& sc, SweepSmem<K, NT>& sm, const CellIO& io,
                                                 int p0, const SweepCtl& w, double (&Jl)[K], double& Jend) {
  constexpr int NW = NT / 32;
  const int t = w.t, lane = w.lane, warp = w.warp;
  double c[NP], c2[NP], wm[NP];
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    c[q] = sc.c[p0 + q];
    c2[q] = 2.0 * c[q];
    wm[q] = sc.wmu[p0 + q];
  }
  double al[NP][K], bp[NP][K], bm[NP][K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const double stj = sm.st[j * NT + t], qj = sm.q2[j * NT + t];
    double a3base = 0.0;
    if constexpr (ANISO) a3base = (t * K + j < sc.n_cells) ? io.ss1[t * K + j] * io.jc[t * K + j] : 0.0;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const double r = rcp_fast(stj + c[q]);
      al[q][j] = fma(c2[q], r, -1.0);
      if constexpr (ANISO) {
        const double a3 = sc.mu3[p0 + q] * a3base;
        bp[q][j] = (qj + a3) * r;
        bm[q][j] = (qj - a3) * r;
      } else {
        bp[q][j] = qj * r;
        bm[q][j] = bp[q][j];
      }
    }
  }
  // compose own chunk: forward (ascending) and backward (descending)
  double Af[NP], Bf[NP], Ab[NP], Bb[NP];
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    Af[q] = al[q][0];
    Bf[q] = bp[q][0];
    Bb[q] = bm[q][K - 1];
  }
#pragma unroll
  for (int j = 1; j < K; ++j)
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      Bf[q] = fma(al[q][j], Bf[q], bp[q][j]);
      Af[q] *= al[q][j];
      Bb[q] = fma(al[q][K - 1 - j], Bb[q], bm[q][K - 1 - j]);
    }
#pragma unroll
  for (int q = 0; q < NP; ++q) Ab[q] = Af[q];
  // warp scans (Kogge-Stone): forward inclusive prefix, backward inclusive suffix; predicated
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const bool up = lane >= o, dn = lane + o < 32;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const double ap = shfl_up_d(Af[q], o), bpv = shfl_up_d(Bf[q], o);
      const double an = shfl_down_d(Ab[q], o), bnv = shfl_down_d(Bb[q], o);
      pfma(Bf[q], Af[q], bpv, Bf[q], up);
      pmul(Af[q], Af[q], ap, up);
      pfma(Bb[q], Ab[q], bnv, Bb[q], dn);
      pmul(Ab[q], Ab[q], an, dn);
    }
  }
  double4* tot = reinterpret_cast<double4*>(&sm.tot[w.slot][0][0][0]);
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    if (lane == 31) { tot[q * NW + warp].x = Af[q]; tot[q * NW + warp].y = Bf[q]; }
    if (lane == 0) { tot[q * NW + warp].z = Ab[q]; tot[q * NW + warp].w = Bb[q]; }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    const double4* T4 = tot + q * NW;
    const int p = p0 + q;
    // boundary values (SURVEY §9 #2 ordering); only the reflective cases need full totals
    double psi_right_in = 0.0, psi_left_in = 0.0;
    if (w.rr || w.rl) {
      if (w.rr && !w.rl) {
        double v = 0.0;
#pragma unroll
        for (int u = 0; u < NW; ++u) { const double4 T = T4[u]; v = fma(T.x, v, T.y); }
        psi_right_in = v;
      } else {
        if (w.rr) psi_right_in = sm.lag[w.it & 1][p];
        if (w.rl) {
          double v = psi_right_in;
#pragma unroll
          for (int u = NW - 1; u >= 0; --u) { const double4 T = T4[u]; v = fma(T.z, v, T.w); }
          psi_left_in = v;
        }
        if (w.rr && w.rl && t == 0) {
          double v = psi_left_in;
#pragma unroll
          for (int u = 0; u < NW; ++u) { const double4 T = T4[u]; v = fma(T.x, v, T.y); }
          sm.lag[(w.it + 1) & 1][p] = v;
        }
      }
    }
    // psi entering this warp (fixed trip count, predicated)
    double wf_in = psi_left_in, wb_in = psi_right_in;
#pragma unroll
    for (int u = 0; u < NW - 1; ++u) {
      const double4 T = T4[u];
      pfma(wf_in, T.x, wf_in, T.y, u < warp);
      const double4 U = T4[NW - 1 - u];
      pfma(wb_in, U.z, wb_in, U.w, NW - 1 - u > warp);
    }
    // psi entering this lane's chunk = psi leaving the neighbour lane's chunk
    double psi = shfl_up_d(fma(Af[q], wf_in, Bf[q]), 1);
    if (lane == 0) psi = wf_in;
    double psib = shfl_down_d(fma(Ab[q], wb_in, Bb[q]), 1);
    if (lane == 31) psib = wb_in;
    const double psib_in = psib;  // psi- entering from the right (= inflow at x=L for the owner)
    // replay: accumulate the edge currents J_e += w mu (psi+ - psi-)
#pragma unroll
    for (int j = 0; j < K; ++j) {
      Jl[j] = fma(wm[q], psi, Jl[j]);
      psi = fma(al[q][j], psi, bp[q][j]);
      psib = fma(al[q][K - 1 - j], psib, bm[q][K - 1 - j]);
      Jl[K - 1 - j] = fma(-wm[q], psib, Jl[K - 1 - j]);
    }
    if (w.owns_last) Jend = fma(wm[q], psi - psib_in, Jend);  // J at x = L
  }
}

// One CTA solves one within-group fixed-source problem by source iteration.
// On entry sm.st (>0; 0 on padding) and sm.phi (initial flux; 0 on padding) hold the own cells;
// io.ss0 / io.src (0 on padding), io.ss1 and io.jc (initial cell current; ANISO) are the
// thread-ordered global arrays. On exit sm.phi holds the final flux and io.jc the cell-average
// current of the last sweep (written when ANISO || CUR). Returns sweeps performed;
// *converged is uniform in the CTA.
template <int K, int NT, bool ANISO, bool CUR, int NP = 1>
__device__ int si_solve(const SweepConsts& sc, const SolveConfig& cfg, SweepSmem<K, NT>& sm, const CellIO& io,
                        bool* converged) {
  const int t = threadIdx.x;
  const int c0 = t * K;
  const int Nc = sc.n_cells, P = sc.n_pairs;
  SweepCtl w;
  w.t = t;
  w.lane = t & 31;
  w.warp = t >> 5;
  w.owns_last = (c0 <= Nc - 1) && (Nc - 1 < c0 + K);
  w.rl = cfg.bc_left == 1;
  w.rr = cfg.bc_right == 1;
  const int jlast = Nc - 1 - c0;

  if (t < kMaxPairs) {
    sm.lag[0][t] = 0.0;
    sm.lag[1][t] = 0.0;
  }
  __syncthreads();

  int it = 0;
  bool conv = false;
  int rphase = 0;
  w.slot = 0;
  while (it < cfg.max_it) {
    ++it;
    w.it = it;
    // emission (x2): q2 = Ss0 phi + S ; angular q_n = q2/2 + 3/2 Ss1 mu_n J
#pragma unroll
    for (int j = 0; j < K; ++j)
      sm.q2[j * NT + t] = (c0 + j < Nc) ? fma(io.ss0[c0 + j], sm.phi[j * NT + t], io.src[c0 + j]) : 0.0;
    double Jl[K];
#pragma unroll
    for (int j = 0; j < K; ++j) Jl[j] = 0.0;
    double Jend = 0.0;
    int p = 0;
    if constexpr (NP == 2) {
      for (; p + 1 < P; p += 2) {
        sweep_pair_group<K, NT, ANISO, 2>(sc, sm, io, p, w, Jl, Jend);
        w.slot ^= 1;
      }
    }
    for (; p < P; ++p) {
      sweep_pair_group<K, NT, ANISO, 1>(sc, sm, io, p, w, Jl, Jend);
      w.slot ^= 1;
    }
    // edge-current exchange: J at the right edge of own last cell = next thread's first edge
    sm.jfirst[t] = Jl[0];
    if (w.owns_last) sm.jfirst[NT] = Jend;
    __syncthreads();
    const double Jnext = sm.jfirst[t + 1 < NT ? t + 1 : NT];
    const double Jlastv = sm.jfirst[NT];
    double num = 0.0, den = 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (c0 + j < Nc) {
        double JR = (j + 1 < K) ? Jl[j + 1] : Jnext;
        if (w.owns_last && j == jlast) JR = Jlastv;
        // balance form of phi = sum_n w_n psi_avg,n
        const double pn = (sm.q2[j * NT + t] - (JR - Jl[j]) * sc.inv_dx) / sm.st[j * NT + t];
        if constexpr (ANISO || CUR) io.jc[c0 + j] = 0.5 * (Jl[j] + JR);
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
