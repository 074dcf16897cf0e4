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
//   * The scalar flux is accumulated on cell EDGES: diamond difference makes every cell average
//     the mean of its two edge fluxes, psi_avg = (psi_L + psi_R)/2, so with the edge scalar flux
//     Phi_e = sum_n w_n psi_n(e)
//        phi_i = sum_n w_n psi_avg,n = (Phi_{i-1/2} + Phi_{i+1/2}) / 2
//     and each update accumulates one edge term (1 FMA) instead of a cell-average one. The sum is
//     of like-signed terms for nonnegative emission, so it is as well conditioned as SPEC's
//     sum of psi_avg at any optical thickness. (Round 1 took phi from the DD balance
//     (q - dJ/dx)/St, whose cancellation grows like 1/(St dx): 4e-10 relative at St = 1e-4.)
//     The edge current J_e = sum_n w_n mu_n psi_n(e) is accumulated as well only when the cell
//     current (P1 emission, current output) or the face leakages are requested.
//   * The convergence norm (relative L-inf or L2 of successive scalar fluxes) is
//     a block reduction fused in the same kernel; max is order-independent (bit-deterministic),
//     the L2 sums use a fixed lane/warp order.
#pragma once

#include <cooperative_groups.h>
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
  double w[kMaxPairs];     // w_p (weight of +mu_p and of -mu_p)
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

#ifndef SNOP_RCP_CUBIC
#define SNOP_RCP_CUBIC 1
#endif
__device__ __forceinline__ double rcp_fast(double t) {
  // MUFU.RCP64H seed + one cubic Newton step: rel. error ~ e0^3 (< 1e-18 for a ~2^-22 seed).
  // (SNOP_RCP_CUBIC=0: quadratic step, ~e0^2.)
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(t));
  double e = fma(-t, r, 1.0);
#if SNOP_RCP_CUBIC
  e = fma(e, e, e);
#endif
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

// Warp maximum of a NON-NEGATIVE double (sign bit clear; +inf and NaN patterns included): for such
// values the order of the bit patterns as unsigned integers is the order of the values, so two
// 32-bit warp reductions (REDUX) give the exact maximum - the high words first, then the low words
// of the lanes that hold the maximal high word.
__device__ __forceinline__ double warp_max_nonneg(double v) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  const unsigned hi = (unsigned)(u >> 32), lo = (unsigned)u;
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  return __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
}

// max(acc, |x|) for a non-negative accumulator, on the bit patterns (4 integer instructions
// instead of the ~8 of fmax's NaN handling; a NaN pattern is larger than every number, so NaNs are
// sticky and reach the convergence test).
__device__ __forceinline__ double absmax_acc(double acc, double x) {
  const unsigned long long a = (unsigned long long)__double_as_longlong(acc);
  const unsigned long long b = (unsigned long long)__double_as_longlong(x) & 0x7fffffffffffffffull;
  return __longlong_as_double((long long)(a > b ? a : b));
}

// Two independent block maxima of non-negative values (|d|, |phi|) with a single barrier.
template <int NT>
__device__ __forceinline__ void block_max2(double& a, double& b, double* scratch, int phase) {
  constexpr int NW = NT / 32;
  a = warp_max_nonneg(a);
  b = warp_max_nonneg(b);
  double* s = scratch + (phase & 1) * 2 * NW;
  if ((threadIdx.x & 31) == 0) {
    s[threadIdx.x >> 5] = a;
    s[NW + (threadIdx.x >> 5)] = b;
  }
  __syncthreads();
  double ra = s[0], rb = s[NW];
#pragma unroll
  for (int w = 1; w < NW; ++w) {  // (non-negative values: maxima on the bit patterns)
    ra = absmax_acc(ra, s[w]);
    rb = absmax_acc(rb, s[NW + w]);
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
// The rel-Linf stopping test on the two reduced maxima without the division: sets `nan` when
// num/den would be NaN (the caller stops, non-converged) and returns num/den < tol otherwise
// (den > 0: num < tol den; 0/0 counts as 0, x/0 as +inf).
__device__ __forceinline__ bool linf_converged(double num, double den, double tol, bool& nan) {
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  nan = (num != num) || (den != den) || (num == inf && den == inf);
  if (den > 0.0) return num < tol * den;
  return num == 0.0 && 0.0 < tol;
}

__device__ __forceinline__ double rel_change(double num, double den, int norm) {
  if (norm == 1) {
    num = sqrt(num);
    den = sqrt(den);
  }
  if (den > 0.0) return num / den;
  return num > 0.0 ? __longlong_as_double(0x7ff0000000000000ll) : 0.0;
}

// Stage Sigma_s0 and the external source in shared memory for the solve (the per-iteration flux
// update then reads no global memory).
#ifndef SNOP_STAGE_SS
#define SNOP_STAGE_SS 1
#endif

// Pairs per pair group (maps/scan/replay are done for NP +/-mu pairs per CTA barrier phase).
#ifndef SNOP_NP
#define SNOP_NP 2
#endif
constexpr int kNP = SNOP_NP;

// Shared-memory workspace of one CTA solver (the P1 moment array, when present, is a separate
// dynamic-smem region passed as a pointer so isotropic launches do not pay for it). Per-cell
// arrays use the [j][t] layout: thread t's cell j sits at j*NT + t (conflict-free, private).
template <int K, int NT>
struct SweepSmem {
  static constexpr int NW = NT / 32;
  double st[K * NT];           // Sigma_t (0 on padding cells)
  double q2[K * NT];           // 2 x isotropic emission: Ss0 phi + S (rebuilt every iteration)
  double phi[K * NT];          // scalar flux
#if SNOP_STAGE_SS
  double ss[K * NT];           // within-group Sigma_s0 and external source, staged at solver entry
  double src[K * NT];
#endif
  // chunk-indexed arrays use spos(): one pad slot per E = NT/32 entries, so the scan warp's
  // lane-strided reads (lane l owns chunks l*E .. l*E+E-1) are bank-conflict free
  static constexpr int E = NT / 32;
  static constexpr int NP_PAD = NT + (E > 1 ? 32 : 0);
  __device__ static constexpr int spos(int idx) { return E > 1 ? idx + idx / E : idx; }
  // chunk maps of the current pair group: [q][{A, Bf, Bb}][chunk]; the scan replaces Bf / Bb in
  // place by the exclusive maps' offsets and writes their slopes to xmap [q][{Af, Ab}][chunk]
  double agg[kNP][3][NP_PAD];
  double xmap[kNP][2][NP_PAD];
  double total[kNP][4];         // whole-domain maps [q][{Af, Bf, Ab, Bb}]
  double leak[2];              // net face currents of the latest sweep (written by the face owners)
  double red[4 * NW];          // reductions inside si_solve
  double red2[4 * NW];         // reductions of the enclosing (eigen) kernel
  double lag[2][kMaxPairs];    // both-reflective: lagged mu>0 outflow at x=L, by iteration parity
  // cluster mode (one instance spread over the CTAs of a thread-block cluster): per-CTA values
  // published for the other CTAs, read through distributed shared memory
  double ctot[2][kNP][4];      // CTA-level scan totals [group slot][q][{Af,Bf,Ab,Bb}]
  double cred[2][2];           // CTA-level reduction results (si_solve), by phase
  double credx[2][8][2];       // every rank's reduction results pushed here (si_solve), [phase][rank]
  double cred2[2][2];          // CTA-level reduction results (enclosing kernel), by phase
  int cflag[2];                // CTA-level flags (validation)
};

// ---- thread-block-cluster helpers ----------------------------------------------------------
__device__ __forceinline__ int cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return (int)r;
}
__device__ __forceinline__ int cl_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return (int)r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <class T>
__device__ __forceinline__ T* cl_map(T* local, int rank) {
  return cooperative_groups::this_cluster().map_shared_rank(local, (unsigned)rank);
}

// Block- then cluster-wide reduction of two values (max if is_max else sum). Ranks are combined
// in rank order, so every CTA of the cluster obtains the bit-identical result.
template <int NT, bool CL, class Smem>
__device__ __forceinline__ void reduce2(double& a, double& b, bool is_max, double* scratch, double (*cred)[2],
                                        int phase, Smem& sm) {
  if (is_max) block_max2<NT>(a, b, scratch, phase);
  else block_sum2<NT>(a, b, scratch, phase);
  if constexpr (CL) {
    const int s = phase & 1, n = cl_size();
    if (cred == sm.cred) {
      // si_solve's reductions: every CTA pushes its pair into every rank's credx slot (remote
      // stores, published by the cluster barrier), so the combine reads local shared memory only
      if ((int)threadIdx.x < n) {
        double* dst = cl_map(&sm.credx[s][cl_rank()][0], (int)threadIdx.x);
        dst[0] = a;
        dst[1] = b;
      }
      cl_sync();
      double ra = sm.credx[s][0][0], rb = sm.credx[s][0][1];
      for (int r = 1; r < n; ++r) {
        const double x = sm.credx[s][r][0], y = sm.credx[s][r][1];
        if (is_max) { ra = fmax(ra, x); rb = fmax(rb, y); }
        else { ra += x; rb += y; }
      }
      a = ra;
      b = rb;
      return;
    }
    if (threadIdx.x == 0) {
      cred[s][0] = a;
      cred[s][1] = b;
    }
    cl_sync();
    double ra = 0.0, rb = 0.0;
    for (int r = 0; r < n; ++r) {
      const double* rc = cl_map(&cred[s][0], r);
      const double x = rc[0], y = rc[1];
      if (r == 0) { ra = x; rb = y; }
      else if (is_max) { ra = fmax(ra, x); rb = fmax(rb, y); }
      else { ra += x; rb += y; }
    }
    a = ra;
    b = rb;
  }
  (void)sm;
}

// any() over the CTA (and the cluster when CL).
template <int NT, bool CL, class Smem>
__device__ __forceinline__ bool cluster_any(bool v, Smem& sm) {
  const bool blk = __syncthreads_or(v);
  if constexpr (!CL) {
    return blk;
  } else {
    if (threadIdx.x == 0) sm.cflag[0] = blk ? 1 : 0;
    cl_sync();
    bool any = false;
    for (int r = 0; r < cl_size(); ++r) any |= *cl_map(&sm.cflag[0], r) != 0;
    cl_sync();  // no CTA may leave (and free its shared memory) before all reads are done
    return any;
  }
}

// Per-cell inputs that are touched once per iteration stay in global memory (L2-resident for
// the active instances), natural layout, already offset to the instance: g[c0 + j] for thread
// t's cell j (c0 = t*K). Padding cells (c0 + j >= Nc) are never read.
struct CellIO {
  const double* __restrict__ ss0;  // within-group Sigma_s0
  const double* __restrict__ src;  // external isotropic source
  const double* __restrict__ ss1;  // P1 moment (ANISO only)
  double* __restrict__ jc;         // cell-average current (ANISO / CUR)
  double* leak = nullptr;          // [2] net outflow at x=0 / x=L of the last sweep (nullable)
};

#ifdef SNOP_PHASE_TIMING
// experiment builds only: per-phase cycle counters (thread 0 and thread 32 of every CTA)
#ifndef SNOP_PHASE_SYM
#define SNOP_PHASE_SYM g_phase_cycles
#endif
static __device__ unsigned long long SNOP_PHASE_SYM[2][10];  // distinct name per translation unit
#define SNOP_TSTAMP(var) long long var = clock64()
#define SNOP_TACC(slot, t0, t1)                                                          \
  do {                                                                                   \
    if ((threadIdx.x & 31) == 0 && threadIdx.x < 64)                                     \
      atomicAdd(&SNOP_PHASE_SYM[threadIdx.x >> 5][slot], (unsigned long long)((t1) - (t0))); \
  } while (0)
#else
#define SNOP_TSTAMP(var)
#define SNOP_TACC(slot, t0, t1)
#endif

struct SweepCtl {
  int t, lane, warp, it, gslot;
  int cbase;      // global index of this CTA's first cell (cluster mode: rank * NT * K)
  int crank, csz; // cluster rank / size (0 / 1 without clusters)
  bool rl, rr, owns_last;
};

// Phase A: per-cell affine maps of NP pairs (registers) and their per-thread chunk compositions
// (-> shared memory). Padding cells carry St = q2 = 0: alpha = 2c/c - 1 = 1 (to 1 ulp), beta = 0.
template <int K, int NT, bool ANISO, int NP>
__device__ __forceinline__ void maps_phase(const SweepConsts& sc, SweepSmem<K, NT>& sm, const CellIO& io, int p0,
                                           const SweepCtl& w, double (&al)[NP][K], double (&bp)[NP][K],
                                           double (&bm)[NP][K]) {
  const int t = w.t;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const double stj = sm.st[j * NT + t], qj = sm.q2[j * NT + t];
    double a3base = 0.0;
    if constexpr (ANISO) {
      const int i = w.cbase + t * K + j;
      a3base = (i < sc.n_cells) ? io.ss1[i] * io.jc[i] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const double c = sc.c[p0 + q];
      const double r = rcp_fast(stj + c);
      al[q][j] = fma(2.0 * c, r, -1.0);
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
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    double A = al[q][0], Bf = bp[q][0], Bb = bm[q][K - 1];
#pragma unroll
    for (int j = 1; j < K; ++j) {
      Bf = fma(al[q][j], Bf, bp[q][j]);
      A *= al[q][j];
      Bb = fma(al[q][K - 1 - j], Bb, bm[q][K - 1 - j]);
    }
    const int pt = SweepSmem<K, NT>::spos(t);
    sm.agg[q][0][pt] = A;
    sm.agg[q][1][pt] = Bf;
    sm.agg[q][2][pt] = Bb;
  }
}

// Phase B: one warp per (pair, direction) scans the NT chunk maps of the CTA: each lane composes
// E = NT/32 consecutive chunks serially, a 5-step shuffle scan joins the lanes, and every chunk
// gets the exclusive map that carries the CTA's inflow to its first edge. Forward = prefix (left
// to right), backward = suffix (right to left). In cluster mode the CTA totals are also
// published (ctot) for the other CTAs of the cluster.
// One (pair, direction) scan by one warp. Lane l owns chunks l*E .. l*E+E-1 in sweep order; with
// the padded layout those E chunk maps are contiguous in shared memory (ascending for the forward
// sweep, descending for the backward one), so every access is base + compile-time offset.
//   1. serial inclusive prefixes over the lane's E chunks, in registers (runs of more than
//      SNOP_SCAN_REG_E chunks keep only the total and recompose the prefixes in step 3);
//   2. the run totals shifted up one lane, then a 5-round shuffle scan of (identity, T_0 .. T_30)
//      -> the lane's exclusive entry map (A, B), with no predicates on the dependent chain;
//   3. exclusive map of chunk e = (A, B) composed with prefix e-1 (E-1 independent compositions).
#ifndef SNOP_SCAN_REG_E
#define SNOP_SCAN_REG_E 4
#endif
template <int K, int NT, bool FWD, bool CL>
__device__ __forceinline__ void scan_one(SweepSmem<K, NT>& sm, int q, int lane, int gslot) {
  constexpr int E = NT / 32;
  constexpr int S = E > 1 ? E + 1 : 1;  // padded stride between consecutive lanes' chunk runs
  constexpr int D = FWD ? 1 : -1;
  const int base = FWD ? lane * S : (31 - lane) * S + (E - 1);
  const double* a = sm.agg[q][0] + base;
  const double* b = sm.agg[q][FWD ? 1 : 2] + base;
  double* XA = sm.xmap[q][FWD ? 0 : 1] + base;
  double* XB = sm.agg[q][FWD ? 1 : 2] + base;  // in place: every offset is read before any is replaced
  // 1. inclusive prefixes of the own run, kept in registers (the kernel is bound by shared-memory
  //    wavefronts as much as by FP64 issue: no scratch round trip). Runs longer than SNOP_SCAN_REG_E chunks keep
  //    only the run total and recompose the prefixes from the chunk maps in step 3.
  constexpr bool REG = E <= SNOP_SCAN_REG_E;
  constexpr int EP = REG ? E : 1;
  double pa[EP], pb[EP];
  if constexpr (REG) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      pa[e] = a[D * e];
      pb[e] = b[D * e];
    }
#pragma unroll
    for (int e = 1; e < E; ++e) {
      pb[e] = fma(pa[e], pb[e - 1], pb[e]);
      pa[e] *= pa[e - 1];
    }
  } else {
    double ta = 1.0, tb = 0.0;
#pragma unroll
    for (int e0 = 0; e0 < E; e0 += 4) {
      double av[4], bv[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        av[h] = a[D * (e0 + h)];
        bv[h] = b[D * (e0 + h)];
      }
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        tb = fma(av[h], tb, bv[h]);
        ta *= av[h];
      }
    }
    pa[0] = ta;
    pb[0] = tb;
  }
  // 2. shift the run totals up one lane: the lanes then hold (identity, T_0, ..., T_30), whose
  //    inclusive scan is the exclusive scan of the totals, and lane 0's identity is what an
  //    out-of-range lane reads in the rounds below (x * 1 and x + A * 0 are exact), so the
  //    dependent chain has no predicates or selects: 5 rounds of shuffle + FMA.
  double A = __shfl_up_sync(0xffffffffu, pa[EP - 1], 1), B = __shfl_up_sync(0xffffffffu, pb[EP - 1], 1);
  if (lane == 0) {
    A = 1.0;
    B = 0.0;
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int srcl = max(lane - o, 0);
    const double ap = __shfl_sync(0xffffffffu, A, srcl), bq = __shfl_sync(0xffffffffu, B, srcl);
    B = fma(A, bq, B);
    A *= ap;
  }
  if (lane == 31) {  // whole-domain map = exclusive map of run 31 followed by run 31
    const double TA = A * pa[EP - 1], TB = fma(pa[EP - 1], B, pb[EP - 1]);
    sm.total[q][FWD ? 0 : 2] = TA;
    sm.total[q][FWD ? 1 : 3] = TB;
    if constexpr (CL) {
      sm.ctot[gslot][q][FWD ? 0 : 2] = TA;
      sm.ctot[gslot][q][FWD ? 1 : 3] = TB;
    }
  }
  // 3. exclusive map of chunk e = (A, B) followed by the prefix through chunk e-1
  if constexpr (REG) {
    XA[0] = A;
    XB[0] = B;
#pragma unroll
    for (int e = 1; e < E; ++e) {
      XA[D * e] = A * pa[e - 1];
      XB[D * e] = fma(pa[e - 1], B, pb[e - 1]);
    }
  } else {
    double ra = A, rb = B;
#pragma unroll
    for (int e0 = 0; e0 < E; e0 += 4) {
      double av[4], bv[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {  // (chunk maps read before their slots are replaced below)
        av[h] = a[D * (e0 + h)];
        bv[h] = b[D * (e0 + h)];
      }
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        XA[D * (e0 + h)] = ra;
        XB[D * (e0 + h)] = rb;
        rb = fma(av[h], rb, bv[h]);
        ra *= av[h];
      }
    }
  }
}

// Phase B: one warp per (pair, direction) scans the NT chunk maps of the CTA into the exclusive
// maps that carry the CTA's inflow to each chunk's first edge. Forward = prefix (left to right),
// backward = suffix (right to left). In cluster mode the CTA totals are also published (ctot)
// for the other CTAs of the cluster.
template <int K, int NT, int NP, bool CL>
__device__ __forceinline__ void scan_phase(SweepSmem<K, NT>& sm, int lane, int warp, int gslot) {
  constexpr int NW = NT / 32;
  for (int s = warp; s < 2 * NP; s += NW) {
    if ((s & 1) == 0) scan_one<K, NT, true, CL>(sm, s >> 1, lane, gslot);
    else scan_one<K, NT, false, CL>(sm, s >> 1, lane, gslot);
  }
}

// Edge accumulators of one thread: the scalar flux Phi at the left edge of each own cell (Fl)
// and at the right edge of the last one (Fr); with WJ also the current J at the same edges.
template <int K, bool WJ>
struct EdgeAcc {
  double Fl[K], Fr;
  double Jl[WJ ? K : 1], Jr;
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int j = 0; j < K; ++j) Fl[j] = 0.0;
    Fr = 0.0;
#pragma unroll
    for (int j = 0; j < (WJ ? K : 1); ++j) Jl[j] = 0.0;
    Jr = 0.0;
  }
};

// Phase C: boundary inflows (SURVEY §9 #2 ordering), the inflow of this CTA (cluster mode:
// composed from the other CTAs' totals read through DSMEM) and of this thread's chunk, then the
// replay that accumulates the edge scalar fluxes Phi_e += w (psi+ + psi-) (and, with WJ, the edge
// currents J_e += w mu (psi+ - psi-)).
template <int K, int NT, int NP, bool CL, bool WJ>
__device__ __forceinline__ void replay_phase(const SweepConsts& sc, SweepSmem<K, NT>& sm, int p0, const SweepCtl& w,
                                             const double (&al)[NP][K], const double (&bp)[NP][K],
                                             const double (&bm)[NP][K], EdgeAcc<K, WJ>& acc) {
  const int t = w.t;
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    const int p = p0 + q;
    const double wq = sc.w[p];
    const double wm = sc.wmu[p];
    // whole-domain totals (needed for reflective faces) and this CTA's entry maps
    double TAf, TBf, TAb, TBb;           // whole domain
    double EfA = 1.0, EfB = 0.0;         // composition of CTAs left of this one (forward)
    double EbA = 1.0, EbB = 0.0;         // composition of CTAs right of this one (backward)
    if constexpr (CL) {
      double fa = 1.0, fb = 0.0;
      for (int r = 0; r < w.csz; ++r) {  // forward: ranks ascending
        const double* T = cl_map(&sm.ctot[w.gslot][q][0], r);
        if (r == w.crank) { EfA = fa; EfB = fb; }
        const double a = T[0], b = T[1];
        fb = fma(a, fb, b);
        fa *= a;
      }
      TAf = fa;
      TBf = fb;
      double ba = 1.0, bb = 0.0;
      for (int r = w.csz - 1; r >= 0; --r) {  // backward: ranks descending
        const double* T = cl_map(&sm.ctot[w.gslot][q][0], r);
        if (r == w.crank) { EbA = ba; EbB = bb; }
        const double a = T[2], b = T[3];
        bb = fma(a, bb, b);
        ba *= a;
      }
      TAb = ba;
      TBb = bb;
    } else {
      TAf = TBf = TAb = TBb = 0.0;
      if (w.rr || w.rl) {  // (vacuum faces need no whole-domain map: no shared-memory reads)
        TAf = sm.total[q][0];
        TBf = sm.total[q][1];
        TAb = sm.total[q][2];
        TBb = sm.total[q][3];
      }
    }
    double psi_right_in = 0.0, psi_left_in = 0.0;
    if (w.rr || w.rl) {
      if (w.rr && !w.rl) {
        psi_right_in = TBf;  // mu>0 outflow at x=L with vacuum left
      } else {
        if (w.rr) psi_right_in = sm.lag[w.it & 1][p];
        if (w.rl) psi_left_in = fma(TAb, psi_right_in, TBb);
        if (w.rr && w.rl && t == 0) sm.lag[(w.it + 1) & 1][p] = fma(TAf, psi_left_in, TBf);
      }
    }
    // (one CTA: the entry maps are the identity; spelled out so no 1 * x + 0 is left on the chain)
    const double cta_left = CL ? fma(EfA, psi_left_in, EfB) : psi_left_in;
    const double cta_right = CL ? fma(EbA, psi_right_in, EbB) : psi_right_in;
    const int pt = SweepSmem<K, NT>::spos(t);
    double psi = fma(sm.xmap[q][0][pt], cta_left, sm.agg[q][1][pt]);
    double psib = fma(sm.xmap[q][1][pt], cta_right, sm.agg[q][2][pt]);
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
    // Phi (and J) at this thread's right chunk edge (no neighbour exchange)
    acc.Fr = fma(wq, psi + psib_in, acc.Fr);
    if constexpr (WJ) acc.Jr = fma(wm, psi - psib_in, acc.Jr);
  }
}

template <int K, int NT, bool ANISO, int NP, bool CL, bool WJ>
__device__ __forceinline__ void sweep_pair_group(const SweepConsts& sc, SweepSmem<K, NT>& sm, const CellIO& io,
                                                 int p0, SweepCtl& w, EdgeAcc<K, WJ>& acc) {
  double al[NP][K], bp[NP][K], bm[NP][K];
  SNOP_TSTAMP(t0);
  maps_phase<K, NT, ANISO, NP>(sc, sm, io, p0, w, al, bp, bm);
  SNOP_TSTAMP(t1);
  __syncthreads();
  SNOP_TSTAMP(t2);
  scan_phase<K, NT, NP, CL>(sm, w.lane, w.warp, w.gslot);
  SNOP_TSTAMP(t3);
  if constexpr (CL) cl_sync();
  else __syncthreads();
  SNOP_TSTAMP(t4);
  replay_phase<K, NT, NP, CL, WJ>(sc, sm, p0, w, al, bp, bm, acc);
  SNOP_TSTAMP(t5);
#ifndef SNOP_PS_TIMING
  SNOP_TACC(0, t0, t1);
  SNOP_TACC(1, t1, t2);
  SNOP_TACC(2, t2, t3);
  SNOP_TACC(3, t3, t4);
  SNOP_TACC(4, t4, t5);
#endif
  w.gslot ^= 1;
}

// One CTA (or, with CL, one thread-block cluster) solves one within-group fixed-source problem
// by source iteration. Thread t of cluster rank r owns the K cells starting at
// global cell r*NT*K + t*K. On entry sm.st (>0; 0 on padding) and sm.phi (initial flux; 0 on
// padding) hold the own cells; io.ss0 / io.src, io.ss1 and io.jc (initial cell current; ANISO)
// are the natural-layout global arrays of the instance. On exit sm.phi holds the final flux and
// io.jc the cell-average current of the last sweep (written when ANISO || CUR). Returns sweeps
// performed; *converged is uniform across the CTA / cluster.
// PS (pair split, eigen kernel only): the CTAs of a thread-block cluster each sweep a contiguous
// range of pair groups over ALL cells of the instance; after the pairs of a source iteration the
// partial edge currents are exchanged through distributed shared memory and summed in rank order,
// so every CTA performs the identical (redundant) flux update and convergence test. One source
// iteration then costs P/(2*CS) pair groups of latency plus one exchange, instead of P/2 groups.
template <int K, int NT, bool ANISO, bool CUR, bool CL = false, int NP = SNOP_NP, bool PS = false>
__device__ int si_solve(const SweepConsts& sc, const SolveConfig& cfg, SweepSmem<K, NT>& sm, const CellIO& io,
                        bool* converged) {
  static_assert(!(PS && CL), "pair split and cell split are exclusive");
  static_assert((K + 1) * NT <= 5 * kNP * SweepSmem<K, NT>::NP_PAD, "exchange buffer must fit in agg + xmap");
  constexpr bool WJ = ANISO || CUR;  // edge currents wanted (P1 emission, current, leakages)
  const int t = threadIdx.x;
  const int Nc = sc.n_cells, P = sc.n_pairs;
  SweepCtl w;
  w.t = t;
  w.lane = t & 31;
  w.warp = __shfl_sync(0xffffffffu, t >> 5, 0);  // warp-uniform for the compiler: uniform branches around the scans
  w.crank = CL ? cl_rank() : 0;
  w.csz = CL ? cl_size() : 1;
  w.cbase = w.crank * NT * K;
  w.gslot = 0;
  const int c0 = w.cbase + t * K;
  w.owns_last = (c0 <= Nc - 1) && (Nc - 1 < c0 + K);
  w.rl = cfg.bc_left == 1;
  w.rr = cfg.bc_right == 1;

  for (int i = t; i < kMaxPairs; i += NT) {  // (NT may be 32 < kMaxPairs)
    sm.lag[0][i] = 0.0;
    sm.lag[1][i] = 0.0;
  }
  if constexpr (CL) cl_sync();
  else __syncthreads();

  int it = 0;
  bool conv = false;
  int rphase = 0;
  // emission (x2): q2 = Ss0 phi + S ; angular q_n = q2/2 + 3/2 Ss1 mu_n J. Built
  // here for the first sweep and then in each flux update for the next one, so the L2 loads of
  // Ss0 and S overlap the flux update and the convergence reduction.
#if SNOP_STAGE_SS
  // (pair split: every CTA stages all cells, so an owner reads any cell's values locally; the
  // barriers of the first exchange order these stores before those reads)
#pragma unroll
  for (int j = 0; j < K; ++j) {
    sm.ss[j * NT + t] = (c0 + j < Nc) ? io.ss0[c0 + j] : 0.0;
    sm.src[j * NT + t] = (c0 + j < Nc) ? io.src[c0 + j] : 0.0;
  }
#endif
#pragma unroll
  for (int j = 0; j < K; ++j)
    sm.q2[j * NT + t] = (c0 + j < Nc) ? fma(io.ss0[c0 + j], sm.phi[j * NT + t], io.src[c0 + j]) : 0.0;
  while (it < cfg.max_it) {
    ++it;
    w.it = it;
    EdgeAcc<K, WJ> acc;
    acc.zero();
    SNOP_TSTAMP(ti0);
    int p = 0, pend = P;
    if constexpr (PS) {  // this CTA's contiguous range of pair groups (the odd tail pair: last rank)
      const int prank = cl_rank(), psz = cl_size(), G2 = P / 2, per = (G2 + psz - 1) / psz;
      const int g0 = min(G2, prank * per), g1 = min(G2, g0 + per);
      p = 2 * g0;
      pend = prank == psz - 1 ? P : 2 * g1;
    }
    if constexpr (NP > 2) {
      for (; p + NP - 1 < pend; p += NP) sweep_pair_group<K, NT, ANISO, NP, CL, WJ>(sc, sm, io, p, w, acc);
    }
    if constexpr (NP >= 2) {
      for (; p + 1 < pend; p += 2) sweep_pair_group<K, NT, ANISO, 2, CL, WJ>(sc, sm, io, p, w, acc);
    }
    for (; p < pend; ++p) sweep_pair_group<K, NT, ANISO, 1, CL, WJ>(sc, sm, io, p, w, acc);
    SNOP_TSTAMP(ti1);
    SNOP_TACC(5, ti0, ti1);
    double num = 0.0, den = 0.0;
    if constexpr (PS) {
      // Rank r owns the flux update of the cells of owner threads [r per, (r+1) per), per = NT/CS.
      // Every CTA pushes its partial edge scalar fluxes (K + 1 per thread) into the owner rank's
      // incoming buffer (agg + xmap, by source rank: [CS][K+1][per]); the owner sums the CS
      // partials in rank order, updates phi locally and pushes the new emission into every CTA.
      // All remote traffic is stores; the convergence norm is a cluster reduction (reduce2<CL =
      // true>) whose barrier also publishes the pushed emission. phi is pushed once, at the end.
      double* xb = &sm.agg[0][0][0];
      const int prank = cl_rank(), psz = cl_size(), per = NT / psz;
      SNOP_TSTAMP(tx0);
      cl_sync();  // every CTA has finished its replays (agg / xmap are free cluster-wide)
      SNOP_TSTAMP(tx1);
      {
        const int ro = t / per, uu = t - ro * per;
        double* dst = cl_map(xb, ro) + (size_t)prank * (K + 1) * per + uu;
#pragma unroll
        for (int j = 0; j < K; ++j) dst[j * per] = acc.Fl[j];
        dst[K * per] = acc.Fr;
      }
      SNOP_TSTAMP(tx2);
      cl_sync();
      SNOP_TSTAMP(tx3);
      for (int idx = t; idx < per * K; idx += NT) {
        const int j = idx / per, uu = idx - j * per, u = prank * per + uu;
        const int i = u * K + j;
        if (i < Nc) {
          double FL = 0.0, FR = 0.0;
          for (int r = 0; r < psz; ++r) {
            const double* src = xb + (size_t)r * (K + 1) * per + uu;
            FL += src[j * per];
            FR += src[(j + 1) * per];
          }
          const int o = j * NT + u;
          const double pn = 0.5 * (FL + FR);
          const double d = pn - sm.phi[o];
          if (cfg.norm == 0) {
            num = absmax_acc(num, d);
            den = absmax_acc(den, pn);
          } else {
            num = fma(d, d, num);
            den = fma(pn, pn, den);
          }
          sm.phi[o] = pn;
#if SNOP_STAGE_SS
          const double q2n = fma(sm.ss[o], pn, sm.src[o]);
#else
          const double q2n = fma(io.ss0[i], pn, io.src[i]);
#endif
          for (int r = 0; r < psz; ++r) cl_map(sm.q2, r)[o] = q2n;
        }
      }
      SNOP_TSTAMP(tx4);
      reduce2<NT, true>(num, den, cfg.norm == 0, sm.red, sm.cred, rphase++, sm);
      SNOP_TSTAMP(tx5);
#ifdef SNOP_PS_TIMING
      SNOP_TACC(0, tx0, tx1);  // wait for the slowest CTA's replays
      SNOP_TACC(1, tx1, tx2);  // push partials
      SNOP_TACC(2, tx2, tx3);  // cluster barrier
      SNOP_TACC(3, tx3, tx4);  // owner sums, flux update, emission push
      SNOP_TACC(4, tx4, tx5);  // norm reduction (block + cluster)
#endif
    } else {
    // Phi (J) at the right edge of the own last cell was accumulated locally (Fr, Jr); padding
    // cells after the global last cell are identity maps, so Jl[j+1] of a padding cell is J at L.
    double ssv[K], srcv[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
#if SNOP_STAGE_SS
      ssv[j] = sm.ss[j * NT + t];  // (own cells: written by this thread at entry)
      srcv[j] = sm.src[j * NT + t];
#else
      ssv[j] = (c0 + j < Nc) ? io.ss0[c0 + j] : 0.0;
      srcv[j] = (c0 + j < Nc) ? io.src[c0 + j] : 0.0;
#endif
    }
    // phi = sum_n w_n psi_avg,n = mean of the two edge scalar fluxes (diamond difference); the
    // next sweep's emission; the convergence norm's two reductions. Specialised per norm and for
    // threads whose K cells are all real cells (no per-cell predicates on the common path).
    auto phi_cell = [&](int j, double& pn) -> double {
      pn = 0.5 * (acc.Fl[j] + ((j + 1 < K) ? acc.Fl[j + 1] : acc.Fr));
      if constexpr (WJ) {
        const double JR = (j + 1 < K) ? acc.Jl[j + 1] : acc.Jr;
        if (io.jc) io.jc[c0 + j] = 0.5 * (acc.Jl[j] + JR);
        if (j == 0 && c0 == 0) sm.leak[0] = -acc.Jl[0];  // J(0) = in - out at the left face
        if (c0 + j == Nc - 1) sm.leak[1] = JR;           // J(L) = out - in at the right face
      }
      const double d = pn - sm.phi[j * NT + t];
      sm.phi[j * NT + t] = pn;
      sm.q2[j * NT + t] = fma(ssv[j], pn, srcv[j]);  // emission of the next sweep
      return d;
    };
    const bool full = c0 + K <= Nc;
    if (cfg.norm == 0) {
      if (full) {
#pragma unroll
        for (int j = 0; j < K; ++j) {
          double pn;
          const double d = phi_cell(j, pn);
          num = absmax_acc(num, d);
          den = absmax_acc(den, pn);
        }
      } else {
#pragma unroll
        for (int j = 0; j < K; ++j)
          if (c0 + j < Nc) {
            double pn;
            const double d = phi_cell(j, pn);
            num = absmax_acc(num, d);
            den = absmax_acc(den, pn);
          }
      }
    } else {
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (c0 + j < Nc) {
          double pn;
          const double d = phi_cell(j, pn);
          num = fma(d, d, num);
          den = fma(pn, pn, den);
        }
    }
    reduce2<NT, CL>(num, den, cfg.norm == 0, sm.red, sm.cred, rphase++, sm);
    }
    SNOP_TSTAMP(ti2);
    SNOP_TACC(6, ti1, ti2);
    if (cfg.norm == 0) {
      bool nan;
      const bool done = linf_converged(num, den, cfg.tol, nan);
      if (nan) break;  // NaN: stop, reported non-converged
      if (done) {
        conv = true;
        break;
      }
    } else {
      const double rel = rel_change(num, den, cfg.norm);
      if (!(rel == rel)) break;
      if (rel < cfg.tol) {
        conv = true;
        break;
      }
    }
  }
  if (WJ && io.leak) {  // balance diagnostic: net leakages of the last sweep
    if (c0 == 0) io.leak[0] = sm.leak[0];  // written by this same thread: no barrier needed
    if (w.owns_last) io.leak[1] = sm.leak[1];
  }
  if constexpr (PS) {  // the owners' final phi -> every CTA
    const int prank = cl_rank(), psz = cl_size(), per = NT / psz;
    for (int idx = t; idx < per * K; idx += NT) {
      const int j = idx / per, u = prank * per + (idx - j * per);
      if (u * K + j < Nc) {
        const int o = j * NT + u;
        const double v = sm.phi[o];
        for (int r = 0; r < psz; ++r) cl_map(sm.phi, r)[o] = v;
      }
    }
  }
  if constexpr (CL || PS) cl_sync();  // keep shared memory alive until every remote access is done
  *converged = conv;
  return it;
}

}  // namespace snop_dev
