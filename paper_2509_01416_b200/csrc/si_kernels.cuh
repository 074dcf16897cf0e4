// si_kernels.cuh — K1 (fused fixed-source source iteration) and K2 (fused power iteration,
// single- and multi-group) for sm_100a. One CTA (or, CL = true, one thread-block cluster of CS
// CTAs, cells split across SMs and joined through DSMEM) = one instance for the whole solve;
// see snop_device.cuh and DESIGN.md §K1/§K2.
#pragma once

#include <cmath>
#include <cstdlib>

#include "snop_internal.h"

namespace snop_si {
using namespace snop_dev;

// Cells per thread of the one-CTA-per-instance layout (8; experiment builds may override).
#ifndef SNOP_K
#define SNOP_K 8
#endif

// Register budget: 128 regs/thread (16 resident warps per SM at NT * minBlocks = 512).
#ifndef SNOP_WARPS_PER_SM
#define SNOP_WARPS_PER_SM 16
#endif
template <int K, int NT>
constexpr int min_blocks() {
  return (SNOP_WARPS_PER_SM * 32) / NT > 0 ? (SNOP_WARPS_PER_SM * 32) / NT : 1;
}

template <int K, int NT>
size_t smem_bytes() {
  return sizeof(SweepSmem<K, NT>);
}

// instance index and cluster rank of this CTA
template <bool CL>
__device__ __forceinline__ void instance_of_block(int& b, int& rank) {
  if constexpr (CL) {
    rank = cl_rank();
    b = blockIdx.x / cl_size();
  } else {
    rank = 0;
    b = blockIdx.x;
  }
}

// ---------------------------------------------------------------------------------------------
// K1: batched fixed-source solve.
// ---------------------------------------------------------------------------------------------
template <int K, int NT, bool ANISO, bool CUR, bool CL>
__global__ void __launch_bounds__(NT, min_blocks<K, NT>())
si_fixed_source_kernel(const __grid_constant__ SweepConsts sc, const SolveConfig cfg,
                       const double* __restrict__ st_g, const double* __restrict__ ss0_g,
                       const double* __restrict__ ss1_g, const double* __restrict__ src_g,
                       const double* __restrict__ phi0_g, double* __restrict__ phi_g,
                       double* __restrict__ jc_g, int32_t* __restrict__ iters, uint8_t* __restrict__ conv,
                       int* __restrict__ flags, const int* __restrict__ order, double* __restrict__ leak_g,
                       double* __restrict__ stage_g, const uint8_t* __restrict__ active) {
  extern __shared__ __align__(32) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<SweepSmem<K, NT>*>(smem_raw);
  const int t = threadIdx.x, Nc = sc.n_cells;
  int b, rank;
  instance_of_block<CL>(b, rank);
  if (order) b = order[b];  // longest-expected-first dispatch (see launch_si_t)
  if (active && !active[b]) return;  // frozen instance of a device loop: outputs left as they are
  const size_t base = (size_t)b * Nc;
  const int c0 = rank * NT * K + t * K;
  CellIO io;
  io.ss0 = ss0_g + base;
  io.src = src_g + base;
  io.ss1 = ANISO ? ss1_g + base : nullptr;
  io.jc = ((ANISO || CUR) && jc_g) ? jc_g + base : nullptr;  // CUR without jc: leakages only
  io.leak = leak_g ? leak_g + 2 * (size_t)b : nullptr;
  bool bad = false;
  if (!CL && stage_g) {
    // Inputs (and outputs) in pinned host memory, read over the bus by the kernel itself: one
    // coalesced pass copies the per-iteration operands (Ss0, S, Ss1) into this instance's rows of
    // a device workspace and Sigma_t / phi0 into shared memory, so the transfer of later
    // instances overlaps the solves of earlier ones.
    constexpr int R = ANISO ? 3 : 2;
    double* ws = stage_g + (size_t)b * R * Nc;
    for (int i = t; i < NT * K; i += NT) {
      const int owner = i / K, j = i - owner * K;
      double stv = 0.0, p0 = 0.0;  // padding: identity map (see maps_phase)
      if (i < Nc) {
        ws[i] = ss0_g[base + i];
        ws[Nc + i] = src_g[base + i];
        if constexpr (ANISO) ws[2 * Nc + i] = ss1_g[base + i];
        stv = st_g[base + i];
        bad |= !(stv > 0.0);
        p0 = phi0_g ? phi0_g[base + i] : 0.0;
      }
      sm.st[j * NT + owner] = stv;
      sm.phi[j * NT + owner] = p0;
    }
    io.ss0 = ws;
    io.src = ws + Nc;
    if constexpr (ANISO) io.ss1 = ws + 2 * Nc;
    if constexpr (ANISO) {
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (c0 + j < Nc) io.jc[c0 + j] = 0.0;
    }
    __syncthreads();
  } else {
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int i = c0 + j;
      if (i < Nc) {
        const double stv = st_g[base + i];
        sm.st[j * NT + t] = stv;
        bad |= !(stv > 0.0);
        sm.phi[j * NT + t] = phi0_g ? phi0_g[base + i] : 0.0;
        if constexpr (ANISO) io.jc[i] = 0.0;
      } else {
        sm.st[j * NT + t] = 0.0;  // padding: identity map (see maps_phase)
        sm.phi[j * NT + t] = 0.0;
      }
    }
  }
  if (cluster_any<NT, CL>(bad, sm)) {  // nonpositive Sigma_t -> invalid argument
    if (t == 0 && rank == 0) {
      atomicOr(flags, snop_impl::FLAG_BAD_SIGMA_T);
      iters[b] = 0;
      conv[b] = 0;
    }
    return;
  }
  bool converged = false;
  const int it = si_solve<K, NT, ANISO, CUR, CL>(sc, cfg, sm, io, &converged);
  if (!CL && stage_g) {  // coalesced write-back (host memory: full bus transactions)
    __syncthreads();
    for (int i = t; i < Nc; i += NT) phi_g[base + i] = sm.phi[(i % K) * NT + i / K];
  } else {
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int i = c0 + j;
      if (i < Nc) phi_g[base + i] = sm.phi[j * NT + t];
    }
  }
  if (t == 0 && rank == 0) {
    iters[b] = it;
    conv[b] = converged ? 1 : 0;
  }
}

// ---------------------------------------------------------------------------------------------
// K2: batched k-eigenvalue power iteration, SPEC.md:179-189 + decisions :206-209, SURVEY §9 #5
// (Gauss-Seidel over groups with upscatter, newest flux), #10 (inner solves warm-started).
// The fission source, inscatter source, k update, renormalisation and dual convergence test are
// all fused into the same persistent CTA / cluster. Group fluxes live in the output array
// (L2-resident, thread-private cells), the previous-outer copy in a workspace.
// ---------------------------------------------------------------------------------------------
// The inner solver is called through a non-inlined boundary: the outer loop's live state is
// saved once per group solve instead of competing with the sweep's maps for registers.
template <int K, int NT, bool ANISO, bool CL, bool PS = false>
__device__ __noinline__ int si_solve_call(const SweepConsts& sc, const SolveConfig& cfg, SweepSmem<K, NT>& sm,
                                          const CellIO& io) {
  bool c = false;
  return si_solve<K, NT, ANISO, false, CL, SNOP_NP, PS>(sc, cfg, sm, io, &c);
}

struct EigenParams {
  int G;
  double tol_k, tol_phi;
  int max_outer;
  int norm;
};

// PS = pair-split cluster (see si_solve): every CTA of the cluster runs the whole outer loop
// redundantly on private working copies of phi / old / q_ext (ranks > 0 in psw_g), only the inner
// sweeps are divided; rank 0 owns the outputs.
// WIDE: one CTA per SM is enough (the batch fits the SMs in one wave), so the register cap of the
// two-CTAs-per-SM build (128; the eigen kernel spills ~450 B per thread under it) is lifted: no
// spills, same arithmetic (C4, one wave of 128 CTAs: 27.6 -> 23.6 ms).
template <int K, int NT, bool ANISO, bool CL, bool PS = false, bool WIDE = false>
__global__ void __launch_bounds__(NT, WIDE ? 1 : min_blocks<K, NT>())
power_iteration_kernel(const __grid_constant__ SweepConsts sc, const SolveConfig icfg, const EigenParams ep,
                       const double* __restrict__ st_g, const double* __restrict__ ss0_g,
                       const double* __restrict__ ss1_g, const double* __restrict__ nsf_g,
                       const double* __restrict__ chi_g, const double* __restrict__ k0_g,
                       const double* __restrict__ phi0_g, double* __restrict__ k_g, double* __restrict__ phi_g,
                       double* __restrict__ old_g, double* __restrict__ qext_g, double* __restrict__ jc_g,
                       int32_t* __restrict__ outer_g, int64_t* __restrict__ inner_g,
                       uint8_t* __restrict__ conv_g, int* __restrict__ flags, double* __restrict__ psw_g,
                       const int* __restrict__ order, const int* __restrict__ order_count, int resume,
                       float* __restrict__ tail_key) {
  static_assert(!(PS && (CL || ANISO)), "pair split: isotropic, no cell split");
  extern __shared__ __align__(32) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<SweepSmem<K, NT>*>(smem_raw);
  const int t = threadIdx.x, Nc = sc.n_cells, G = ep.G;
  int b, rank;
  if constexpr (PS) {
    rank = cl_rank();
    b = blockIdx.x / cl_size();
  } else {
    instance_of_block<CL>(b, rank);
  }
  if (order) {  // sub-batch through an instance list (tail phase); the whole cluster leaves together
    if (b >= *order_count) return;
    b = order[b];
  }
  // resume (tail phase): continue the iteration counts of an earlier launch of the same solve
  const int outer0 = resume ? outer_g[b] : 0;
  const int64_t inner0 = resume ? inner_g[b] : 0;
  const int cb = CL ? rank * NT * K : 0;  // first cell of this CTA (cell split only)
  const int c0 = cb + t * K;
  const size_t GN = (size_t)G * Nc;
  const double* st_b = st_g + (size_t)b * GN;
  const double* ss_b = ss0_g + (size_t)b * GN * G;
  const double* nsf_b = nsf_g + (size_t)b * GN;
  double* phi_b = phi_g + (size_t)b * GN;
  double* old_b = old_g + (size_t)b * GN;
  double* qext_b = qext_g + (size_t)b * Nc;
  if constexpr (PS) {
    if (rank > 0) {
      double* wsp = psw_g + ((size_t)b * (cl_size() - 1) + rank - 1) * (2 * GN + Nc);
      phi_b = wsp;
      old_b = wsp + GN;
      qext_b = wsp + 2 * GN;
    }
  }
  double* jc_b = ANISO ? jc_g + (size_t)b * Nc : nullptr;
  auto cell = [&](int g, int j) -> size_t { return (size_t)g * Nc + c0 + j; };
  // Coalesced mapping for the per-cell outer-loop work (fission density, in-scatter source,
  // renormalisation): r-th cell of thread t = cb + r * NT + t, so a warp touches 256 contiguous
  // bytes per load; the thread-owned chunk mapping (c0 + j) is kept for shared-memory staging.
  auto cc = [&](int r) -> int { return cb + r * NT + t; };

  // validation + initial flux (flat) and k
  bool bad = false;
  for (int g = 0; g < G; ++g) {
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (c0 + j < Nc) {
        bad |= !(st_b[cell(g, j)] > 0.0);
        phi_b[cell(g, j)] = phi0_g ? phi0_g[(size_t)b * GN + cell(g, j)] : 1.0;
      }
    }
  }
  double k = k0_g ? k0_g[b] : 1.0;
  // pair split: phi0 may alias rank 0's working array (resume) -> every rank has its copy first
  if constexpr (PS) cl_sync();
  int rphase = 0;
  // Loops over groups are outermost and the thread's K cells innermost (unrolled) throughout: the
  // per-group global loads of all K cells are then independent and in flight together, instead of
  // one dependent L2 round trip per (cell, group). Per-cell summation order is unchanged (g ascending).
  auto fission_integral = [&]() {
    double f[K];
#pragma unroll
    for (int r = 0; r < K; ++r) f[r] = 0.0;
#pragma unroll 2
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int r = 0; r < K; ++r)
        if (cc(r) < Nc) f[r] = fma(nsf_b[(size_t)g * Nc + cc(r)], phi_b[(size_t)g * Nc + cc(r)], f[r]);
    }
    double s = 0.0, dummy = 0.0;
#pragma unroll
    for (int r = 0; r < K; ++r)
      if (cc(r) < Nc) s += f[r];
    reduce2<NT, CL>(s, dummy, false, sm.red2, sm.cred2, rphase++, sm);
    return s * sc.dx;
  };
  int64_t inner_total = 0;
  int outer = 0;
  auto fail = [&](int flag) {
    if (t == 0 && rank == 0) {
      atomicOr(flags, flag);
      k_g[b] = __longlong_as_double(0x7ff8000000000000ll);
      outer_g[b] = outer0 + outer;  // counts so far (a resumed phase keeps the earlier phase's)
      inner_g[b] = inner0 + inner_total;
      conv_g[b] = 0;
    }
    if constexpr (CL) cl_sync();  // no CTA of the cluster leaves while others may read its smem
  };
  if (cluster_any<NT, CL>(bad, sm) || !(k > 0.0)) {
    fail(snop_impl::FLAG_BAD_SIGMA_T);
    return;
  }
  if (!resume) {  // a resumed phase continues from the already normalised flux of the earlier phase
    const double F = fission_integral();
    if (!(F != 0.0) || !isfinite(F)) {
      fail(snop_impl::FLAG_DEGENERATE);
      return;
    }
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int r = 0; r < K; ++r)
        if (cc(r) < Nc) phi_b[(size_t)g * Nc + cc(r)] /= F;
  }
  // coalesced-mapped writes above -> owner-mapped reads of the first group's staging below
  __syncthreads();

  bool converged = false;
  double gap = 0.0;  // distance from the dual test at the last outer: max(dk / tol_k, dphi / tol_phi)
  double gap4 = -1.0;  // the same 4 outers before the end of this launch (convergence-rate estimate)
  SNOP_TSTAMP(tpi0);
  while (outer < ep.max_outer) {
    ++outer;
    // fission density from the flux at the start of the outer (frozen during the GS pass)
    double fiss[K];
#pragma unroll
    for (int j = 0; j < K; ++j) fiss[j] = 0.0;
#pragma unroll 2
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int r = 0; r < K; ++r) {
        if (cc(r) < Nc) {
          const size_t i = (size_t)g * Nc + cc(r);
          const double v = phi_b[i];
          old_b[i] = v;
          fiss[r] = fma(nsf_b[i], v, fiss[r]);
        }
      }
    }
    const double inv_k = 1.0 / k;
    for (int g = 0; g < G; ++g) {
      SNOP_TSTAMP(tq0);
      const double chig = chi_g[(size_t)b * G + g] * inv_k;
      double q[K];
#pragma unroll
      for (int j = 0; j < K; ++j) q[j] = chig * fiss[j];
#pragma unroll 2
      for (int gp = 0; gp < G; ++gp) {
        if (gp == g) continue;
#pragma unroll
        for (int r = 0; r < K; ++r)
          if (cc(r) < Nc)
            q[r] = fma(ss_b[((size_t)gp * G + g) * Nc + cc(r)], phi_b[(size_t)gp * Nc + cc(r)], q[r]);
      }
#pragma unroll
      for (int r = 0; r < K; ++r) {
        if (cc(r) < Nc) {
          qext_b[cc(r)] = q[r];
          if constexpr (ANISO) jc_b[cc(r)] = 0.0;
        }
      }
      // (si_solve's entry barrier orders these coalesced writes before the owner-mapped reads)
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (c0 + j < Nc) {
          const size_t i = (size_t)c0 + j;
          sm.st[j * NT + t] = st_b[(size_t)g * Nc + i];
          sm.phi[j * NT + t] = phi_b[(size_t)g * Nc + i];
        } else {
          sm.st[j * NT + t] = 0.0;  // padding: identity map (see maps_phase)
          sm.phi[j * NT + t] = 0.0;
        }
      }
      CellIO io;
      io.ss0 = ss_b + ((size_t)g * G + g) * Nc;
      io.src = qext_b;
      io.ss1 = ANISO ? ss1_g + (size_t)b * GN + (size_t)g * Nc : nullptr;
      io.jc = jc_b;
      SNOP_TSTAMP(tsol0);
      SNOP_TACC(9, tq0, tsol0);
      inner_total += si_solve_call<K, NT, ANISO, CL, PS>(sc, icfg, sm, io);
      SNOP_TSTAMP(tsol1);
      SNOP_TACC(7, tsol0, tsol1);
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (c0 + j < Nc) phi_b[cell(g, j)] = sm.phi[j * NT + t];
      __syncthreads();  // owner-mapped writes -> coalesced reads of the next group / the update
    }
    const double F1 = fission_integral();
    if (!(F1 != 0.0) || !isfinite(F1)) {
      fail(snop_impl::FLAG_DEGENERATE);
      return;
    }
    const double k_new = k * F1;
    double num = 0.0, den = 0.0;
#pragma unroll 2
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int r = 0; r < K; ++r) {
        if (cc(r) < Nc) {
          const size_t i = (size_t)g * Nc + cc(r);
          const double pn = phi_b[i] / F1;
          phi_b[i] = pn;
          const double d = pn - old_b[i];
          if (ep.norm == 0) {
            num = fmax(num, fabs(d));
            den = fmax(den, fabs(pn));
          } else {
            num = fma(d, d, num);
            den = fma(pn, pn, den);
          }
        }
      }
    }
    reduce2<NT, CL>(num, den, ep.norm == 0, sm.red2, sm.cred2, rphase++, sm);
    const double dphi = rel_change(num, den, ep.norm);
    const double dk = fabs(k_new - k) / fabs(k_new);
    k = k_new;
    gap = fmax(dk / ep.tol_k, dphi / ep.tol_phi);
    if (outer == ep.max_outer - 4) gap4 = gap;
    if (dk < ep.tol_k && dphi < ep.tol_phi) {
      converged = true;
      break;
    }
  }
  SNOP_TSTAMP(tpi1);
  SNOP_TACC(8, tpi0, tpi1);
  if (t == 0 && rank == 0) {
    k_g[b] = k;
    outer_g[b] = outer0 + outer;
    inner_g[b] = inner0 + inner_total;
    conv_g[b] = converged ? 1 : 0;
    if (tail_key) {  // predicted remaining outers (tail-phase routing and order, launch_power_iteration)
      double rem = gap;
      if (gap4 > 0.0 && gap > 0.0) {  // geometric convergence: gap ~ rho^n -> n_rem = log(gap) / -log(rho)
        const double rho = fmin(fmax(pow(gap / gap4, 0.25), 1e-6), 1.0 - 1e-9);
        rem = log(fmax(gap, 1.0)) / -log(rho);
      }
      tail_key[b] = converged ? 0.f : (float)fmin(rem, 3.0e38);
    }
  }
  if constexpr (CL) cl_sync();
}

// ---------------------------------------------------------------------------------------------
// Dispatch order for K1: instances with a larger scattering ratio need more source iterations
// (the iteration matrix has spectral radius ~ max sigma_s0/sigma_t), so launching them first
// shortens the tail of the batch. Any permutation gives identical per-instance results.
// key_b = max_i Ss0_i / St_i, quantised into NBUCKET buckets, bucket sort (descending).
// ---------------------------------------------------------------------------------------------
constexpr int NBUCKET = 1024;

static __global__ void order_keys_kernel(int Nc, const double* __restrict__ st, const double* __restrict__ ss,
                                  int* __restrict__ bucket, int* __restrict__ hist, int sampled) {
  const int b = blockIdx.x;
  double m = 0.0;
  if (sampled && Nc > (int)blockDim.x) {
    // host-resident inputs: 4 contiguous runs of blockDim/4 cells spread over the slab (whole bus
    // transactions instead of one per strided cell)
    const int run = blockDim.x / 4, r = threadIdx.x / run;
    const int i = (int)((long long)r * (Nc - run) / 3) + (int)(threadIdx.x % run);
    const double t = st[(size_t)b * Nc + i];
    if (t > 0.0) m = fmax(m, ss[(size_t)b * Nc + i] / t);
  } else {
    for (int i = threadIdx.x; i < Nc; i += blockDim.x) {
      const double t = st[(size_t)b * Nc + i];
      if (t > 0.0) m = fmax(m, ss[(size_t)b * Nc + i] / t);
    }
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double sh[32];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, sh[w]);
    m = fmin(fmax(m, 0.0), 1.0);
    const int k = NBUCKET - 1 - (int)fmin(m * (NBUCKET - 1), (double)(NBUCKET - 1));  // descending
    bucket[b] = k;
    atomicAdd(&hist[k], 1);
  }
}

static __global__ void order_scan_kernel(int* __restrict__ hist) {  // exclusive scan, one block of NBUCKET
  __shared__ int s[NBUCKET];
  const int t = threadIdx.x;
  s[t] = hist[t];
  __syncthreads();
  for (int o = 1; o < NBUCKET; o <<= 1) {
    const int v = t >= o ? s[t - o] : 0;
    __syncthreads();
    s[t] += v;
    __syncthreads();
  }
  hist[t] = t > 0 ? s[t - 1] : 0;
}

static __global__ void order_scatter_kernel(int B, const int* __restrict__ bucket, int* __restrict__ cursor,
                                     int* __restrict__ order) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) order[atomicAdd(&cursor[bucket[b]], 1)] = b;
}

// sampled = true when st / ss live in host memory: the key is taken over 128 sampled cells
// (it only steers dispatch order; results do not depend on it)
static inline const int* make_order(snop_impl::Ctx& ctx, int batch, int Nc, const double* st, const double* ss,
                                    bool sampled = false) {
  int* buf = static_cast<int*>(ctx.slot(23, ((size_t)2 * batch + NBUCKET) * sizeof(int)));
  if (!buf) return nullptr;
  int *bucket = buf, *order = buf + batch, *hist = buf + 2 * batch;
  cudaMemsetAsync(hist, 0, NBUCKET * sizeof(int), ctx.stream);
  order_keys_kernel<<<batch, 128, 0, ctx.stream>>>(Nc, st, ss, bucket, hist, sampled ? 1 : 0);
  order_scan_kernel<<<1, NBUCKET, 0, ctx.stream>>>(hist);
  order_scatter_kernel<<<(batch + 255) / 256, 256, 0, ctx.stream>>>(batch, bucket, hist, order);
  ctx.launches += 3;
  return cudaGetLastError() == cudaSuccess ? order : nullptr;
}

// Launch helper: plain launch for CS = 1, cluster launch (CS CTAs per instance) otherwise.
template <class Kern, class... Args>
inline cudaError_t launch_k(Kern kern, int batch, int cs, int nt, size_t smem, cudaStream_t s, Args... args) {
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cs <= 1) {
    kern<<<batch, nt, smem, s>>>(args...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(batch * cs));
  cfg.blockDim = dim3((unsigned)nt);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <int K, int NT, bool CL>
inline snop_status launch_si_t(snop_impl::Ctx& ctx, const SweepConsts& sc, const SolveConfig& cfg, int batch, int cs,
                               const double* st, const double* ss0, const double* ss1, const double* src,
                               const double* phi0, double* phi, double* cur, int32_t* iters, uint8_t* conv,
                               double* leak, double* stage, const uint8_t* active) {
  const bool aniso = ss1 != nullptr;
  const size_t smem = smem_bytes<K, NT>();
  // the edge currents are accumulated only when wanted: P1 emission, current output, leakages
  auto kern = aniso ? si_fixed_source_kernel<K, NT, true, true, CL>
                    : ((cur || leak) ? si_fixed_source_kernel<K, NT, false, true, CL>
                                     : si_fixed_source_kernel<K, NT, false, false, CL>);
  double* jc = cur;
  if (aniso && !jc) {  // P1 needs the cell current even when the caller does not want it
    jc = static_cast<double*>(ctx.slot(21, (size_t)batch * sc.n_cells * sizeof(double)));
    if (!jc) {
      snop_impl::set_error("cudaMalloc (current workspace) failed");
      return SNOP_CUDA_ERROR;
    }
  }
  // longest-expected-first order pays off once the batch spans several waves of CTAs
  const int* order =
      (!CL && batch > 4 * ctx.sm_count) ? make_order(ctx, batch, sc.n_cells, st, ss0, stage != nullptr) : nullptr;
  const cudaError_t e = launch_k(kern, batch, CL ? cs : 1, NT, smem, ctx.stream, sc, cfg, st, ss0, ss1, src, phi0,
                                 phi, jc, iters, conv, ctx.d_flags, order, leak, CL ? nullptr : stage, active);
  ctx.launches++;
  if (e != cudaSuccess) {
    snop_impl::set_error(std::string("si_fixed_source_kernel launch: ") + cudaGetErrorString(e));
    return SNOP_CUDA_ERROR;
  }
  return SNOP_OK;
}

template <int K, int NT, bool CL, bool PS = false>
inline snop_status launch_pi_t(snop_impl::Ctx& ctx, const SweepConsts& sc, const SolveConfig& icfg,
                               const EigenParams& ep, int batch, int cs, const double* st, const double* ss0,
                               const double* ss1, const double* nsf, const double* chi, const double* k0,
                               const double* phi0, double* k, double* phi, double* old, int32_t* outer,
                               int64_t* inner, uint8_t* conv, const int* order = nullptr,
                               const int* order_count = nullptr, int resume = 0, float* tail_key = nullptr) {
  const bool aniso = ss1 != nullptr;
  const size_t smem = smem_bytes<K, NT>();
  auto kern = PS ? power_iteration_kernel<K, NT, false, false, PS>
                 : (aniso ? power_iteration_kernel<K, NT, true, CL> : power_iteration_kernel<K, NT, false, CL>);
  if constexpr (!CL && !PS && (min_blocks<K, NT>() > 1)) {
    if (batch <= ctx.sm_count)  // one wave at one CTA per SM: the register-rich build
      kern = aniso ? power_iteration_kernel<K, NT, true, false, false, true>
                   : power_iteration_kernel<K, NT, false, false, false, true>;
  }
  if (PS && aniso) {
    snop_impl::set_error("pair-split eigen kernel is isotropic only");
    return SNOP_INVALID_ARGUMENT;
  }
  const size_t n = (size_t)batch * sc.n_cells;
  double* qext = static_cast<double*>(ctx.slot(22, n * sizeof(double)));
  double* jc = aniso ? static_cast<double*>(ctx.slot(21, n * sizeof(double))) : nullptr;
  double* psw = nullptr;
  if (PS && cs > 1) {  // private phi / old / q_ext of the ranks > 0
    const size_t GN = (size_t)ep.G * sc.n_cells;
    psw = static_cast<double*>(ctx.slot(27, (size_t)batch * (cs - 1) * (2 * GN + sc.n_cells) * sizeof(double)));
    if (!psw) {
      snop_impl::set_error("cudaMalloc (pair-split workspace) failed");
      return SNOP_CUDA_ERROR;
    }
  }
  if (!qext || (aniso && !jc)) {
    snop_impl::set_error("cudaMalloc (eigen workspace) failed");
    return SNOP_CUDA_ERROR;
  }
  const cudaError_t e = launch_k(kern, batch, (CL || PS) ? cs : 1, NT, smem, ctx.stream, sc, icfg, ep, st, ss0, ss1,
                                 nsf, chi, k0, phi0, k, phi, old, qext, jc, outer, inner, conv, ctx.d_flags, psw,
                                 order, order_count, resume, tail_key);
  ctx.launches++;
  if (e != cudaSuccess) {
    snop_impl::set_error(std::string("power_iteration_kernel launch: ") + cudaGetErrorString(e));
    return SNOP_CUDA_ERROR;
  }
  return SNOP_OK;
}

// Tail phase of a split power iteration: the instances still iterating after a launch (not
// converged, outer count == cap) -> list A (key > thresh) or list B (the rest; no list B: all in A),
// each ordered by key descending (ties by index): key = the predicted remaining outers, so the
// slowest instance gets its cluster first. Rank by counting (deterministic); an instance's list
// depends on its own key only, and positions never affect its results. cand (nullable): consider
// only the instances of that list (cand[0 .. *cand_count)), e.g. while other instances are still
// being solved by a concurrent launch.
static __global__ void pi_tail_list_kernel(int B, int cap, const int32_t* __restrict__ outer,
                                           const uint8_t* __restrict__ conv, const float* __restrict__ key,
                                           float thresh, int* __restrict__ orderA, int* __restrict__ countA,
                                           int* __restrict__ orderB, int* __restrict__ countB,
                                           const int* __restrict__ cand = nullptr,
                                           const int* __restrict__ cand_count = nullptr) {
  const int n = cand ? *cand_count : B;
  auto in = [&](int c) { return !conv[c] && outer[c] == cap; };
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int b = cand ? cand[i] : i;
    if (!in(b)) continue;
    const float kb = key[b];
    const bool a = !orderB || kb > thresh;
    atomicAdd(a ? countA : countB, 1);
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const int c = cand ? cand[j] : j;
      if (in(c) && ((!orderB || key[c] > thresh) == a) && (key[c] > kb || (key[c] == kb && c < b))) ++rank;
    }
    (a ? orderA : orderB)[rank] = b;
  }
}

// K1 for slabs of any length (streaming, per-cell state in a global workspace): si_tiled.cu.
template <int K, int NT>
snop_status launch_tiled_t(snop_impl::Ctx& ctx, const SweepConsts& sc, const SolveConfig& cfg, int batch,
                           const double* st, const double* ss0, const double* ss1, const double* src,
                           const double* phi0, double* phi, double* cur, int32_t* iters, uint8_t* conv,
                           double* leak, const uint8_t* active);

// Explicitly instantiated in si_k8_{fixed,eigen}{,_cl}.cu (one TU per variant, parallel build).
#define SNOP_SI_ARGS                                                                                          \
  snop_impl::Ctx&, const SweepConsts&, const SolveConfig&, int, int, const double*, const double*, const double*, \
      const double*, const double*, double*, double*, int32_t*, uint8_t*, double*, double*, const uint8_t*
#define SNOP_PI_ARGS                                                                                          \
  snop_impl::Ctx&, const SweepConsts&, const SolveConfig&, const EigenParams&, int, int, const double*,          \
      const double*, const double*, const double*, const double*, const double*, const double*, double*, double*, \
      double*, int32_t*, int64_t*, uint8_t*, const int*, const int*, int, float*
#define SNOP_DECL_SI(KK, NN, CC) extern template snop_status launch_si_t<KK, NN, CC>(SNOP_SI_ARGS);
#define SNOP_DECL_PI(KK, NN, CC) extern template snop_status launch_pi_t<KK, NN, CC>(SNOP_PI_ARGS);
#define SNOP_DECL_PS(KK, NN) extern template snop_status launch_pi_t<KK, NN, false, true>(SNOP_PI_ARGS);
#define SNOP_INST_PS(KK, NN) template snop_status launch_pi_t<KK, NN, false, true>(SNOP_PI_ARGS);
#define SNOP_INST_SI(KK, NN, CC) template snop_status launch_si_t<KK, NN, CC>(SNOP_SI_ARGS);
#define SNOP_INST_PI(KK, NN, CC) template snop_status launch_pi_t<KK, NN, CC>(SNOP_PI_ARGS);

}  // namespace snop_si
