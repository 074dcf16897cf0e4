// sweep.cu — the standalone transport sweep as a streaming sm_100a kernel.
//
// One diamond-difference sweep of all N directions of B instances with a PER-DIRECTION emission:
//   psi_avg = (q + c psi_in) / (Sigma_t + c),  psi_out = 2 psi_avg - psi_in,  c = 2|mu|/dx.
// Unlike the fused solvers (K1/K2), which never materialise psi, this operator reads the
// emission q(x_i, mu_n) and writes the cell-average angular flux for every cell and direction:
// 16 B of HBM traffic per cell.angle update (+ Sigma_t, 8 B per cell, served once from DRAM and
// then from L1/L2), so it is HBM-bound and is measured against the copy roofline.
//
// Mapping. Thread = one direction of one instance, marching the slab (mu > 0 left to right,
// mu < 0 right to left): B*N chains are the parallelism (65536 for BASELINE C2/C5), CTA = one
// warp, so the grid balances over the 148 SMs at ~14 resident warps each. The recurrence is serial
// in the cell index but needs one dependent 3-instruction chain per cell; everything else
// (reciprocal, loads, stores) is off the chain. A reflective face makes the directions of one sign
// wait for the others' outflow (SURVEY §9 #2 ordering): two launches, the second reading its
// inflows from the first one's outflow workspace.
//   * loads: emission [B][Nc][N] makes the N/2 same-sign directions of a cell contiguous, so the
//     lanes of an instance read one segment per cell. Each thread copies its own q and Sigma_t
//     values with 8-byte cp.async into a private slot of an S-stage shared-memory ring (tiles of
//     T cells), S-1 tiles ahead: bytes in flight without holding registers.
//   * stores: psi_avg [B][N][Nc] is direction-major, so a thread's T results of a tile are
//     contiguous but the lanes are Nc apart: the warp transposes each tile through shared memory
//     and writes whole rows (T contiguous cells per row, 32/T rows per instruction).
//   * partial currents: every chain's outflow goes to a workspace [B][N]; a tiny kernel forms
//     w mu (psi_out - psi_in) per pair and sums the pairs of an instance in ascending order
//     (deterministic, the oracle's order).
#include <mutex>
#include <string>

#define SNOP_PHASE_SYM g_phase_cycles_sweep
#include "snop_internal.h"

using namespace snop_impl;
using namespace snop_dev;

namespace {

constexpr int kS = 4;   // ring stages (kS - 1 tiles of T = 8 or 16 cells in flight per warp)
constexpr int kG = 16;  // most (instance, sign) groups a warp can span on the vector path (N/2 >= 2)

// V16 = false (any order / cell count / alignment): every thread copies its own q and Sigma_t
// values with 8-byte cp.async. V16 = true (N/2 a power of two, even cell count, 16-byte aligned
// arrays): even lanes copy the q of a lane pair (adjacent directions) with 16-byte cp.async.cg
// (8-byte cp.async.ca serialises its shared-memory writes: 17 wavefronts per request in ncu, the
// LSU data pipe at 87%), and Sigma_t is copied once per (instance, sign) group of the warp.
template <bool V16, int T>
struct SweepTileSmem {
  double q[kS][T][32];                           // emission, [stage][cell in sweep order][lane]
  double st[kS][V16 ? kG : T][V16 ? T : 32];    // Sigma_t: [..][group][ascending cell] or [..][cell][lane]
  double out[32][T + 1];                         // psi_avg of the current tile, [lane][cell] (+1: conflict-free)
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 8 : 0;  // src-size 0: zero fill (cells beyond the slab)
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Directions [n_lo, n_lo + n_cnt) of every instance; chain gt = b * n_cnt + (n - n_lo). infl: null
// (vacuum inflow) or the outflow workspace of the previous launch (inflow of direction n = outflow
// of its mirror image N-1-n at the same face).
template <bool V16, int T>
__global__ void __launch_bounds__(32, T == 8 ? 14 : 7)
sweep_kernel(const __grid_constant__ SweepConsts sc, int batch, int order, int n_lo, int n_cnt,
             const double* __restrict__ st_g, const double* __restrict__ em_g, double* __restrict__ psi,
             const double* __restrict__ infl, double* __restrict__ outw /* [B][N] */, int* __restrict__ flags) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<SweepTileSmem<V16, T>*>(smem_raw);
  const int lane = threadIdx.x, Nc = sc.n_cells, H = sc.n_pairs, N = order;
  const long long total = (long long)batch * n_cnt;
  const long long gt = (long long)blockIdx.x * 32 + lane;
  const bool valid = gt < total;
  const long long g = valid ? gt : total - 1;
  const int b = (int)(g / n_cnt), n = n_lo + (int)(g - (long long)b * n_cnt);
  const bool fwd = n >= H;
  const double c = sc.c[fwd ? n - H : H - 1 - n];
  const double* st_b = st_g + (size_t)b * Nc;
  const double* em_n = em_g + (size_t)b * Nc * N + n;
  const size_t row = valid ? ((size_t)b * N + n) * Nc : ~(size_t)0;
  // vector path: the lanes of this warp that share (instance, sign) (N/2 a power of two)
  const int hw = H < 32 ? H : 32;
  const int grp = V16 ? lane / hw : 0, grank = lane % hw;
  const int ntiles = (Nc + T - 1) / T, nfull = Nc / T;

  // Loop-invariant addressing (the kernel was issue-bound at ~66 instructions per cell with the
  // addresses and bounds recomputed per cell): global q pointer of tile 0 / cell 0 and its
  // per-cell and per-tile steps; Sigma_t tile read offsets; write-out row pointers.
  const long long dq = fwd ? (long long)N : -(long long)N;       // doubles per cell step
  const double* qp = em_n + (fwd ? 0 : (size_t)(Nc - 1) * N);    // cell of sweep step 0
  const int xr = fwd ? 0 : 1;  // V16: a backward group's tile is stored ascending: sweep step j at j ^ 1 of
                               // the reversed pair order (see issue()), i.e. compile-time j +- xr
  constexpr int RPI = 32 / T;
  const int e = lane % T, rsub = lane / T;
  const unsigned fwd_mask = __ballot_sync(0xffffffffu, fwd);
  double* wb[T];     // row r = it * RPI + rsub: address of this lane's element in the row's current tile
  int wo[T];         // its index in sm.out
  unsigned rfw = 0, rok = 0;
#pragma unroll
  for (int it = 0; it < T; ++it) {
    const int r = it * RPI + rsub;
    const size_t base = __shfl_sync(0xffffffffu, (unsigned long long)row, r);
    const bool rf = (fwd_mask >> r) & 1u;
    rfw |= (rf ? 1u : 0u) << it;
    rok |= (base != ~(size_t)0 ? 1u : 0u) << it;
    wb[it] = psi + (base != ~(size_t)0 ? base : 0) + e + (rf ? 0 : Nc - T);
    wo[it] = r * (T + 1) + (rf ? e : T - 1 - e);
  }
  double* const outp = &sm.out[0][0];

  // Sigma_t tile copies of the vector path: lane rank r of a group copies cell pair r (and, in
  // 2-lane groups, also pair r + 2) of the group's 8-cell tile; a backward group stores the pairs in
  // descending order, so sweep step j reads slot j ^ 1.
  constexpr int NCP = T / 4;  // most Sigma_t copies per lane (2-lane groups)
  auto issue = [&](int k) {
    if (k < ntiles) {
      const int slot = k % kS;
      const double* src = qp + (long long)k * T * dq;
      const int a0 = fwd ? k * T : Nc - (k + 1) * T;  // first (ascending) cell of the group's tile
      if (k < nfull) {  // interior tile: no bounds to check
        if constexpr (V16) {
          if ((lane & 1) == 0) {  // q of this lane and the next (adjacent directions, same cell)
#pragma unroll
            for (int j = 0; j < T; ++j) {
              cp_async16(&sm.q[slot][j][lane], src, valid);
              src += dq;
            }
          }
#pragma unroll
          for (int cpy = 0; cpy < NCP; ++cpy) {
            const int m2 = grank + cpy * hw;
            if (m2 < T / 2)
              cp_async16(&sm.st[slot][grp][fwd ? 2 * m2 : T - 2 - 2 * m2], st_b + a0 + 2 * m2, valid);
          }
        } else {
#pragma unroll
          for (int j = 0; j < T; ++j) {
            cp_async8(&sm.q[slot][j][lane], src, valid);
            cp_async8(&sm.st[slot][j][lane], st_b + (fwd ? a0 + j : a0 + T - 1 - j), valid);
            src += dq;
          }
        }
      } else {  // ragged last tile
        if constexpr (V16) {
          if ((lane & 1) == 0) {
#pragma unroll
            for (int j = 0; j < T; ++j) {
              const bool ok = valid && k * T + j < Nc;
              cp_async16(&sm.q[slot][j][lane], ok ? src : em_n, ok);
              src += dq;
            }
          }
          for (int m2 = grank; m2 < T / 2; m2 += hw) {
            const int i = a0 + 2 * m2;
            const bool ok = valid && i >= 0 && i < Nc;  // (even Nc and T: a pair is never split)
            cp_async16(&sm.st[slot][grp][fwd ? 2 * m2 : T - 2 - 2 * m2], st_b + (ok ? i : 0), ok);
          }
        } else {
#pragma unroll
          for (int j = 0; j < T; ++j) {
            const int sidx = k * T + j, i = fwd ? sidx : Nc - 1 - sidx;
            const bool ok = valid && sidx < Nc;
            cp_async8(&sm.q[slot][j][lane], ok ? src : em_n, ok);
            cp_async8(&sm.st[slot][j][lane], st_b + (ok ? i : 0), ok);
            src += dq;
          }
        }
      }
    }
    cp_async_commit();  // (an empty group past the last tile keeps the wait count uniform)
  };

#pragma unroll
  for (int k = 0; k < kS - 1; ++k) issue(k);
  double psi_e = infl ? infl[(size_t)b * N + (N - 1 - n)] : 0.0;  // edge flux entering the next cell
  bool bad = false;
  auto cell = [&](int slot, int j) {
    double s;
    if constexpr (V16) s = (&sm.st[slot][grp][0])[(j & 1) ? j - xr : j + xr];
    else s = sm.st[slot][j][lane];
    const double q = sm.q[slot][j][lane];
    bad |= !(s > 0.0);
    const double avg = fma(c, psi_e, q) * rcp_fast(s + c);
    psi_e = fma(2.0, avg, -psi_e);
    sm.out[lane][j] = avg;
  };
  for (int k = 0; k < ntiles; ++k) {
    issue(k + kS - 1);
    cp_async_wait<kS - 1>();          // this thread's copies of tile k have landed
    if constexpr (V16) __syncwarp();  // ... and the other lanes' (pair partner, Sigma_t tile)
    const int slot = k % kS;
    if (k < nfull) {
      // all loads, then the independent part (reciprocals, q r, c r), then the dependent chain:
      // written out in phases because the compiler otherwise serialises the cells (each cell's
      // loads after the previous cell's store)
      double sv[T], qv[T];
#pragma unroll
      for (int j = 0; j < T; ++j) {
        if constexpr (V16) sv[j] = (&sm.st[slot][grp][0])[(j & 1) ? j - xr : j + xr];
        else sv[j] = sm.st[slot][j][lane];
        qv[j] = sm.q[slot][j][lane];
      }
#pragma unroll
      for (int j = 0; j < T; ++j) {
        bad |= !(sv[j] > 0.0);
        const double r = rcp_fast(sv[j] + c);
        qv[j] *= r;     // q r
        sv[j] = c * r;  // c r
      }
#pragma unroll
      for (int j = 0; j < T; ++j) {
        const double avg = fma(sv[j], psi_e, qv[j]);  // (q + c psi_in) r
        psi_e = fma(2.0, avg, -psi_e);
        qv[j] = avg;
      }
#pragma unroll
      for (int j = 0; j < T; ++j) sm.out[lane][j] = qv[j];
      __syncwarp();
      // write-out: 32/T rows of T contiguous cells per instruction; the row pointers advance by
      // one tile in their sweep direction
#pragma unroll
      for (int it = 0; it < T; ++it) {
        const double v = outp[wo[it]];
        if ((rok >> it) & 1u) __stcs(wb[it], v);
        wb[it] += ((rfw >> it) & 1u) ? T : -T;
      }
    } else {  // ragged last tile
#pragma unroll
      for (int j = 0; j < T; ++j)
        if (k * T + j < Nc) cell(slot, j);
      __syncwarp();
#pragma unroll
      for (int it = 0; it < T; ++it) {
        const bool rf = (rfw >> it) & 1u;
        const int i = rf ? k * T + e : Nc - (k + 1) * T + e;
        const double v = outp[wo[it]];
        if (((rok >> it) & 1u) && i >= 0 && i < Nc) __stcs(wb[it], v);
        wb[it] += rf ? T : -T;
      }
    }
    __syncwarp();
  }
  bad = bad && valid;
  if (valid) outw[(size_t)b * N + n] = psi_e;
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, FLAG_BAD_SIGMA_T);
}

// Net outgoing partial currents: sum over pairs, ascending (the oracle's order), of
// w mu (psi_out - psi_in); a reflected inflow equals the outflow it mirrors.
__global__ void sweep_outflow_kernel(const __grid_constant__ SweepConsts sc, int batch, int order, int refl_left,
                                     int refl_right_first, const double* __restrict__ outw,
                                     double* __restrict__ out_left, double* __restrict__ out_right) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const int H = sc.n_pairs;
  const double* o = outw + (size_t)b * order;
  double l = 0.0, r = 0.0;
  for (int p = 0; p < H; ++p) {
    const double lo = o[H - 1 - p], ro = o[H + p];
    l += sc.wmu[p] * (lo - (refl_left ? lo : 0.0));
    r += sc.wmu[p] * (ro - (refl_right_first ? ro : 0.0));
  }
  if (out_left) out_left[b] = l;
  if (out_right) out_right[b] = r;
}

}  // namespace

namespace snop_impl {

snop_status launch_sweep(Ctx& ctx, const snop_grid& g, int order, int batch, const double* st, const double* em,
                         int bc_left, int bc_right, double* psi, double* out_left, double* out_right) {
  if (batch == 0) return SNOP_OK;
  const SweepConsts sc = make_consts(g, order);
  const int H = order / 2;
  double* outw = static_cast<double*>(ctx.slot(130, (size_t)batch * order * sizeof(double)));
  if (!outw) {
    set_error("sweep: workspace allocation failed");
    return SNOP_CUDA_ERROR;
  }
  static_assert(sizeof(SweepTileSmem<false, 16>) <= 48 * 1024 && sizeof(SweepTileSmem<true, 16>) <= 48 * 1024,
                "sweep tile ring exceeds the default dynamic smem limit");
  static std::once_flag carveout_once[64];  // per device: 7-14 one-warp CTAs per SM need the full carve-out
  if (ctx.device >= 0 && ctx.device < 64)
    std::call_once(carveout_once[ctx.device], [] {
      const auto a = cudaFuncAttributePreferredSharedMemoryCarveout;
      cudaFuncSetAttribute(sweep_kernel<true, 8>, a, cudaSharedmemCarveoutMaxShared);
      cudaFuncSetAttribute(sweep_kernel<false, 8>, a, cudaSharedmemCarveoutMaxShared);
      cudaFuncSetAttribute(sweep_kernel<true, 16>, a, cudaSharedmemCarveoutMaxShared);
      cudaFuncSetAttribute(sweep_kernel<false, 16>, a, cudaSharedmemCarveoutMaxShared);
    });
  const bool pow2 = (H & (H - 1)) == 0;
  const bool aligned = ((reinterpret_cast<uintptr_t>(st) | reinterpret_cast<uintptr_t>(em)) & 15) == 0;
  const bool v16 = pow2 && H >= 2 && g.n_cells % 2 == 0 && aligned;
  auto launch = [&](int n_lo, int n_cnt, const double* infl) {
    const unsigned blocks = (unsigned)(((size_t)batch * n_cnt + 31) / 32);
    // 16-cell tiles (128-byte output rows, half the per-tile overhead) for narrow quadratures, when
    // the launch still fits one wave at their 7 CTAs per SM (a second wave would double the time of
    // these long marches). Measured: C5 (S16) 0.296 -> 0.292 ms, but C2 (S32) 0.421 -> 0.433 ms.
    const bool t16 = order <= 16 && blocks <= 7u * (unsigned)ctx.sm_count && g.n_cells >= 64;
#define SNOP_SWEEP_LAUNCH(V, TT)                                                                              \
  sweep_kernel<V, TT><<<blocks, 32, sizeof(SweepTileSmem<V, TT>), ctx.stream>>>(sc, batch, order, n_lo, n_cnt, st, em, \
                                                                                psi, infl, outw, ctx.d_flags)
    if (v16 && t16) SNOP_SWEEP_LAUNCH(true, 16);
    else if (v16) SNOP_SWEEP_LAUNCH(true, 8);
    else if (t16) SNOP_SWEEP_LAUNCH(false, 16);
    else SNOP_SWEEP_LAUNCH(false, 8);
#undef SNOP_SWEEP_LAUNCH
    ctx.launches++;
  };
  const bool rl = bc_left == 1, rr = bc_right == 1;
  if (!rl && !rr) {
    // Both inflows known. One launch per direction sign: run back to back they beat one launch of
    // mixed-direction work on C2 (0.421 vs 0.461 ms: with both ends of every slab streaming at once
    // the DRAM efficiency drops); for narrow quadratures (half rows of q shorter than a 128-byte DRAM
    // line) the second launch goes to a second stream so its ramp-up overlaps the first one's tail
    // (C5 0.292 -> 0.284 ms; on C2 the concurrent form is the slow one again, 0.462 ms).
    if (order <= 16) {
      if (!ctx.aux) {
        if (cudaStreamCreateWithFlags(&ctx.aux, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx.ev_fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx.ev_join, cudaEventDisableTiming) != cudaSuccess) {
          set_error("sweep: stream / event creation failed");
          return SNOP_CUDA_ERROR;
        }
      }
      cudaEventRecord(ctx.ev_fork, ctx.stream);
      cudaStreamWaitEvent(ctx.aux, ctx.ev_fork, 0);
      launch(0, H, nullptr);
      cudaStream_t main_s = ctx.stream;
      ctx.stream = ctx.aux;
      launch(H, H, nullptr);
      cudaEventRecord(ctx.ev_join, ctx.aux);
      ctx.stream = main_s;
      cudaStreamWaitEvent(ctx.stream, ctx.ev_join, 0);
    } else {
      launch(0, H, nullptr);
      launch(H, H, nullptr);
    }
  } else if (rr && !rl) {
    launch(H, H, nullptr);  // mu > 0 first; its outflow at x = L is the mu < 0 inflow
    launch(0, H, outw);
  } else {
    launch(0, H, nullptr);  // reflective left: mu < 0 first (a reflective right face is lagged:
    launch(H, H, outw);     // zero inflow for a single sweep)
  }
  sweep_outflow_kernel<<<(batch + 127) / 128, 128, 0, ctx.stream>>>(sc, batch, order, rl ? 1 : 0,
                                                                     (rr && !rl) ? 1 : 0, outw, out_left, out_right);
  ctx.launches++;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("sweep_kernel: ") + cudaGetErrorString(e));
    return SNOP_CUDA_ERROR;
  }
  return SNOP_OK;
}

}  // namespace snop_impl
