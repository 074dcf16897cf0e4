// sweep.cu — the standalone transport sweep as a streaming sm_100a kernel.
//
// One diamond-difference sweep of all N directions of B instances with a PER-DIRECTION emission:
//   psi_avg = (q + c psi_in) / (Sigma_t + c),  psi_out = 2 psi_avg - psi_in,  c = 2|mu|/dx.
// Unlike the fused solvers (K1/K2), which never materialise psi, this operator reads the
// emission q(x_i, mu_n) and writes the cell-average angular flux for every cell and direction:
// 16 B of HBM traffic per cell.angle update (+ Sigma_t, 8 B per cell, served once from DRAM and
// then from L1/L2), so it is HBM-bound and is measured against the copy roofline.
//
// Mapping. Thread = one +/-mu pair of one instance; it marches the mu > 0 direction left to
// right and the mu < 0 direction right to left (two independent recurrences per thread; a
// reflective face makes one wait for the other's outflow, SURVEY §9 #2 ordering). B*N/2 chains
// are the parallelism (65536 for BASELINE C2/C5); CTA = one warp, so the grid balances over the
// 148 SMs. The recurrence is serial in the cell index but needs one dependent 3-instruction
// chain per cell; everything else (reciprocal, loads, stores) is off the chain.
//   * loads: emission [B][Nc][N] makes the N/2 same-sign directions of a cell contiguous, so the
//     lanes of an instance read one segment per cell. Each thread copies its own q and Sigma_t
//     values with 8-byte cp.async into a private slot of an S-stage shared-memory ring (tiles of
//     T cells), S-1 tiles ahead: bytes in flight without holding registers.
//   * stores: psi_avg [B][N][Nc] is direction-major, so a thread's T results of a tile are
//     contiguous but the lanes are Nc apart: the warp transposes each tile through shared memory
//     and writes whole rows (T contiguous cells per row, 32/T rows per instruction).
//   * partial currents: w mu (psi_out - psi_in) at both faces per pair into a workspace; a second
//     tiny kernel sums the pairs of an instance in ascending order (deterministic, the oracle's
//     order).
#include <string>

#define SNOP_PHASE_SYM g_phase_cycles_sweep
#include "snop_internal.h"

using namespace snop_impl;
using namespace snop_dev;

namespace {

constexpr int kT = 8;  // cells per tile
constexpr int kS = 3;  // ring stages (kS - 1 tiles in flight; 7 one-warp CTAs per SM must fit: 28.6 KB each)

constexpr int kG = 16;  // most instances a warp can span on the vector path (H >= 2)

// V16 = false (any order / cell count / alignment): every thread copies its own q and Sigma_t
// values with 8-byte cp.async. V16 = true (N/2 a power of two, even cell count, 16-byte aligned
// arrays): even lanes copy the q of a lane pair with 16-byte cp.async.cg (8-byte cp.async.ca
// serialises its shared-memory writes: 17 wavefronts per request in ncu, the LSU data pipe at 87%),
// and Sigma_t is copied once per instance of the warp instead of once per lane.
template <bool V16>
struct SweepTileSmem {
  double q[kS][2][kT][32];   // emission of the thread's two directions, [stage][fwd/bwd][cell][lane]
  double st[kS][2][V16 ? kG : kT][V16 ? kT : 32];  // Sigma_t: [..][instance][cell] or [..][cell][lane]
  double out[2][32][kT + 1]; // psi_avg of the current tile, [fwd/bwd][lane][cell] (+1: conflict-free)
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 8 : 0;  // src-size 0: zero fill (cells beyond the slab)
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// One march over the slab for the enabled directions of this thread's pair.
//   F: mu > 0, cells ascending, inflow in_f at x = 0;  Bk: mu < 0, cells descending, inflow in_b.
template <bool F, bool Bk, bool V16>
__device__ __forceinline__ void march(SweepTileSmem<V16>& sm, int Nc, int N, int lane, bool valid, double c,
                                      int grp, int grank, int gsize,     // V16: instance slot / rank / lanes in the warp
                                      const double* __restrict__ st_b,   // Sigma_t of the instance
                                      const double* __restrict__ em_f,   // &emission[b][0][n+]
                                      const double* __restrict__ em_b,   // &emission[b][0][n-]
                                      double* __restrict__ psi, size_t row_f, size_t row_b,
                                      double in_f, double in_b, double& out_f, double& out_b, bool& bad) {
  const int ntiles = (Nc + kT - 1) / kT;
  auto issue = [&](int k) {
    if (k < ntiles) {
      const int slot = k % kS;
      if constexpr (V16) {
        // q: the even lane of a lane pair copies both lanes' values (adjacent directions); the
        // mu < 0 directions descend with the lane, so their pair lands swapped (read at lane ^ 1)
        if ((lane & 1) == 0) {
#pragma unroll
          for (int j = 0; j < kT; ++j) {
            if constexpr (F) {
              const int i = k * kT + j;
              const bool ok = valid && i < Nc;
              cp_async16(&sm.q[slot][0][j][lane], em_f + (size_t)(ok ? i : 0) * N, ok);
            }
            if constexpr (Bk) {
              const int i = Nc - 1 - k * kT - j;
              const bool ok = valid && i >= 0;
              cp_async16(&sm.q[slot][1][j][lane], em_b - 1 + (size_t)(ok ? i : 0) * N, ok);
            }
          }
        }
        // Sigma_t: the lanes of an instance copy its tile once, two cells per copy, ascending
        for (int m2 = grank; m2 < kT / 2; m2 += gsize) {
          if constexpr (F) {
            const int i = k * kT + 2 * m2;
            const bool ok = valid && i < Nc;  // (even Nc: i + 1 < Nc as well)
            cp_async16(&sm.st[slot][0][grp][2 * m2], st_b + (ok ? i : 0), ok);
          }
          if constexpr (Bk) {
            const int i = Nc - (k + 1) * kT + 2 * m2;
            const bool ok = valid && i >= 0;
            cp_async16(&sm.st[slot][1][grp][2 * m2], st_b + (ok ? i : 0), ok);
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < kT; ++j) {
          if constexpr (F) {
            const int i = k * kT + j;
            const bool ok = valid && i < Nc;
            cp_async8(&sm.q[slot][0][j][lane], em_f + (size_t)(ok ? i : 0) * N, ok);
            cp_async8(&sm.st[slot][0][j][lane], st_b + (ok ? i : 0), ok);
          }
          if constexpr (Bk) {
            const int i = Nc - 1 - k * kT - j;
            const bool ok = valid && i >= 0;
            cp_async8(&sm.q[slot][1][j][lane], em_b + (size_t)(ok ? i : 0) * N, ok);
            cp_async8(&sm.st[slot][1][j][lane], st_b + (ok ? i : 0), ok);
          }
        }
      }
    }
    cp_async_commit();  // (an empty group past the last tile keeps the wait count uniform)
  };
#pragma unroll
  for (int k = 0; k < kS - 1; ++k) issue(k);
  double pf = in_f, pb = in_b;
  for (int k = 0; k < ntiles; ++k) {
    issue(k + kS - 1);
    cp_async_wait<kS - 1>();  // this thread's copies of tile k have landed
    if constexpr (V16) __syncwarp();  // ... and the other lanes' (pair partner, Sigma_t tile)
    const int slot = k % kS;
#pragma unroll
    for (int j = 0; j < kT; ++j) {
      if constexpr (F) {
        const int i = k * kT + j;
        if (i < Nc) {
          const double s = V16 ? sm.st[slot][0][grp][j] : sm.st[slot][0][j][lane], q = sm.q[slot][0][j][lane];
          bad |= valid && !(s > 0.0);
          const double avg = fma(c, pf, q) * rcp_fast(s + c);
          pf = fma(2.0, avg, -pf);
          sm.out[0][lane][j] = avg;
        }
      }
      if constexpr (Bk) {
        const int i = Nc - 1 - k * kT - j;
        if (i >= 0) {
          const double s = V16 ? sm.st[slot][1][grp][kT - 1 - j] : sm.st[slot][1][j][lane];
          const double q = sm.q[slot][1][j][V16 ? lane ^ 1 : lane];
          bad |= valid && !(s > 0.0);
          const double avg = fma(c, pb, q) * rcp_fast(s + c);
          pb = fma(2.0, avg, -pb);
          sm.out[1][lane][j] = avg;
        }
      }
    }
    __syncwarp();
    // write-out: 32/kT rows of kT contiguous cells per instruction
    constexpr int RPI = 32 / kT;
    const int e = lane % kT, rsub = lane / kT;
#pragma unroll
    for (int it = 0; it < kT; ++it) {
      const int row = it * RPI + rsub;
      if constexpr (F) {
        const size_t base = __shfl_sync(0xffffffffu, (unsigned long long)row_f, row);
        const int i = k * kT + e;
        const double v = sm.out[0][row][e];
        if (base != ~(size_t)0 && i < Nc) __stcs(psi + base + i, v);
      }
      if constexpr (Bk) {
        const size_t base = __shfl_sync(0xffffffffu, (unsigned long long)row_b, row);
        const int i = Nc - (k + 1) * kT + e;  // ascending cells of the descending tile
        const double v = sm.out[1][row][kT - 1 - e];
        if (base != ~(size_t)0 && i >= 0) __stcs(psi + base + i, v);
      }
    }
    __syncwarp();
  }
  out_f = pf;
  out_b = pb;
}

template <bool V16>
__global__ void __launch_bounds__(32)
sweep_kernel(const __grid_constant__ SweepConsts sc, int batch, int order, int bc_left, int bc_right,
             const double* __restrict__ st_g, const double* __restrict__ em_g, double* __restrict__ psi_g,
             double* __restrict__ part /* [B][H][2] */, int* __restrict__ flags) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<SweepTileSmem<V16>*>(smem_raw);
  const int lane = threadIdx.x, Nc = sc.n_cells, H = sc.n_pairs, N = order;
  const long long total = (long long)batch * H;
  const long long gt = (long long)blockIdx.x * 32 + lane;
  const bool valid = gt < total;
  const long long g = valid ? gt : total - 1;
  const int b = (int)(g / H), p = (int)(g - (long long)b * H);
  const double c = sc.c[p];
  const double* st_b = st_g + (size_t)b * Nc;
  const double* em_f = em_g + (size_t)b * Nc * N + (H + p);
  const double* em_b = em_g + (size_t)b * Nc * N + (H - 1 - p);
  const size_t row_f = valid ? ((size_t)b * N + (H + p)) * Nc : ~(size_t)0;
  const size_t row_b = valid ? ((size_t)b * N + (H - 1 - p)) * Nc : ~(size_t)0;
  // vector path: the lanes of this warp that belong to the same instance (H a power of two)
  const int hw = H < 32 ? H : 32;
  const int grp = V16 ? lane / hw : 0, grank = lane % hw, gsize = hw;
  const bool rl = bc_left == 1, rr = bc_right == 1;
  bool bad = false;
  double in_l = 0.0, in_r = 0.0, out_l = 0.0, out_r = 0.0, d0, d1;
  if (!rl && !rr) {  // both inflows known: the two directions march together
    march<true, true, V16>(sm, Nc, N, lane, valid, c, grp, grank, gsize, st_b, em_f, em_b, psi_g, row_f, row_b, 0.0, 0.0, out_r, out_l, bad);
  } else if (rr && !rl) {  // mu > 0 first; its outflow at x = L is the mu < 0 inflow
    march<true, false, V16>(sm, Nc, N, lane, valid, c, grp, grank, gsize, st_b, em_f, em_b, psi_g, row_f, row_b, 0.0, 0.0, out_r, d0, bad);
    in_r = out_r;
    march<false, true, V16>(sm, Nc, N, lane, valid, c, grp, grank, gsize, st_b, em_f, em_b, psi_g, row_f, row_b, 0.0, in_r, d1, out_l, bad);
  } else {  // reflective left (a reflective right face is lagged: zero inflow for a single sweep)
    march<false, true, V16>(sm, Nc, N, lane, valid, c, grp, grank, gsize, st_b, em_f, em_b, psi_g, row_f, row_b, 0.0, 0.0, d0, out_l, bad);
    in_l = out_l;
    march<true, false, V16>(sm, Nc, N, lane, valid, c, grp, grank, gsize, st_b, em_f, em_b, psi_g, row_f, row_b, in_l, 0.0, out_r, d1, bad);
  }
  (void)d0;
  (void)d1;
  if (valid) {
    const double wm = sc.wmu[p];
    part[2 * gt] = wm * (out_l - in_l);
    part[2 * gt + 1] = wm * (out_r - in_r);
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, FLAG_BAD_SIGMA_T);
}

__global__ void sweep_outflow_kernel(int batch, int H, const double* __restrict__ part,
                                     double* __restrict__ out_left, double* __restrict__ out_right) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  double l = 0.0, r = 0.0;
  for (int p = 0; p < H; ++p) {  // ascending pair order (the oracle's)
    l += part[2 * ((size_t)b * H + p)];
    r += part[2 * ((size_t)b * H + p) + 1];
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
  const size_t chains = (size_t)batch * H;
  double* part = static_cast<double*>(ctx.slot(130, chains * 2 * sizeof(double)));
  if (!part) {
    set_error("sweep: workspace allocation failed");
    return SNOP_CUDA_ERROR;
  }
  static_assert(sizeof(SweepTileSmem<false>) <= 48 * 1024 && sizeof(SweepTileSmem<true>) <= 48 * 1024,
                "sweep tile ring exceeds the default dynamic smem limit");
  static bool carveout_set[64] = {};
  if (ctx.device >= 0 && ctx.device < 64 && !carveout_set[ctx.device]) {  // 7 one-warp CTAs per SM
    cudaFuncSetAttribute(sweep_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(sweep_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    carveout_set[ctx.device] = true;
  }
  const unsigned blocks = (unsigned)((chains + 31) / 32);
  const bool pow2 = (H & (H - 1)) == 0;
  const bool aligned = ((reinterpret_cast<uintptr_t>(st) | reinterpret_cast<uintptr_t>(em)) & 15) == 0;
  if (pow2 && H >= 2 && g.n_cells % 2 == 0 && aligned)
    sweep_kernel<true><<<blocks, 32, sizeof(SweepTileSmem<true>), ctx.stream>>>(sc, batch, order, bc_left, bc_right, st,
                                                                                em, psi, part, ctx.d_flags);
  else
    sweep_kernel<false><<<blocks, 32, sizeof(SweepTileSmem<false>), ctx.stream>>>(sc, batch, order, bc_left, bc_right,
                                                                                  st, em, psi, part, ctx.d_flags);
  ctx.launches++;
  sweep_outflow_kernel<<<(batch + 127) / 128, 128, 0, ctx.stream>>>(batch, H, part, out_left, out_right);
  ctx.launches++;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("sweep_kernel: ") + cudaGetErrorString(e));
    return SNOP_CUDA_ERROR;
  }
  return SNOP_OK;
}

}  // namespace snop_impl
