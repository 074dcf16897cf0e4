// snop_internal.h — host-side internals shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/snop_cuda.h"
#include "snop_device.cuh"

namespace snop_impl {

// Error flags written by kernels into ctx->d_flags (bitwise OR).
enum : int { FLAG_BAD_SIGMA_T = 1, FLAG_DEGENERATE = 2, FLAG_NONFINITE = 4, FLAG_ZERO_PRODUCTION = 8 };

void set_error(const std::string& msg);

struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
};

struct Ctx {
  snop_ctx_options opt{};  // execution options (snop_ctx_set_options); zero = automatic
  int device = 0;
  cudaStream_t stream = nullptr;
  int* d_flags = nullptr;
  int sm_count = 148;
  std::atomic<int64_t> launches{0};
  std::vector<DevBuf> slots;  // scratch buffers for host-memspace staging and workspaces
  uint64_t slot_gen = 0;      // bumped whenever a slot is (re)allocated: cached graphs key on it
  std::vector<double> grf_key;  // (length, n_cells, variance, length scale, jitter) of the cached GRF factor
  void* slot(size_t i, size_t bytes);  // grow-only
  // Device-looped iterations (a CUDA graph whose WHILE conditional node re-runs a captured body
  // until a kernel of the body clears the condition; loops nest): executables cached by their
  // parameters, so a repeated call relaunches without re-capture. Launch accounting: each pass of
  // a loop body adds its kernel count to a device counter; synchronisation folds it into launches.
  struct LoopGraph {
    std::vector<uint64_t> key;
    cudaGraphExec_t exec = nullptr;
  };
  std::vector<LoopGraph> graphs;
  unsigned long long* d_loop_launches = nullptr;  // device counter (kernels launched by loop bodies)
  unsigned long long loop_launches_seen = 0;
  cudaStream_t side = nullptr;                    // capture stream for nested loop bodies
  cudaStream_t aux = nullptr;                     // second stream of the eigen tail split
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  void settle_loops();  // call after the stream has been synchronised
  // Sub-contexts (own stream, flag word and workspace) for host-memspace calls that pipeline
  // H2D / compute / D2H over chunks of the batch; created on first use, owned by this context.
  std::vector<Ctx*> subs;
  Ctx* sub(size_t i);
  ~Ctx();
};

// Builds the per-launch quadrature/mesh constants (mu_p > 0 ascending).
snop_dev::SweepConsts make_consts(const snop_grid& g, int order);

// Kernel launchers (si_kernels.cu). All pointers are device pointers.
snop_status launch_source_iteration(Ctx& ctx, const snop_grid& g, int order, int batch, const double* st,
                                    const double* ss0, const double* ss1, const double* src,
                                    const snop_solver_config& cfg, const double* phi0, double* phi,
                                    double* cur, int32_t* iters, uint8_t* conv, double* leak = nullptr,
                                    double* stage = nullptr, const uint8_t* active = nullptr);
// active != nullptr: instances b with active[b] == 0 are skipped (their outputs are not written).
// stage != nullptr: st/ss0/ss1/src/phi0 and phi/iters/conv/leak may be pinned host memory (read
// and written by the kernel over the bus); stage is a device workspace of batch * (ss1 ? 3 : 2) *
// n_cells doubles. cur must then be device memory or null.

snop_status launch_power_iteration(Ctx& ctx, const snop_grid& g, int order, int batch, int G, const double* st,
                                   const double* ss0, const double* ss1, const double* nsf, const double* chi,
                                   const snop_solver_config& cfg, const double* k0, const double* phi0,
                                   double* k, double* phi, double* phi_old_ws, int32_t* outer, int64_t* inner,
                                   uint8_t* conv);

// Power iteration for slabs beyond the resident kernels (op_capi.cu): device-looped outer
// iterations around the streaming K1.
snop_status launch_power_iteration_big(Ctx& ctx, const snop_grid& g, int order, int batch, int G, const double* st,
                                       const double* ss0, const double* ss1, const double* nsf, const double* chi,
                                       const snop_solver_config& cfg, const double* k0, const double* phi0, double* k,
                                       double* phi, int32_t* outer, int64_t* inner, uint8_t* conv);

// balance_report, batched: residual[b] = |leak_l + leak_r + absorption - production|
// / production with absorption = dx sum (Sigma_t - Sigma_s0,out) phi, production = dx sum S.
snop_status launch_balance(Ctx& ctx, const snop_grid& g, int batch, const double* st, const double* ss_out,
                           const double* src, const double* phi, const double* leak, double* residual);

// Standalone transport sweep (sweep.cu): emission [B][Nc][N], psi_avg [B][N][Nc],
// net outgoing partial currents per instance (nullable).
snop_status launch_sweep(Ctx& ctx, const snop_grid& g, int order, int batch, const double* st, const double* em,
                         int bc_left, int bc_right, double* psi, double* out_left, double* out_right);

snop_status launch_recast(Ctx& ctx, size_t n, const double* S, const double* phi, const double* st,
                          const double* ss, double tstar, double sstar, double* out);

// Largest n_cells one CTA's register-resident sweep holds, and the largest a cluster holds; above
// it the streaming path (si_tiled.cu) runs, up to kMaxCellsAny.
constexpr int kMaxCtaCells = 4096;
constexpr int kMaxCells = 16384;
constexpr int kMaxCellsAny = 1 << 26;

}  // namespace snop_impl

struct snop_ctx : snop_impl::Ctx {};
