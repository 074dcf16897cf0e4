// capi.cu — the extern "C" boundary (include/snop_cuda.h): argument validation, host<->device
// staging for SNOP_MEM_HOST calls, error mapping onto the reference's exception classes
// (proj/core/include/snop/errors.hpp:8-41) and the per-context stream/workspace.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#define SNOP_PHASE_SYM g_phase_cycles_capi
#include "snop_internal.h"

namespace snop_impl {

namespace {
thread_local std::string g_err;
}

void set_error(const std::string& msg) { g_err = msg; }

void* Ctx::slot(size_t i, size_t bytes) {
  if (slots.size() <= i) slots.resize(i + 1);
  DevBuf& b = slots[i];
  if (b.bytes < bytes) {
    ++slot_gen;
    if (b.ptr) cudaFree(b.ptr);
    b.ptr = nullptr;
    b.bytes = 0;
    if (cudaMalloc(&b.ptr, bytes) != cudaSuccess) {
      b.ptr = nullptr;
      return nullptr;
    }
    b.bytes = bytes;
  }
  return b.ptr;
}

Ctx* Ctx::sub(size_t i) {
  while (subs.size() <= i) {
    Ctx* c = new (std::nothrow) Ctx;
    if (!c) return nullptr;
    c->device = device;
    c->sm_count = sm_count;
    c->opt = opt;
    // later sub-contexts get higher stream priority: in the chunked host pipeline the last chunk's
    // data arrives last, so its CTAs must be dispatched ahead of earlier chunks' remaining ones
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    const int prio = std::max(greatest, least - (int)subs.size());
    if (cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio) != cudaSuccess ||
        cudaMalloc(&c->d_flags, sizeof(int)) != cudaSuccess || cudaMemset(c->d_flags, 0, sizeof(int)) != cudaSuccess) {
      delete c;
      return nullptr;
    }
    subs.push_back(c);
  }
  return subs[i];
}

void Ctx::settle_loops() {
  if (!d_loop_launches) return;
  unsigned long long n = 0;
  if (cudaMemcpy(&n, d_loop_launches, sizeof(n), cudaMemcpyDeviceToHost) != cudaSuccess) return;
  launches += (int64_t)(n - loop_launches_seen);
  loop_launches_seen = n;
}

Ctx::~Ctx() {
  if (stream) cudaStreamSynchronize(stream);
  for (auto& g : graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (d_loop_launches) cudaFree(d_loop_launches);
  if (side) cudaStreamDestroy(side);
  if (aux) cudaStreamDestroy(aux);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  for (Ctx* c : subs) delete c;
  for (auto& b : slots)
    if (b.ptr) cudaFree(b.ptr);
  if (d_flags) cudaFree(d_flags);
  if (stream) cudaStreamDestroy(stream);
}

// Gauss-Legendre nodes (same Newton recurrence as SPEC.md:64-72 requires; mirrored symmetric).
static bool gauss_legendre_host(int N, double* mu, double* w) {
  if (N < 2 || N > 128 || N % 2) return false;
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < N / 2; ++i) {
    double x = std::cos(pi * (i + 0.75) / (N + 0.5)), dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= N; ++k) {
        const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = N * (x * p1 - p0) / (x * x - 1.0);
      const double d = p1 / dp;
      x -= d;
      if (std::fabs(d) < 1e-16) break;
    }
    double p0 = 1.0, p1 = x;
    for (int k = 2; k <= N; ++k) {
      const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    dp = N * (x * p1 - p0) / (x * x - 1.0);
    const double wt = 2.0 / ((1.0 - x * x) * dp * dp);
    mu[N - 1 - i] = x;
    mu[i] = -x;
    w[N - 1 - i] = wt;
    w[i] = wt;
  }
  return true;
}

snop_dev::SweepConsts make_consts(const snop_grid& g, int order) {
  snop_dev::SweepConsts sc{};
  double mu[128], w[128];
  gauss_legendre_host(order, mu, w);
  sc.n_cells = g.n_cells;
  sc.n_pairs = order / 2;
  sc.dx = g.length_cm / g.n_cells;
  sc.inv_dx = 1.0 / sc.dx;
  for (int p = 0; p < order / 2; ++p) {
    const double m = mu[order / 2 + p];
    sc.c[p] = 2.0 * m / sc.dx;
    sc.w[p] = w[order / 2 + p];
    sc.wmu[p] = w[order / 2 + p] * m;
    sc.mu3[p] = 3.0 * m;
  }
  return sc;
}

}  // namespace snop_impl

using namespace snop_impl;

namespace {

#define SNOP_TRY(expr)                  \
  do {                                  \
    const snop_status _s = (expr);      \
    if (_s != SNOP_OK) return _s;       \
  } while (0)

snop_status cuda_fail(const char* what, cudaError_t e) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return SNOP_CUDA_ERROR;
}

snop_status invalid(const std::string& m) {
  set_error(m);
  return SNOP_INVALID_ARGUMENT;
}

snop_status check_grid(const snop_grid* g, int order) {
  if (!g) return invalid("grid is NULL");
  if (!(g->length_cm > 0.0) || g->n_cells < 1) return invalid("grid: length and n_cells must be positive");
  if (g->n_cells > kMaxCellsAny) return invalid("grid: n_cells exceeds 2^26");
  if (order < 2 || order > 128 || order % 2) return invalid("quadrature order must be even in [2,128]");
  return SNOP_OK;
}

snop_status check_cfg(const snop_solver_config* c) {
  if (!c) return invalid("config is NULL");
  if (!(c->tolerance > 0.0) || !(c->tolerance_k > 0.0) || !(c->tolerance_phi > 0.0))
    return invalid("config: tolerances must be positive");
  if (c->max_inner < 1 || c->max_outer < 1) return invalid("config: iteration limits must be >= 1");
  if ((c->bc_left != 0 && c->bc_left != 1) || (c->bc_right != 0 && c->bc_right != 1))
    return invalid("config: boundary must be vacuum(0) or reflective(1)");
  if (c->norm != 0 && c->norm != 1) return invalid("config: norm must be rel-Linf(0) or rel-L2(1)");
  return SNOP_OK;
}

// Kernel-raised flags -> status (reads and clears the context's flag word; synchronises).
snop_status drain_flags(Ctx& ctx) {
  int flags = 0;
  cudaError_t e = cudaMemcpyAsync(&flags, ctx.d_flags, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx.stream);
  if (e != cudaSuccess) return cuda_fail("synchronize", e);
  ctx.settle_loops();
  if (flags) cudaMemsetAsync(ctx.d_flags, 0, sizeof(int), ctx.stream);
  if (flags & FLAG_BAD_SIGMA_T) return invalid("nonpositive sigma_t (or initial k) in at least one instance");
  if (flags & FLAG_DEGENERATE) {
    set_error("zero fission integral in at least one instance");
    return SNOP_DEGENERATE_PROBLEM;
  }
  if (flags & FLAG_NONFINITE) {
    set_error("non-finite values produced");
    return SNOP_NUMERICAL_ERROR;
  }
  if (flags & FLAG_ZERO_PRODUCTION) {
    set_error("balance_report: zero production (division guard)");
    return SNOP_NUMERICAL_ERROR;
  }
  return SNOP_OK;
}

// Host staging: copy `bytes` from host `src` into ctx slot `i` (nullptr passes through).
template <class T>
snop_status stage_in(Ctx& ctx, size_t i, const T* src, size_t n, const T** dst) {
  if (!src) {
    *dst = nullptr;
    return SNOP_OK;
  }
  void* d = ctx.slot(i, n * sizeof(T));
  if (!d) return cuda_fail("cudaMalloc", cudaErrorMemoryAllocation);
  const cudaError_t e = cudaMemcpyAsync(d, src, n * sizeof(T), cudaMemcpyHostToDevice, ctx.stream);
  if (e != cudaSuccess) return cuda_fail("H2D copy", e);
  *dst = static_cast<const T*>(d);
  return SNOP_OK;
}

template <class T>
snop_status stage_out_alloc(Ctx& ctx, size_t i, T* host, size_t n, T** dst) {
  if (!host) {
    *dst = nullptr;
    return SNOP_OK;
  }
  void* d = ctx.slot(i, n * sizeof(T));
  if (!d) return cuda_fail("cudaMalloc", cudaErrorMemoryAllocation);
  *dst = static_cast<T*>(d);
  return SNOP_OK;
}

template <class T>
snop_status copy_out(Ctx& ctx, T* host, const T* dev, size_t n) {
  if (!host) return SNOP_OK;
  const cudaError_t e = cudaMemcpyAsync(host, dev, n * sizeof(T), cudaMemcpyDeviceToHost, ctx.stream);
  if (e != cudaSuccess) return cuda_fail("D2H copy", e);
  return SNOP_OK;
}

// Pinned (page-locked, UVA-mapped) host memory can be addressed by kernels directly.
bool pinned(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost && a.devicePointer != nullptr;
}

template <class T>
T* dev_ptr(T* p) {
  if (!p) return nullptr;
  cudaPointerAttributes a{};
  cudaPointerGetAttributes(&a, p);
  return static_cast<T*>(a.devicePointer);
}

}  // namespace

namespace snop_impl {
const char* last_error_cstr() { return g_err.c_str(); }
}  // namespace snop_impl

extern "C" {

int32_t snop_abi_version(void) { return SNOP_ABI_VERSION; }

const char* snop_last_error(void) { return snop_impl::last_error_cstr(); }

snop_status snop_ctx_create(int32_t device, snop_ctx** out) {
  if (!out) return invalid("out is NULL");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return cuda_fail("no CUDA device", e == cudaSuccess ? cudaErrorNoDevice : e);
  if (device < 0 || device >= n) return invalid("device index out of range");
  if ((e = cudaSetDevice(device)) != cudaSuccess) return cuda_fail("cudaSetDevice", e);
  cudaDeviceProp prop;
  if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) return cuda_fail("cudaGetDeviceProperties", e);
  if (prop.major != 10) {
    set_error("libsnop_cuda is built for sm_100a (B200); device is sm_" + std::to_string(prop.major) +
              std::to_string(prop.minor));
    return SNOP_CUDA_ERROR;
  }
  auto* c = new (std::nothrow) snop_ctx;
  if (!c) return cuda_fail("alloc ctx", cudaErrorMemoryAllocation);
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  if ((e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaMalloc(&c->d_flags, sizeof(int))) != cudaSuccess ||
      (e = cudaMemset(c->d_flags, 0, sizeof(int))) != cudaSuccess) {
    delete c;
    return cuda_fail("ctx init", e);
  }
  *out = c;
  return SNOP_OK;
}

snop_status snop_ctx_destroy(snop_ctx* ctx) {
  if (!ctx) return SNOP_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  delete ctx;
  return SNOP_OK;
}

snop_status snop_ctx_synchronize(snop_ctx* ctx) {
  if (!ctx) return invalid("ctx is NULL");
  return drain_flags(*ctx);
}

snop_status snop_ctx_set_options(snop_ctx* ctx, const snop_ctx_options* o) {
  if (!ctx || !o) return invalid("ctx/options is NULL");
  const int cc = o->cell_cluster;
  if (!(cc == -1 || cc == 0 || cc == 1 || cc == 2 || cc == 4 || cc == 8))
    return invalid("options: cell_cluster must be -1, 0, 1, 2, 4 or 8");
  if (o->pair_split < -1 || o->pair_split > 8 || o->pair_split == 1)
    return invalid("options: pair_split must be -1, 0 or 2..8");
  if (o->pi_tail_cap < -1) return invalid("options: pi_tail_cap must be >= -1");
  if (o->host_chunks < 0 || o->host_chunks > 8) return invalid("options: host_chunks must be in [0, 8]");
  if (o->gemm_engine < 0 || o->gemm_engine > 2) return invalid("options: gemm_engine must be 0, 1 or 2");
  if (o->fno_dft < 0 || o->fno_dft > 1 || o->fno_mix < 0 || o->fno_mix > 1)
    return invalid("options: fno_dft / fno_mix must be 0 or 1");
  ctx->opt = *o;
  for (Ctx* s : ctx->subs) s->opt = *o;
  return SNOP_OK;
}

snop_status snop_ctx_get_options(const snop_ctx* ctx, snop_ctx_options* o) {
  if (!ctx || !o) return invalid("ctx/options is NULL");
  *o = ctx->opt;
  return SNOP_OK;
}

int64_t snop_ctx_launch_count(const snop_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

void* snop_ctx_stream(snop_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

snop_status snop_gauss_legendre(int32_t order, double* mu, double* w) {
  if (!mu || !w) return invalid("mu/w NULL");
  if (!gauss_legendre_host(order, mu, w)) return invalid("gauss_legendre: order must be even in [2,128]");
  return SNOP_OK;
}

// Host-memspace source iteration over a large batch: the instances are independent, so the batch
// is cut into NCH chunks, each with its own stream (sub-context): H2D of chunk c+1 overlaps the
// solve of chunk c, chunk kernels run concurrently (later chunks back-fill SMs while earlier ones
// drain their longest instances), and every chunk's D2H starts as soon as its solve ends.
static snop_status si_host_pipelined(Ctx& ctx, const snop_grid& grid, int order, int batch, const double* sigma_t,
                                     const double* sigma_s0, const double* sigma_s1, const double* source,
                                     const snop_solver_config& cfg, const double* initial_phi, double* phi_out,
                                     double* current_out, int32_t* iterations, uint8_t* converged,
                                     double* leakage_out) {
  const int NCH = ctx.opt.host_chunks > 0 ? std::min(ctx.opt.host_chunks, 8) : 4;
  const size_t Nc = grid.n_cells, n = (size_t)batch * Nc;
  auto dbuf = [&](size_t i, size_t count) { return static_cast<double*>(ctx.slot(i, count * sizeof(double))); };
  double* st = dbuf(0, n);
  double* ss = dbuf(1, n);
  double* s1 = sigma_s1 ? dbuf(2, n) : nullptr;
  double* src = dbuf(3, n);
  double* p0 = initial_phi ? dbuf(4, n) : nullptr;
  double* phi = dbuf(5, n);
  double* cur = current_out ? dbuf(6, n) : nullptr;
  int32_t* it = static_cast<int32_t*>(ctx.slot(7, (size_t)batch * sizeof(int32_t)));
  uint8_t* cv = static_cast<uint8_t*>(ctx.slot(8, (size_t)batch));
  double* lk = leakage_out ? dbuf(9, 2 * (size_t)batch) : nullptr;
  if (!st || !ss || (sigma_s1 && !s1) || !src || (initial_phi && !p0) || !phi || (current_out && !cur) || !it ||
      !cv || (leakage_out && !lk))
    return cuda_fail("cudaMalloc", cudaErrorMemoryAllocation);
  cudaEvent_t ready;
  cudaError_t e = cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
  if (e != cudaSuccess) return cuda_fail("cudaEventCreate", e);
  cudaEventRecord(ready, ctx.stream);  // earlier work on the context's stream may still use the slots
  Ctx* subs[8];
  for (int c = 0; c < NCH; ++c) {
    subs[c] = ctx.sub(c);
    if (!subs[c]) {
      cudaEventDestroy(ready);
      return cuda_fail("sub-context", cudaErrorMemoryAllocation);
    }
    cudaStreamWaitEvent(subs[c]->stream, ready, 0);
  }
  cudaEventDestroy(ready);
  auto h2d = [&](double* d, const double* h, size_t b0, size_t nb, cudaStream_t s) {
    return h ? cudaMemcpyAsync(d + b0 * Nc, h + b0 * Nc, nb * Nc * sizeof(double), cudaMemcpyHostToDevice, s)
             : cudaSuccess;
  };
  snop_status st_out = SNOP_OK;
  size_t bounds[9];
  for (int c = 0; c <= NCH; ++c) bounds[c] = (size_t)batch * c / NCH;
  for (int c = 0; c < NCH && st_out == SNOP_OK; ++c) {
    const size_t b0 = bounds[c], nb = bounds[c + 1] - b0;
    Ctx& sc = *subs[c];
    cudaError_t ce = h2d(st, sigma_t, b0, nb, sc.stream);
    if (ce == cudaSuccess) ce = h2d(ss, sigma_s0, b0, nb, sc.stream);
    if (ce == cudaSuccess) ce = h2d(s1, sigma_s1, b0, nb, sc.stream);
    if (ce == cudaSuccess) ce = h2d(src, source, b0, nb, sc.stream);
    if (ce == cudaSuccess) ce = h2d(p0, initial_phi, b0, nb, sc.stream);
    if (ce != cudaSuccess) {
      st_out = cuda_fail("H2D copy", ce);
      break;
    }
    const size_t o = b0 * Nc;
    st_out = launch_source_iteration(sc, grid, order, (int)nb, st + o, ss + o, s1 ? s1 + o : nullptr, src + o, cfg,
                                     p0 ? p0 + o : nullptr, phi + o, cur ? cur + o : nullptr, it + b0, cv + b0,
                                     lk ? lk + 2 * b0 : nullptr);
  }
  for (int c = 0; c < NCH && st_out == SNOP_OK; ++c) {
    const size_t b0 = bounds[c], nb = bounds[c + 1] - b0;
    const cudaStream_t s = subs[c]->stream;
    cudaError_t ce = cudaMemcpyAsync(phi_out + b0 * Nc, phi + b0 * Nc, nb * Nc * sizeof(double),
                                     cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess && current_out)
      ce = cudaMemcpyAsync(current_out + b0 * Nc, cur + b0 * Nc, nb * Nc * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(iterations + b0, it + b0, nb * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(converged + b0, cv + b0, nb, cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess && leakage_out)
      ce = cudaMemcpyAsync(leakage_out + 2 * b0, lk + 2 * b0, 2 * nb * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (ce != cudaSuccess) st_out = cuda_fail("D2H copy", ce);
  }
  snop_status drained = SNOP_OK;
  for (int c = 0; c < NCH; ++c) {  // always synchronise every chunk stream, even after an error
    const snop_status d = drain_flags(*subs[c]);
    if (drained == SNOP_OK) drained = d;
    ctx.launches += subs[c]->launches.exchange(0);
  }
  return st_out != SNOP_OK ? st_out : drained;
}

static snop_status si_entry(snop_ctx* ctx, int32_t memspace, const snop_grid* grid, int32_t order, int32_t batch,
                            const double* sigma_t, const double* sigma_s0, const double* sigma_s1,
                            const double* source, const snop_solver_config* cfg, const double* initial_phi,
                            double* phi_out, double* current_out, int32_t* iterations, uint8_t* converged,
                            double* leakage_out) {
  if (!ctx) return invalid("ctx is NULL");
  SNOP_TRY(check_grid(grid, order));
  SNOP_TRY(check_cfg(cfg));
  if (batch < 0) return invalid("batch must be >= 0");
  if (batch == 0) return SNOP_OK;
  if (!sigma_t || !sigma_s0 || !source || !phi_out || !iterations || !converged)
    return invalid("required array pointer is NULL");
  cudaSetDevice(ctx->device);
  const size_t n = (size_t)batch * grid->n_cells;
  if (memspace == SNOP_MEM_DEVICE) {
    return launch_source_iteration(*ctx, *grid, order, batch, sigma_t, sigma_s0, sigma_s1, source, *cfg,
                                   initial_phi, phi_out, current_out, iterations, converged, leakage_out);
  }
  if (memspace != SNOP_MEM_HOST) return invalid("memspace must be HOST(0) or DEVICE(1)");
  const bool one_cta = grid->n_cells <= kMaxCtaCells && ctx->opt.cell_cluster <= 1;
  if (one_cta && !current_out && pinned(sigma_t) && pinned(sigma_s0) && pinned(source) && (!sigma_s1 || pinned(sigma_s1)) &&
      (!initial_phi || pinned(initial_phi)) && pinned(phi_out) && pinned(iterations) && pinned(converged) &&
      (!leakage_out || pinned(leakage_out))) {
    // zero-copy: the kernel reads its instance's inputs over the bus and writes its results back
    // as it finishes, so transfers overlap the solves of other instances (no staging copies)
    double* stage = static_cast<double*>(ctx->slot(24, n * (sigma_s1 ? 3 : 2) * sizeof(double)));
    if (!stage) return cuda_fail("cudaMalloc", cudaErrorMemoryAllocation);
    SNOP_TRY(launch_source_iteration(*ctx, *grid, order, batch, dev_ptr(sigma_t), dev_ptr(sigma_s0),
                                     dev_ptr(sigma_s1), dev_ptr(source), *cfg, dev_ptr(initial_phi), dev_ptr(phi_out),
                                     nullptr, dev_ptr(iterations), dev_ptr(converged), dev_ptr(leakage_out), stage));
    return drain_flags(*ctx);
  }
  if (batch >= 4 * ctx->sm_count)
    return si_host_pipelined(*ctx, *grid, order, batch, sigma_t, sigma_s0, sigma_s1, source, *cfg, initial_phi,
                             phi_out, current_out, iterations, converged, leakage_out);
  const double *st, *ss, *s1, *src, *p0;
  double *phi, *cur;
  int32_t* it;
  uint8_t* cv;
  SNOP_TRY(stage_in(*ctx, 0, sigma_t, n, &st));
  SNOP_TRY(stage_in(*ctx, 1, sigma_s0, n, &ss));
  SNOP_TRY(stage_in(*ctx, 2, sigma_s1, n, &s1));
  SNOP_TRY(stage_in(*ctx, 3, source, n, &src));
  SNOP_TRY(stage_in(*ctx, 4, initial_phi, n, &p0));
  SNOP_TRY(stage_out_alloc(*ctx, 5, phi_out, n, &phi));
  SNOP_TRY(stage_out_alloc(*ctx, 6, current_out, n, &cur));
  SNOP_TRY(stage_out_alloc(*ctx, 7, iterations, (size_t)batch, &it));
  SNOP_TRY(stage_out_alloc(*ctx, 8, converged, (size_t)batch, &cv));
  double* lk;
  SNOP_TRY(stage_out_alloc(*ctx, 9, leakage_out, 2 * (size_t)batch, &lk));
  SNOP_TRY(launch_source_iteration(*ctx, *grid, order, batch, st, ss, s1, src, *cfg, p0, phi, cur, it, cv, lk));
  SNOP_TRY(copy_out(*ctx, phi_out, phi, n));
  SNOP_TRY(copy_out(*ctx, current_out, cur, n));
  SNOP_TRY(copy_out(*ctx, iterations, it, (size_t)batch));
  SNOP_TRY(copy_out(*ctx, converged, cv, (size_t)batch));
  SNOP_TRY(copy_out(*ctx, leakage_out, lk, 2 * (size_t)batch));
  return drain_flags(*ctx);
}

snop_status snop_source_iteration_batched(snop_ctx* ctx, int32_t memspace, const snop_grid* grid, int32_t order,
                                          int32_t batch, const double* sigma_t, const double* sigma_s0,
                                          const double* sigma_s1, const double* source,
                                          const snop_solver_config* cfg, const double* initial_phi,
                                          double* phi_out, double* current_out, int32_t* iterations,
                                          uint8_t* converged) {
  return si_entry(ctx, memspace, grid, order, batch, sigma_t, sigma_s0, sigma_s1, source, cfg, initial_phi, phi_out,
                  current_out, iterations, converged, nullptr);
}

snop_status snop_source_iteration_leakage_batched(snop_ctx* ctx, int32_t memspace, const snop_grid* grid,
                                                  int32_t order, int32_t batch, const double* sigma_t,
                                                  const double* sigma_s0, const double* sigma_s1,
                                                  const double* source, const snop_solver_config* cfg,
                                                  const double* initial_phi, double* phi_out, double* current_out,
                                                  int32_t* iterations, uint8_t* converged, double* leakage_out) {
  if (!leakage_out) return invalid("leakage_out is NULL");
  return si_entry(ctx, memspace, grid, order, batch, sigma_t, sigma_s0, sigma_s1, source, cfg, initial_phi, phi_out,
                  current_out, iterations, converged, leakage_out);
}

snop_status snop_balance_report(snop_ctx* ctx, int32_t memspace, const snop_grid* grid, int32_t batch,
                                const double* sigma_t, const double* sigma_s0_out, const double* source,
                                const double* phi, const double* leakage, double* residual_out) {
  if (!ctx || !grid) return invalid("ctx/grid is NULL");
  if (!(grid->length_cm > 0.0) || grid->n_cells < 1 || batch < 0) return invalid("bad grid / batch");
  if (batch == 0) return SNOP_OK;
  if (!sigma_t || !sigma_s0_out || !source || !phi || !leakage || !residual_out) return invalid("NULL array");
  cudaSetDevice(ctx->device);
  const size_t n = (size_t)batch * grid->n_cells;
  if (memspace == SNOP_MEM_DEVICE)
    return launch_balance(*ctx, *grid, batch, sigma_t, sigma_s0_out, source, phi, leakage, residual_out);
  if (memspace != SNOP_MEM_HOST) return invalid("memspace must be HOST(0) or DEVICE(1)");
  const double *st, *ss, *src, *p, *lk;
  double* res;
  SNOP_TRY(stage_in(*ctx, 0, sigma_t, n, &st));
  SNOP_TRY(stage_in(*ctx, 1, sigma_s0_out, n, &ss));
  SNOP_TRY(stage_in(*ctx, 3, source, n, &src));
  SNOP_TRY(stage_in(*ctx, 4, phi, n, &p));
  SNOP_TRY(stage_in(*ctx, 10, leakage, 2 * (size_t)batch, &lk));
  SNOP_TRY(stage_out_alloc(*ctx, 11, residual_out, (size_t)batch, &res));
  SNOP_TRY(launch_balance(*ctx, *grid, batch, st, ss, src, p, lk, res));
  SNOP_TRY(copy_out(*ctx, residual_out, res, (size_t)batch));
  return drain_flags(*ctx);
}

snop_status snop_power_iteration_batched(snop_ctx* ctx, int32_t memspace, const snop_grid* grid, int32_t order,
                                         int32_t batch, int32_t n_groups, const double* sigma_t,
                                         const double* sigma_s0, const double* sigma_s1, const double* nu_sigma_f,
                                         const double* chi, const snop_solver_config* cfg, const double* initial_k,
                                         const double* initial_phi, double* k_out, double* phi_out,
                                         int32_t* outer_iterations, int64_t* inner_iterations,
                                         uint8_t* converged) {
  if (!ctx) return invalid("ctx is NULL");
  SNOP_TRY(check_grid(grid, order));
  SNOP_TRY(check_cfg(cfg));
  if (batch < 0) return invalid("batch must be >= 0");
  if (n_groups < 1 || n_groups > 64) return invalid("n_groups must be in [1,64]");
  if (batch == 0) return SNOP_OK;
  if (!sigma_t || !sigma_s0 || !nu_sigma_f || !chi || !k_out || !phi_out || !outer_iterations ||
      !inner_iterations || !converged)
    return invalid("required array pointer is NULL");
  cudaSetDevice(ctx->device);
  const size_t G = n_groups, Nc = grid->n_cells, B = batch;
  const size_t n = B * G * Nc;
  double* old = static_cast<double*>(ctx->slot(20, n * sizeof(double)));
  if (!old) return cuda_fail("cudaMalloc", cudaErrorMemoryAllocation);
  if (memspace == SNOP_MEM_DEVICE) {
    return launch_power_iteration(*ctx, *grid, order, batch, n_groups, sigma_t, sigma_s0, sigma_s1, nu_sigma_f,
                                  chi, *cfg, initial_k, initial_phi, k_out, phi_out, old, outer_iterations,
                                  inner_iterations, converged);
  }
  if (memspace != SNOP_MEM_HOST) return invalid("memspace must be HOST(0) or DEVICE(1)");
  const double *st, *ss, *s1, *nsf, *ch, *k0, *p0;
  double *k, *phi;
  int32_t* outer;
  int64_t* inner;
  uint8_t* cv;
  SNOP_TRY(stage_in(*ctx, 0, sigma_t, n, &st));
  SNOP_TRY(stage_in(*ctx, 1, sigma_s0, n * G, &ss));
  SNOP_TRY(stage_in(*ctx, 2, sigma_s1, n, &s1));
  SNOP_TRY(stage_in(*ctx, 3, nu_sigma_f, n, &nsf));
  SNOP_TRY(stage_in(*ctx, 4, chi, B * G, &ch));
  SNOP_TRY(stage_in(*ctx, 5, initial_k, B, &k0));
  SNOP_TRY(stage_in(*ctx, 6, initial_phi, n, &p0));
  SNOP_TRY(stage_out_alloc(*ctx, 7, k_out, B, &k));
  SNOP_TRY(stage_out_alloc(*ctx, 8, phi_out, n, &phi));
  SNOP_TRY(stage_out_alloc(*ctx, 9, outer_iterations, B, &outer));
  SNOP_TRY(stage_out_alloc(*ctx, 10, inner_iterations, B, &inner));
  SNOP_TRY(stage_out_alloc(*ctx, 11, converged, B, &cv));
  SNOP_TRY(launch_power_iteration(*ctx, *grid, order, batch, n_groups, st, ss, s1, nsf, ch, *cfg, k0, p0, k, phi,
                                  old, outer, inner, cv));
  SNOP_TRY(copy_out(*ctx, k_out, k, B));
  SNOP_TRY(copy_out(*ctx, phi_out, phi, n));
  SNOP_TRY(copy_out(*ctx, outer_iterations, outer, B));
  SNOP_TRY(copy_out(*ctx, inner_iterations, inner, B));
  SNOP_TRY(copy_out(*ctx, converged, cv, B));
  return drain_flags(*ctx);
}

snop_status snop_sweep_batched(snop_ctx* ctx, int32_t memspace, const snop_grid* grid, int32_t order, int32_t batch,
                               const double* sigma_t, const double* emission, int32_t bc_left, int32_t bc_right,
                               double* psi_avg_out, double* outflow_left, double* outflow_right) {
  if (!ctx) return invalid("ctx is NULL");
  SNOP_TRY(check_grid(grid, order));
  if (batch < 0) return invalid("batch must be >= 0");
  if ((bc_left != 0 && bc_left != 1) || (bc_right != 0 && bc_right != 1))
    return invalid("boundary must be VACUUM(0) or REFLECTIVE(1)");
  if (batch == 0) return SNOP_OK;
  if (!sigma_t || !emission || !psi_avg_out) return invalid("required array pointer is NULL");
  cudaSetDevice(ctx->device);
  const size_t B = batch, Nc = grid->n_cells, N = order;
  if (memspace == SNOP_MEM_DEVICE)
    return launch_sweep(*ctx, *grid, order, batch, sigma_t, emission, bc_left, bc_right, psi_avg_out, outflow_left,
                        outflow_right);
  if (memspace != SNOP_MEM_HOST) return invalid("memspace must be HOST(0) or DEVICE(1)");
  const double *st, *em;
  double *psi, *ol, *orr;
  SNOP_TRY(stage_in(*ctx, 0, sigma_t, B * Nc, &st));
  SNOP_TRY(stage_in(*ctx, 1, emission, B * Nc * N, &em));
  SNOP_TRY(stage_out_alloc(*ctx, 2, psi_avg_out, B * Nc * N, &psi));
  SNOP_TRY(stage_out_alloc(*ctx, 3, outflow_left, B, &ol));
  SNOP_TRY(stage_out_alloc(*ctx, 4, outflow_right, B, &orr));
  SNOP_TRY(launch_sweep(*ctx, *grid, order, batch, st, em, bc_left, bc_right, psi, ol, orr));
  SNOP_TRY(copy_out(*ctx, psi_avg_out, psi, B * Nc * N));
  SNOP_TRY(copy_out(*ctx, outflow_left, ol, B));
  SNOP_TRY(copy_out(*ctx, outflow_right, orr, B));
  return drain_flags(*ctx);
}

snop_status snop_recast_source(snop_ctx* ctx, int32_t memspace, int32_t batch, int32_t n_cells, const double* source,
                               const double* phi, const double* sigma_t, const double* sigma_s0,
                               double sigma_t_star, double sigma_s0_star, double* out) {
  if (!ctx) return invalid("ctx is NULL");
  if (batch < 0 || n_cells < 1) return invalid("batch must be >= 0 and n_cells >= 1");
  if (batch == 0) return SNOP_OK;
  if (!source || !phi || !sigma_t || !sigma_s0 || !out) return invalid("required array pointer is NULL");
  cudaSetDevice(ctx->device);
  const size_t n = (size_t)batch * n_cells;
  if (memspace == SNOP_MEM_DEVICE)
    return launch_recast(*ctx, n, source, phi, sigma_t, sigma_s0, sigma_t_star, sigma_s0_star, out);
  if (memspace != SNOP_MEM_HOST) return invalid("memspace must be HOST(0) or DEVICE(1)");
  const double *S, *p, *st, *ss;
  double* o;
  SNOP_TRY(stage_in(*ctx, 0, source, n, &S));
  SNOP_TRY(stage_in(*ctx, 1, phi, n, &p));
  SNOP_TRY(stage_in(*ctx, 2, sigma_t, n, &st));
  SNOP_TRY(stage_in(*ctx, 3, sigma_s0, n, &ss));
  SNOP_TRY(stage_out_alloc(*ctx, 4, out, n, &o));
  SNOP_TRY(launch_recast(*ctx, n, S, p, st, ss, sigma_t_star, sigma_s0_star, o));
  SNOP_TRY(copy_out(*ctx, out, o, n));
  return drain_flags(*ctx);
}

}  // extern "C"
