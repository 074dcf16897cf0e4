// grf.cu — Gaussian-random-field sources and training-dataset generation on the device
// (paper Appendix A1).
//
//   sample s  : z = N(0,1) stream of snop::Rng(seed + s) (rng.hpp:17-49: std::mt19937_64, Box-Muller
//               with cached spare, u1 in (0,1]), field = mean + L z, L L^T = C + jitter I
//   normalize : S = raw / (dx sum raw)                                     (Eq. 13)
//   dataset   : normalize(sample(s)) -> source iteration at p* (zero guess, vacuum)
//
// Device mapping: one warp per sample regenerates that sample's mt19937_64 stream in shared memory
// (seeding recurrence on lane 0, the state twist in three dependency-free slices across the warp,
// tempering + Box-Muller on pairs in parallel — a normal pair consumes two consecutive outputs and a
// 312-word block holds whole pairs), so the u64 stream is bit-identical to the host engine. The
// correlation z -> L z is a lower-triangular fp64 GEMM (smem-tiled DFMA; triangular tiles skipped).
// The Cholesky factor is computed once per (grid, spec) on the host, Cholesky-Banachiewicz row by
// row with jitter escalation x10 up to 1e-6, and cached on the context. The
// jitter is relative to the variance (C + jitter var I): SPEC.md:245's degenerate-variance example
// requires it.
#include <cmath>
#include <string>
#include <vector>

#define SNOP_PHASE_SYM g_phase_cycles_grf
#include "snop_internal.h"

namespace snop_impl {

namespace {

#define SNOP_TRY(expr)             \
  do {                             \
    const snop_status _s = (expr); \
    if (_s != SNOP_OK) return _s;  \
  } while (0)

snop_status fail(snop_status s, const std::string& m) {
  set_error(m);
  return s;
}
snop_status cuda_ok(const char* what, cudaError_t e) {
  if (e == cudaSuccess) return SNOP_OK;
  return fail(SNOP_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

constexpr int MT_N = 312, MT_M = 156;
constexpr uint64_t MT_A = 0xB5026F5AA96619E9ull, MT_UPPER = 0xFFFFFFFF80000000ull, MT_LOWER = 0x7FFFFFFFull;
constexpr int GRF_WARPS = 4;

__device__ __forceinline__ uint64_t mt_mix(uint64_t cur, uint64_t nxt, uint64_t far) {
  const uint64_t x = (cur & MT_UPPER) | (nxt & MT_LOWER);
  return far ^ (x >> 1) ^ ((x & 1ull) ? MT_A : 0ull);
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  return y ^ (y >> 43);
}

// In-place std::mt19937_64 state transition by one warp. Element i reads mt[i], mt[i+1] (old) and
// mt[i+M] (old) for i < N-M, mt[i+M-N] (already new) after; all reads of a slice precede its writes.
__device__ void mt_twist_warp(uint64_t* mt, int lane) {
  uint64_t v[5];
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const int i = lane + 32 * r;
    if (i < MT_N - MT_M) v[r] = mt_mix(mt[i], mt[i + 1], mt[i + MT_M]);
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const int i = lane + 32 * r;
    if (i < MT_N - MT_M) mt[i] = v[r];
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const int i = MT_N - MT_M + lane + 32 * r;
    if (i < MT_N - 1) v[r] = mt_mix(mt[i], mt[i + 1], mt[i - (MT_N - MT_M)]);
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const int i = MT_N - MT_M + lane + 32 * r;
    if (i < MT_N - 1) mt[i] = v[r];
  }
  __syncwarp();
  if (lane == 0) mt[MT_N - 1] = mt_mix(mt[MT_N - 1], mt[0], mt[MT_M - 1]);
  __syncwarp();
}

// z[s][0..n) = the first n normals of Rng(seed + first + s).
__global__ void __launch_bounds__(32 * GRF_WARPS) grf_normals_kernel(int n_samples, uint64_t seed, int64_t first,
                                                                     int n, double* __restrict__ z) {
  __shared__ uint64_t state[GRF_WARPS][MT_N];
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int s = blockIdx.x * GRF_WARPS + w;
  if (s >= n_samples) return;
  uint64_t* mt = state[w];
  if (lane == 0) {
    uint64_t x = seed + (uint64_t)(first + s);
    mt[0] = x;
    for (int i = 1; i < MT_N; ++i) {
      x = 6364136223846793005ull * (x ^ (x >> 62)) + (uint64_t)i;
      mt[i] = x;
    }
  }
  __syncwarp();
  const int npairs = (n + 1) / 2;
  double* zs = z + (size_t)s * n;
  const double two_pi = 2.0 * 3.14159265358979323846;
  for (int base = 0; base < npairs; base += MT_N / 2) {
    mt_twist_warp(mt, lane);
    for (int p = lane; p < MT_N / 2 && base + p < npairs; p += 32) {
      const uint64_t a = mt_temper(mt[2 * p]), b = mt_temper(mt[2 * p + 1]);
      const double u1 = ((double)(a >> 11) + 1.0) * 0x1.0p-53;
      const double u2 = (double)(b >> 11) * 0x1.0p-53;
      const double r = sqrt(-2.0 * log(u1));
      const double ang = two_pi * u2;
      const int j = 2 * (base + p);
      zs[j] = r * cos(ang);
      if (j + 1 < n) zs[j + 1] = r * sin(ang);
    }
    __syncwarp();
  }
}

// out[s][i] = mean + sum_{j<=i} L[i][j] z[s][j]; negatives[s] += #(out < 0). Tile 32 samples x 32 cells.
constexpr int CT = 32;
__global__ void __launch_bounds__(256) grf_correlate_kernel(int n_samples, int n, const double* __restrict__ L,
                                                            const double* __restrict__ z, double mean,
                                                            double* __restrict__ out, int64_t* __restrict__ negatives) {
  __shared__ double Zs[CT][CT + 1], Ls[CT][CT + 1];
  const int tx = threadIdx.x % CT, ty = threadIdx.x / CT;  // 32 x 8
  const int s0 = blockIdx.y * CT, i0 = blockIdx.x * CT;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int jmax = min(n, i0 + CT);  // L is lower triangular: no tile beyond the diagonal block
  for (int j0 = 0; j0 < jmax; j0 += CT) {
    for (int r = ty; r < CT; r += 8) {
      const int s = s0 + r, j = j0 + tx, i = i0 + r;
      Zs[r][tx] = (s < n_samples && j < n) ? z[(size_t)s * n + j] : 0.0;
      Ls[r][tx] = (i < n && j < n && j <= i) ? L[(size_t)i * n + j] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < CT; ++k) {
      const double l = Ls[tx][k];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(Zs[ty + 8 * q][k], l, acc[q]);
    }
    __syncthreads();
  }
  const int i = i0 + tx;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int s = s0 + ty + 8 * q;
    if (s < n_samples && i < n) {
      const double v = mean + acc[q];
      out[(size_t)s * n + i] = v;
      if (negatives && v < 0.0) atomicAdd(reinterpret_cast<unsigned long long*>(negatives + s), 1ull);
    }
  }
}

// S = raw / (dx sum raw) per sample; the smallest offending sample index goes to *bad.
__global__ void __launch_bounds__(256) normalize_kernel(int n, double dx, const double* __restrict__ raw,
                                                        double* __restrict__ out, int* __restrict__ bad) {
  __shared__ double sh[8];
  const int s = blockIdx.x;
  const double* r = raw + (size_t)s * n;
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) acc += r[i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (threadIdx.x % 32 == 0) sh[threadIdx.x / 32] = acc;
  __syncthreads();
  double tot = 0.0;
  for (int u = 0; u < 8; ++u) tot += sh[u];
  tot *= dx;
  if (!(tot > 0.0) || !isfinite(tot)) {
    if (threadIdx.x == 0) atomicMin(bad, s);
    return;
  }
  for (int i = threadIdx.x; i < n; i += 256) out[(size_t)s * n + i] = r[i] / tot;
}

__global__ void fill_kernel(size_t n, double v, double* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = v;
}

snop_status check_spec(const snop_grid* g, const snop_grf_spec* sp) {
  if (!g || !sp) return fail(SNOP_INVALID_ARGUMENT, "grid/spec is NULL");
  if (!(g->length_cm > 0.0) || g->n_cells < 2) return fail(SNOP_INVALID_ARGUMENT, "grf: need length > 0, n_cells >= 2");
  if (!(sp->variance > 0.0) || !(sp->length_scale_cm > 0.0) || !(sp->jitter > 0.0))
    return fail(SNOP_INVALID_ARGUMENT, "grf: variance, length scale and jitter must be positive");
  return SNOP_OK;
}

// Host Cholesky (once per grid/spec, cached on the context with the device copy in slot 120).
snop_status grf_factor(Ctx& ctx, const snop_grid& g, const snop_grf_spec& sp, const double** dL) {
  const int n = g.n_cells;
  const double key[5] = {g.length_cm, (double)n, sp.variance, sp.length_scale_cm, sp.jitter};
  bool hit = ctx.grf_key.size() == 5;
  for (int i = 0; hit && i < 5; ++i) hit = ctx.grf_key[i] == key[i];
  double* d = static_cast<double*>(ctx.slot(120, (size_t)n * n * sizeof(double)));
  if (!d) return cuda_ok("cudaMalloc", cudaErrorMemoryAllocation);
  if (!hit) {
    const double dx = g.length_cm / n, inv2l2 = 1.0 / (2.0 * sp.length_scale_cm * sp.length_scale_cm);
    std::vector<double> L((size_t)n * n);
    bool ok = false;
    for (double jitter = sp.jitter; !ok && jitter <= 1e-6 * (1.0 + 1e-12); jitter *= 10.0) {
      std::fill(L.begin(), L.end(), 0.0);
      ok = true;
      for (int i = 0; i < n && ok; ++i) {
        const double xi = (i + 0.5) * dx;
        double* Li = L.data() + (size_t)i * n;
        for (int j = 0; j <= i; ++j) {
          const double d = xi - (j + 0.5) * dx;
          const double* Lj = L.data() + (size_t)j * n;
          double s = sp.variance * (std::exp(-d * d * inv2l2) + (i == j ? jitter : 0.0));
          for (int k = 0; k < j; ++k) s -= Li[k] * Lj[k];
          if (i == j) {
            if (!(s > 0.0)) {
              ok = false;
              break;
            }
            Li[i] = std::sqrt(s);
          } else {
            Li[j] = s / Lj[j];
          }
        }
      }
    }
    if (!ok) return fail(SNOP_NUMERICAL_ERROR, "grf: covariance factorization failed after jitter escalation to 1e-6");
    SNOP_TRY(cuda_ok("H2D", cudaMemcpyAsync(d, L.data(), L.size() * sizeof(double), cudaMemcpyHostToDevice,
                                             ctx.stream)));
    SNOP_TRY(cuda_ok("H2D", cudaStreamSynchronize(ctx.stream)));
    ctx.grf_key.assign(key, key + 5);
  }
  *dL = d;
  return SNOP_OK;
}

snop_status grf_sample_dev(Ctx& ctx, const snop_grid& g, const snop_grf_spec& sp, int64_t first, int n_samples,
                           double* out, int64_t* negatives) {
  const double* L = nullptr;
  SNOP_TRY(grf_factor(ctx, g, sp, &L));
  const int n = g.n_cells;
  double* z = static_cast<double*>(ctx.slot(121, (size_t)n_samples * n * sizeof(double)));
  if (!z) return cuda_ok("cudaMalloc", cudaErrorMemoryAllocation);
  grf_normals_kernel<<<(n_samples + GRF_WARPS - 1) / GRF_WARPS, 32 * GRF_WARPS, 0, ctx.stream>>>(n_samples, sp.seed,
                                                                                              first, n, z);
  ctx.launches++;
  if (negatives) cudaMemsetAsync(negatives, 0, (size_t)n_samples * sizeof(int64_t), ctx.stream);
  const dim3 grid((n + CT - 1) / CT, (n_samples + CT - 1) / CT);
  grf_correlate_kernel<<<grid, 256, 0, ctx.stream>>>(n_samples, n, L, z, sp.mean, out, negatives);
  ctx.launches++;
  return cuda_ok("grf sample", cudaGetLastError());
}

snop_status normalize_dev(Ctx& ctx, const snop_grid& g, int n_samples, const double* raw, double* out,
                          int* bad_index) {
  int* bad = static_cast<int*>(ctx.slot(122, sizeof(int)));
  if (!bad) return cuda_ok("cudaMalloc", cudaErrorMemoryAllocation);
  const int big = 0x7fffffff;
  cudaMemcpyAsync(bad, &big, sizeof(int), cudaMemcpyHostToDevice, ctx.stream);
  normalize_kernel<<<n_samples, 256, 0, ctx.stream>>>(g.n_cells, g.length_cm / g.n_cells, raw, out, bad);
  ctx.launches++;
  SNOP_TRY(cuda_ok("normalize", cudaMemcpyAsync(bad_index, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream)));
  return cuda_ok("normalize", cudaStreamSynchronize(ctx.stream));
}

template <class T>
snop_status to_dev(Ctx& ctx, size_t slot, const T* h, size_t n, T** d) {
  *d = static_cast<T*>(ctx.slot(slot, n * sizeof(T)));
  if (!*d) return cuda_ok("cudaMalloc", cudaErrorMemoryAllocation);
  return h ? cuda_ok("H2D", cudaMemcpyAsync(*d, h, n * sizeof(T), cudaMemcpyHostToDevice, ctx.stream)) : SNOP_OK;
}
template <class T>
snop_status to_host(Ctx& ctx, T* h, const T* d, size_t n) {
  if (!h) return SNOP_OK;
  return cuda_ok("D2H", cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, ctx.stream));
}

}  // namespace
}  // namespace snop_impl

using namespace snop_impl;

extern "C" {

snop_status snop_grf_sample(snop_ctx* ctx, int32_t memspace, const snop_grid* grid, const snop_grf_spec* spec,
                            int64_t first_sample, int32_t n_samples, double* field_out, int64_t* negatives) {
  if (!ctx) return fail(SNOP_INVALID_ARGUMENT, "ctx is NULL");
  SNOP_TRY(check_spec(grid, spec));
  if (n_samples < 0 || first_sample < 0) return fail(SNOP_INVALID_ARGUMENT, "n_samples/first_sample must be >= 0");
  if (n_samples == 0) return SNOP_OK;
  if (!field_out) return fail(SNOP_INVALID_ARGUMENT, "field_out is NULL");
  cudaSetDevice(ctx->device);
  const size_t N = (size_t)n_samples * grid->n_cells;
  if (memspace == SNOP_MEM_DEVICE) return grf_sample_dev(*ctx, *grid, *spec, first_sample, n_samples, field_out, negatives);
  if (memspace != SNOP_MEM_HOST) return fail(SNOP_INVALID_ARGUMENT, "memspace must be HOST(0) or DEVICE(1)");
  double* out;
  int64_t* neg = nullptr;
  SNOP_TRY(to_dev<double>(*ctx, 123, nullptr, N, &out));
  if (negatives) SNOP_TRY(to_dev<int64_t>(*ctx, 124, nullptr, (size_t)n_samples, &neg));
  SNOP_TRY(grf_sample_dev(*ctx, *grid, *spec, first_sample, n_samples, out, neg));
  SNOP_TRY(to_host(*ctx, field_out, out, N));
  SNOP_TRY(to_host(*ctx, negatives, neg, (size_t)n_samples));
  return cuda_ok("grf sample", cudaStreamSynchronize(ctx->stream));
}

snop_status snop_normalize_source(snop_ctx* ctx, int32_t memspace, const snop_grid* grid, int32_t n_samples,
                                  const double* raw, double* out) {
  if (!ctx || !grid) return fail(SNOP_INVALID_ARGUMENT, "ctx/grid is NULL");
  if (!(grid->length_cm > 0.0) || grid->n_cells < 1 || n_samples < 0) return fail(SNOP_INVALID_ARGUMENT, "bad grid/n");
  if (n_samples == 0) return SNOP_OK;
  if (!raw || !out) return fail(SNOP_INVALID_ARGUMENT, "NULL array");
  cudaSetDevice(ctx->device);
  const size_t N = (size_t)n_samples * grid->n_cells;
  const double* r = raw;
  double* o = out;
  const bool host = memspace == SNOP_MEM_HOST;
  if (!host && memspace != SNOP_MEM_DEVICE) return fail(SNOP_INVALID_ARGUMENT, "memspace must be HOST(0) or DEVICE(1)");
  if (host) {
    double* d;
    SNOP_TRY(to_dev<double>(*ctx, 123, raw, N, &d));
    r = d;
    SNOP_TRY(to_dev<double>(*ctx, 125, nullptr, N, &o));
  }
  int bad = 0;
  SNOP_TRY(normalize_dev(*ctx, *grid, n_samples, r, o, &bad));
  if (bad != 0x7fffffff)
    return fail(SNOP_INVALID_ARGUMENT,
                "normalize_source: sample " + std::to_string(bad) + " has a non-positive integral (resample)");
  if (host) {
    SNOP_TRY(to_host(*ctx, out, static_cast<const double*>(o), N));
    return cuda_ok("normalize", cudaStreamSynchronize(ctx->stream));
  }
  return SNOP_OK;
}

snop_status snop_generate_dataset(snop_ctx* ctx, int32_t memspace, const snop_grid* grid, int32_t order,
                                  const snop_grf_spec* spec, int32_t n_samples, double sigma_t_star,
                                  double sigma_s0_star, double tolerance, double* sources, double* fluxes,
                                  int32_t* iterations) {
  if (!ctx) return fail(SNOP_INVALID_ARGUMENT, "ctx is NULL");
  SNOP_TRY(check_spec(grid, spec));
  if (grid->n_cells > kMaxCells) return fail(SNOP_INVALID_ARGUMENT, "n_cells exceeds the per-CTA sweep limit");
  if (order < 2 || order > 128 || order % 2) return fail(SNOP_INVALID_ARGUMENT, "quadrature order must be even in [2,128]");
  if (!(sigma_t_star > 0.0) || !(tolerance > 0.0)) return fail(SNOP_INVALID_ARGUMENT, "need sigma_t* > 0, tolerance > 0");
  if (n_samples < 0) return fail(SNOP_INVALID_ARGUMENT, "n_samples must be >= 0");
  if (n_samples == 0) return SNOP_OK;
  if (!sources || !fluxes || !iterations) return fail(SNOP_INVALID_ARGUMENT, "NULL array");
  const bool host = memspace == SNOP_MEM_HOST;
  if (!host && memspace != SNOP_MEM_DEVICE) return fail(SNOP_INVALID_ARGUMENT, "memspace must be HOST(0) or DEVICE(1)");
  cudaSetDevice(ctx->device);
  const size_t N = (size_t)n_samples * grid->n_cells;
  double *S = sources, *phi = fluxes, *st, *ss;
  int32_t* it = iterations;
  if (host) {
    SNOP_TRY(to_dev<double>(*ctx, 126, nullptr, N, &S));
    SNOP_TRY(to_dev<double>(*ctx, 127, nullptr, N, &phi));
    SNOP_TRY(to_dev<int32_t>(*ctx, 128, nullptr, (size_t)n_samples, &it));
  }
  double* raw;
  uint8_t* conv;
  SNOP_TRY(to_dev<double>(*ctx, 123, nullptr, N, &raw));
  SNOP_TRY(to_dev<double>(*ctx, 129, nullptr, N, &st));
  SNOP_TRY(to_dev<double>(*ctx, 130, nullptr, N, &ss));
  SNOP_TRY(to_dev<uint8_t>(*ctx, 131, nullptr, (size_t)n_samples, &conv));
  SNOP_TRY(grf_sample_dev(*ctx, *grid, *spec, 0, n_samples, raw, nullptr));
  int bad = 0;
  SNOP_TRY(normalize_dev(*ctx, *grid, n_samples, raw, S, &bad));
  if (bad != 0x7fffffff)
    return fail(SNOP_NUMERICAL_ERROR, "generate_dataset: sample " + std::to_string(bad) + " has a non-positive integral");
  fill_kernel<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(N, sigma_t_star, st);
  fill_kernel<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(N, sigma_s0_star, ss);
  ctx->launches += 2;
  snop_solver_config cfg{};
  cfg.tolerance = cfg.tolerance_k = cfg.tolerance_phi = tolerance;
  cfg.max_inner = 10000;
  cfg.max_outer = 1;
  SNOP_TRY(launch_source_iteration(*ctx, *grid, order, n_samples, st, ss, nullptr, S, cfg, nullptr, phi, nullptr, it,
                                   conv));
  std::vector<uint8_t> cv(n_samples);
  SNOP_TRY(to_host(*ctx, cv.data(), static_cast<const uint8_t*>(conv), (size_t)n_samples));
  if (host) {
    SNOP_TRY(to_host(*ctx, sources, static_cast<const double*>(S), N));
    SNOP_TRY(to_host(*ctx, fluxes, static_cast<const double*>(phi), N));
    SNOP_TRY(to_host(*ctx, iterations, static_cast<const int32_t*>(it), (size_t)n_samples));
  }
  SNOP_TRY(cuda_ok("generate_dataset", cudaStreamSynchronize(ctx->stream)));
  for (int s = 0; s < n_samples; ++s)
    if (!cv[s]) return fail(SNOP_NUMERICAL_ERROR, "generate_dataset: sample " + std::to_string(s) + " did not converge");
  return SNOP_OK;
}

}  // extern "C"
