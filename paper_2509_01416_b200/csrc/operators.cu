// operators.cu — K3 recast-source kernel and the SolutionOperator entry points.
#include <string>

#define SNOP_PHASE_SYM g_phase_cycles_ops
#include "snop_internal.h"

using namespace snop_impl;

namespace {

// K3 (paper Eq. 24): s = S + [(Ss0 - Ss0*) - (St - St*)] phi. Pure streaming:
// 32 B read + 8 B written per cell; grid-stride over the flattened batch, 2 cells per thread
// with 16-byte vector accesses when aligned.
__global__ void recast_source_kernel(size_t n, const double* __restrict__ S, const double* __restrict__ phi,
                                     const double* __restrict__ st, const double* __restrict__ ss,
                                     double tstar, double sstar, double* __restrict__ out) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t n2 = n / 2;
  const double2* S2 = reinterpret_cast<const double2*>(S);
  const double2* P2 = reinterpret_cast<const double2*>(phi);
  const double2* T2 = reinterpret_cast<const double2*>(st);
  const double2* C2 = reinterpret_cast<const double2*>(ss);
  double2* O2 = reinterpret_cast<double2*>(out);
  const double d0 = tstar - sstar;  // s = S + (Ss0 - St + (St* - Ss0*)) phi
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
    const double2 s = __ldcs(S2 + i), p = __ldcs(P2 + i), t = __ldcs(T2 + i), c = __ldcs(C2 + i);
    double2 o;
    o.x = fma((c.x - t.x) + d0, p.x, s.x);
    o.y = fma((c.y - t.y) + d0, p.y, s.y);
    __stcs(O2 + i, o);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) {
    const size_t i = n - 1;
    out[i] = fma((ss[i] - st[i]) + d0, phi[i], S[i]);
  }
}

// balance_report, one CTA per instance.
__global__ void __launch_bounds__(256) balance_kernel(int n, double dx, const double* __restrict__ st,
                                                      const double* __restrict__ ss, const double* __restrict__ src,
                                                      const double* __restrict__ phi, const double* __restrict__ leak,
                                                      double* __restrict__ residual, int* __restrict__ flags) {
  __shared__ double sh[2][8];
  const int b = blockIdx.x;
  const size_t o = (size_t)b * n;
  double ab = 0.0, pr = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) {
    ab = fma(st[o + i] - ss[o + i], phi[o + i], ab);
    pr += src[o + i];
  }
  for (int k = 16; k > 0; k >>= 1) {
    ab += __shfl_xor_sync(0xffffffffu, ab, k);
    pr += __shfl_xor_sync(0xffffffffu, pr, k);
  }
  if (threadIdx.x % 32 == 0) {
    sh[0][threadIdx.x / 32] = ab;
    sh[1][threadIdx.x / 32] = pr;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, p = 0.0;
    for (int u = 0; u < 8; ++u) {
      a += sh[0][u];
      p += sh[1][u];
    }
    a *= dx;
    p *= dx;
    if (p == 0.0) {
      atomicOr(flags, FLAG_ZERO_PRODUCTION);
      residual[b] = __longlong_as_double(0x7ff8000000000000ll);
    } else {
      residual[b] = fabs(leak[2 * b] + leak[2 * b + 1] + a - p) / fabs(p);
    }
  }
}

}  // namespace

namespace snop_impl {

snop_status launch_balance(Ctx& ctx, const snop_grid& g, int batch, const double* st, const double* ss_out,
                           const double* src, const double* phi, const double* leak, double* residual) {
  if (batch == 0) return SNOP_OK;
  balance_kernel<<<batch, 256, 0, ctx.stream>>>(g.n_cells, g.length_cm / g.n_cells, st, ss_out, src, phi, leak,
                                                 residual, ctx.d_flags);
  ctx.launches++;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("balance_kernel: ") + cudaGetErrorString(e));
    return SNOP_CUDA_ERROR;
  }
  return SNOP_OK;
}

snop_status launch_recast(Ctx& ctx, size_t n, const double* S, const double* phi, const double* st,
                          const double* ss, double tstar, double sstar, double* out) {
  if (n == 0) return SNOP_OK;
  const bool aligned = ((reinterpret_cast<uintptr_t>(S) | reinterpret_cast<uintptr_t>(phi) |
                         reinterpret_cast<uintptr_t>(st) | reinterpret_cast<uintptr_t>(ss) |
                         reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  if (!aligned) {
    set_error("recast_source: device arrays must be 16-byte aligned");
    return SNOP_INVALID_ARGUMENT;
  }
  const int threads = 256;
  size_t blocks = (n / 2 + threads - 1) / threads;
  const size_t cap = (size_t)ctx.sm_count * 8;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  recast_source_kernel<<<(unsigned)blocks, threads, 0, ctx.stream>>>(n, S, phi, st, ss, tstar, sstar, out);
  ctx.launches++;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("recast_source_kernel: ") + cudaGetErrorString(e));
    return SNOP_CUDA_ERROR;
  }
  return SNOP_OK;
}

}  // namespace snop_impl
