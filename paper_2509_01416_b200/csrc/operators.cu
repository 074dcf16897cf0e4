// operators.cu — K3 recast-source kernel and the SolutionOperator entry points.
#include <string>

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

}  // namespace

namespace snop_impl {

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
