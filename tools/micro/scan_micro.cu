// Microbenchmark: cycles of K1's scan phase (scan_one) in isolation, one CTA of NT threads.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2509_01416_b200/csrc/snop_device.cuh"
using namespace snop_dev;
constexpr int K = 8, NT = 256;

template <bool FWD>
__device__ __forceinline__ void part(SweepSmem<K, NT>& sm, int q, int lane, int what) {
  constexpr int E = NT / 32, S = E + 1, D = FWD ? 1 : -1;
  const int base = FWD ? lane * S : (31 - lane) * S + (E - 1);
  const double* a = sm.agg[q][0] + base;
  const double* b = sm.agg[q][FWD ? 1 : 2] + base;
  double* XA = sm.xmap[q][FWD ? 0 : 2] + base;
  double* XB = sm.xmap[q][FWD ? 1 : 3] + base;
  double A = a[0], B = b[0];
  if (what & 8) {  // preloaded registers, prefixes kept in registers, tail from registers
    double pa[E], pb[E];
#pragma unroll
    for (int e = 0; e < E; ++e) { pa[e] = a[D * e]; pb[e] = b[D * e]; }
#pragma unroll
    for (int e = 1; e < E; ++e) { pb[e] = fma(pa[e], pb[e - 1], pb[e]); pa[e] *= pa[e - 1]; }
    A = pa[E - 1]; B = pb[E - 1];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double ap = __shfl_up_sync(0xffffffffu, A, o), bq = __shfl_up_sync(0xffffffffu, B, o);
      if (lane >= o) { B = fma(A, bq, B); A *= ap; }
    }
    double Ax = __shfl_up_sync(0xffffffffu, A, 1), Bx = __shfl_up_sync(0xffffffffu, B, 1);
    if (lane == 0) { Ax = 1.0; Bx = 0.0; }
    XA[0] = Ax; XB[0] = Bx;
#pragma unroll
    for (int e = 1; e < E; ++e) { XA[D * e] = Ax * pa[e - 1]; XB[D * e] = fma(pa[e - 1], Bx, pb[e - 1]); }
    return;
  }
  if (what & 1) {
    XA[0] = A; XB[0] = B;
#pragma unroll
    for (int e = 1; e < E; ++e) {
      const double ae = a[D * e];
      B = fma(ae, B, b[D * e]);
      A *= ae;
      XA[D * e] = A; XB[D * e] = B;
    }
  }
  if (what & 2) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double ap = __shfl_up_sync(0xffffffffu, A, o), bq = __shfl_up_sync(0xffffffffu, B, o);
      if (lane >= o) { B = fma(A, bq, B); A *= ap; }
    }
  }
  if (what & 4) {
#pragma unroll
    for (int e = E - 1; e >= 1; --e) {
      const double pa = XA[D * (e - 1)], pb = XB[D * (e - 1)];
      XA[D * e] = A * pa; XB[D * e] = fma(pa, B, pb);
    }
  }
  XA[0] = A; XB[0] = B;
}

__global__ void bench(int reps, int mode, unsigned long long* out, double* sink, int nscan) {
  extern __shared__ __align__(32) unsigned char raw[];
  auto& sm = *reinterpret_cast<SweepSmem<K, NT>*>(raw);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int i = t; i < SweepSmem<K, NT>::NP_PAD; i += NT)
    for (int q = 0; q < 2; ++q) {
      sm.agg[q][0][i] = 0.99 + 1e-4 * i;
      sm.agg[q][1][i] = 0.01 * i;
      sm.agg[q][2][i] = 0.02 * i;
    }
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (mode == 0) scan_phase<K, NT, 2, false>(sm, lane, warp, 0);
    else if (mode >= 2 && warp < nscan) {
      const int what = mode == 9 ? 8 : mode - 1;
      if ((warp & 1) == 0) part<true>(sm, warp >> 1, lane, what);
      else part<false>(sm, warp >> 1, lane, what);
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (t == 0) out[0] = (unsigned long long)(t1 - t0);
  if (t == 0) sink[0] = sm.xmap[0][1][100] + sm.total[1][3];
}

int main() {
  unsigned long long* d;
  double* s;
  cudaMalloc(&d, 8);
  cudaMalloc(&s, 8);
  size_t smem = sizeof(SweepSmem<K, NT>);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int nscan = 1; nscan <= 4; nscan *= 2)
  for (int mode = 0; mode < 10; ++mode) {
    bench<<<1, NT, smem>>>(1000, mode, d, s, nscan);
    unsigned long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("nscan %d mode %d (parts mask %d): %.1f cycles per scan phase (+barrier)\n", nscan, mode, mode - 1, c / 1000.0);
  }
  return 0;
}
