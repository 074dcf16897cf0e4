// Microbenchmark: FP64 FMA throughput, SHFL throughput, rcp.approx.ftz.f64 accuracy on this B200.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__global__ void dfma_tp(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void shfl_tp(double* out, int iters) {
  double a = threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
  for (int i = 0; i < iters; ++i) {
    a = __shfl_xor_sync(0xffffffff, a, 1); b = __shfl_xor_sync(0xffffffff, b, 2);
    c = __shfl_xor_sync(0xffffffff, c, 4); d = __shfl_xor_sync(0xffffffff, d, 8);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}

__global__ void rcp_err(double* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double t = 0.1 + 500.0 * (double)i / n;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(t));
  double e = fma(-t, r, 1.0);
  e = fma(e, e, e);
  double r2 = fma(r, e, r);
  out[2 * i] = fabs(r * t - 1.0);
  out[2 * i + 1] = fabs(r2 - 1.0 / t) * t;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("%s SMs=%d clock=%d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  double* d; cudaMalloc(&d, 1 << 26);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 20000;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  dfma_tp<<<blocks, threads>>>(d, 100);
  cudaEventRecord(a); dfma_tp<<<blocks, threads>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double fmas = (double)blocks * threads * iters * 8;
  printf("DFMA: %.3f TFMA/s = %.2f TFLOP/s, %.1f FMA/clk/SM at nominal clock\n", fmas / ms / 1e9, 2 * fmas / ms / 1e9,
         fmas / (ms * 1e-3) / p.multiProcessorCount / (p.clockRate * 1e3));
  shfl_tp<<<blocks, threads>>>(d, 100);
  cudaEventRecord(a); shfl_tp<<<blocks, threads>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  double sh = (double)blocks * threads * iters * 4 * 2;  // 64-bit shfl = 2 SHFL.32
  printf("SHFL: %.2f lane-shfl32/clk/SM\n", sh / (ms * 1e-3) / p.multiProcessorCount / (p.clockRate * 1e3));
  int n = 1 << 20;
  rcp_err<<<(n + 255) / 256, 256>>>(d, n);
  double* h = new double[2 * n];
  cudaMemcpy(h, d, 16 * (size_t)n, cudaMemcpyDeviceToHost);
  double m0 = 0, m1 = 0;
  for (int i = 0; i < n; ++i) { m0 = fmax(m0, h[2 * i]); m1 = fmax(m1, h[2 * i + 1]); }
  printf("rcp.approx.ftz.f64 max rel err %.3e (log2 %.1f); after cubic Newton %.3e\n", m0, log2(m0), m1);
  return 0;
}
