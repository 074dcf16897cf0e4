// Microbenchmark: DFMA dependent latency, MUFU.RCP64H throughput, SHFL latency (one warp / full SM).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_lat(double* out, long long* cyc, int iters) {
  double a = threadIdx.x * 1e-3;
  const double b = 0.999999, c = 1e-7;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); }
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void shfl_lat(double* out, long long* cyc, int iters) {
  double a = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = __shfl_up_sync(0xffffffff, a, 1) + 1.0; }
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void rcp_tp(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double s = 0;
  for (int i = 0; i < iters; ++i) {
    double r0, r1, r2, r3;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(a0));
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r1) : "d"(a1));
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r2) : "d"(a2));
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r3) : "d"(a3));
    a0 += 1e-9; a1 += 1e-9; a2 += 1e-9; a3 += 1e-9;
    s += r0 + r1 + r2 + r3;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_tp_warps(double* out, int iters) {  // 2 independent chains per thread
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) { a0 = fma(a0, b, c); a1 = fma(a1, b, c); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* d; long long* c; cudaMalloc(&d, 1 << 26); cudaMalloc(&c, 64);
  long long h;
  dfma_lat<<<1, 32>>>(d, c, 1000); dfma_lat<<<1, 32>>>(d, c, 10000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)h / 40000);
  shfl_lat<<<1, 32>>>(d, c, 1000); shfl_lat<<<1, 32>>>(d, c, 10000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("SHFL.64(2x32)+DADD dependent latency: %.2f cycles\n", (double)h / 10000);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 8, thr = 256, it = 4000;
  rcp_tp<<<blocks, thr>>>(d, 10);
  cudaEventRecord(e0); rcp_tp<<<blocks, thr>>>(d, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("MUFU.RCP64H: %.2f lanes/clk/SM (at 1.965 GHz)\n", (double)blocks * thr * it * 4 / (ms * 1e-3) / p.multiProcessorCount / 1.965e9);
  for (int w = 1; w <= 16; w *= 2) {
    dfma_tp_warps<<<p.multiProcessorCount, 32 * w>>>(d, 100);
    cudaEventRecord(e0); dfma_tp_warps<<<p.multiProcessorCount, 32 * w>>>(d, 20000); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA 2-chain/thread, %2d warps/SM: %.1f FMA/clk/SM\n", w, (double)p.multiProcessorCount * 32 * w * 20000 * 2 / (ms * 1e-3) / p.multiProcessorCount / 1.965e9);
  }
  return 0;
}
