// Dependent-chain latencies on B200 (one warp): DFMA, DMUL, SHFL (double = 2 x 32-bit), LDS.64.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(int n, double seed, unsigned long long* out, double* sink) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (double)((i * 7 + 1) & 1023);
  __syncthreads();
  double x = seed + threadIdx.x, y = 0.999, z = 1e-3;
  int idx = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < n; ++i) {
    if (MODE == 0) x = fma(x, y, z);
    else if (MODE == 1) x = x * y;
    else if (MODE == 2) x = __shfl_up_sync(0xffffffffu, x, 1);
    else if (MODE == 3) { idx = (int)sm[idx & 1023]; }
    else if (MODE == 4) { x = fma(__shfl_up_sync(0xffffffffu, x, 1), y, z); }
    else if (MODE == 5) { double t = __shfl_up_sync(0xffffffffu, x, 1); if (threadIdx.x >= 1) x = fma(x, t, z); }
    else if (MODE == 6) { x = __int_as_float(__shfl_up_sync(0xffffffffu, __float_as_int((float)x), 1)); }
    else if (MODE == 7) { float f = (float)x; f = __fmaf_rn(f, 0.999f, 1e-3f); x = f; }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  sink[threadIdx.x] = x + idx;
}
template <int M>
void run(const char* name, unsigned long long* d, double* s) {
  k<M><<<1, 32>>>(8000, 1.0, d, s);
  unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("%-24s %.1f cycles per dependent step\n", name, c / 8000.0);
}
int main() {
  unsigned long long* d; double* s;
  cudaMalloc(&d, 8); cudaMalloc(&s, 8 * 1024);
  run<0>("DFMA", d, s); run<1>("DMUL", d, s); run<2>("SHFL.UP f64 (2x32)", d, s); run<3>("LDS.64 -> idx", d, s);
  run<4>("SHFL f64 + DFMA", d, s); run<5>("SHFL f64 + pred DFMA", d, s); run<6>("SHFL f32 + cvt", d, s);
  run<7>("cvt + FFMA + cvt", d, s);
  return 0;
}
