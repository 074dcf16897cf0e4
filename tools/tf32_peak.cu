// tf32_peak.cu — measured tcgen05 kind::tf32 tensor throughput of one B200 (the denominator of the
// operator GEMMs' tensor roofline; MEASURED_PEAKS.json carries bf16 only). One CTA per SM, one
// elected thread issues back-to-back tcgen05.mma.cta_group::1.kind::tf32 (M = 128, N = 256, K = 8)
// on shared-memory operands (K-major, no swizzle), accumulating in TMEM; the kernel is timed with
// CUDA events. Also times kind::f16 (bf16, K = 16) the same way as a cross-check against the
// cuBLAS bf16 number. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tf32_peak
// tools/tf32_peak.cu ; run on a B200: tools/tf32_peak  -> one JSON line.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// kind::tf32: a/b format 2 (TF32); kind::f16 with bf16 inputs: a/b format 1 (BF16). D = F32.
template <bool BF16>
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
  return (1u << 4) | ((BF16 ? 1u : 2u) << 7) | ((BF16 ? 1u : 2u) << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

template <bool BF16>
__global__ void __launch_bounds__(128) mma_loop(int iters, unsigned long long* sink) {
  constexpr int M = 128, N = 256;
  __shared__ __align__(1024) uint8_t a_s[M * 32];  // 128 rows x 32 B (tf32 K = 8 / bf16 K = 16)
  __shared__ __align__(1024) uint8_t b_s[N * 32];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < M * 32 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(a_s)[i] = 0;
  for (int i = threadIdx.x; i < N * 32 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(b_s)[i] = 0;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (threadIdx.x == 0) {
    // core matrix = 8 rows x 16 B; two core matrices along K (32 B per row): LBO 128 B, SBO 256 B
    const uint64_t ad = sdesc(smem_u32(a_s), 128, 256), bd = sdesc(smem_u32(b_s), 128, 256);
    constexpr uint32_t id = idesc<BF16>(M, N);
    for (int i = 0; i < iters; ++i) {
      if (BF16)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                     "l"(ad), "l"(bd), "r"(id), "r"(i > 0 ? 1u : 0u) : "memory");
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                     "l"(ad), "l"(bd), "r"(id), "r"(i > 0 ? 1u : 0u) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((threadIdx.x / 32 * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  if (v == 0x7fc00001u) atomicAdd(sink, 1ull);  // keep the result live
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

template <bool BF16>
double run(int sms, int iters, unsigned long long* sink) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mma_loop<BF16><<<sms, 128>>>(1000, sink);  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    mma_loop<BF16><<<sms, 128>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double k = BF16 ? 16 : 8;
  return 2.0 * 128 * 256 * k * (double)iters * sms / (best * 1e-3) / 1e12;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const int iters = 200000;
  const double tf32 = run<false>(sms, iters, sink);
  const double bf16 = run<true>(sms, iters, sink);
  const cudaError_t e = cudaDeviceSynchronize();
  printf("{\"tf32_tflops\": %.1f, \"bf16_tflops_tcgen05_loop\": %.1f, \"sms\": %d, \"max_clock_mhz\": %d, "
         "\"shape\": \"M128 N256 (tf32 K8 / bf16 K16), cta_group::1, smem operands\", \"iters_per_cta\": %d, "
         "\"cuda_status\": \"%s\"}\n",
         tf32, bf16, sms, clk / 1000, iters, cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
