// Bring-up test: one tcgen05.mma.kind::tf32 (M = 128, N = 32, K = 8) with an MN-major A operand,
// B K-major 128-byte-swizzled. Round 1 used the plain 128-B swizzle for MN-major A and got zeros:
// for MN-major tf32 the only valid layout is SWIZZLE_128B_BASE32B (layout type 1; CUTLASS
// Layout_MN_SW128_32B_Atom): 128-B rows (32 MN elements) per K index, atoms of 4 K rows with the
// 32-byte chunk index XOR (k % 4), K groups of 4 rows SBO apart, 32-element MN blocks LBO apart.
// amaj = 2 tests that layout (M-block stride MBS, K-group stride KGS).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o umma_mn_test umma_mn_test.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const float* A, const float* Bm, float* D, uint32_t mbs, uint32_t lbo, uint32_t sbo, int amaj,
                  uint32_t kgs) {
  extern __shared__ __align__(1024) unsigned char raw[];
  const uint32_t pad = (1024u - (su32(raw) & 1023u)) & 1023u;
  unsigned char* sm = raw + pad;
  float* sa = reinterpret_cast<float*>(sm);                 // A region: 4 M blocks at mbs bytes
  float* sb = reinterpret_cast<float*>(sm + 4 * 4096);      // B region: 32 rows x 128 B (K-major SW128)
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x;
  // zero
  for (int i = t; i < (4 * 4096 + 4096) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  __syncthreads();
  // A[m][k], k < 8: MN-major SW128: block m/32 at mbs, row k (128 B), 16-B chunk ((m%32)/4) ^ (k%8)
  for (int i = t; i < 128 * 8; i += blockDim.x) {
    const int m = i / 8, kk = i % 8;
    const uint32_t off = amaj == 2 ? (m / 32) * mbs + (kk / 4) * kgs + (kk % 4) * 128 +
                                         ((((m % 32) / 8) ^ (kk % 4)) * 32) + (m % 8) * 4
                       : amaj ? (m / 32) * mbs + kk * 128 + ((((m % 32) / 4) ^ (kk % 8)) * 16) + (m % 4) * 4
                              : (m / 8) * 1024 + (m % 8) * 128 + (((kk / 4) ^ (m % 8)) * 16) + (kk % 4) * 4;
    *reinterpret_cast<float*>(sm + off) = A[m * 8 + kk];
  }
  // B[n][k]: K-major SW128: row n at (n/8)*1024 + (n%8)*128, 16-B chunk (k/4) ^ (n%8)
  for (int i = t; i < 32 * 8; i += blockDim.x) {
    const int n = i / 8, kk = i % 8;
    const uint32_t off = (n / 8) * 1024 + (n % 8) * 128 + (((kk / 4) ^ (n % 8)) * 16) + (kk % 4) * 4;
    *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(sb) + off) = Bm[n * 8 + kk];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  if (t == 0) {
    const uint32_t ad = su32(sa), bd = su32(sb);
    const uint64_t adesc = (uint64_t)((ad >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
                           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) |
                           ((uint64_t)(amaj == 2 ? 1 : 2) << 61);
    const uint64_t bdesc = (uint64_t)((bd >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
                           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
    const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(amaj ? 1 : 0) << 15) | ((uint32_t)(32 >> 3) << 17) |
                        ((uint32_t)(128 >> 4) << 24);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(tmem), "l"(adesc), "l"(bdesc), "r"(id) : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(su32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t v[32];
  const int w = t >> 5, lane = t & 31;
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(tmem + ((uint32_t)(w * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int j = 0; j < 32; ++j) D[(w * 32 + lane) * 32 + j] = __uint_as_float(v[j]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

static float tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y; }

int main() {
  std::vector<float> A(128 * 8), B(32 * 8), D(128 * 32), R(128 * 32);
  for (int m = 0; m < 128; ++m) for (int k = 0; k < 8; ++k) A[m * 8 + k] = (float)((m * 7 + k * 3) % 11) - 5.f + 0.25f * k;
  for (int n = 0; n < 32; ++n) for (int k = 0; k < 8; ++k) B[n * 8 + k] = (float)((n * 5 + k) % 7) - 3.f;
  for (int m = 0; m < 128; ++m) for (int n = 0; n < 32; ++n) { double s = 0; for (int k = 0; k < 8; ++k) s += (double)tf32(A[m*8+k]) * tf32(B[n*8+k]); R[m*32+n] = (float)s; }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  const uint32_t opts[4] = {128, 1024, 4096, 8192};
  for (int amaj = 0; amaj <= 2; amaj += 2)
    for (uint32_t mbs : {1024u, 2048u, 4096u})
      for (uint32_t kgs : {512u, 1024u})
        for (int swap = 0; swap < 2; ++swap) {
          const uint32_t lbo = amaj ? (swap ? kgs : mbs) : 128u, sbo = amaj ? (swap ? mbs : kgs) : 1024u;
          if (amaj == 0 && (mbs != 1024u || kgs != 512u || swap)) continue;
          if (amaj == 2 && kgs * 2 > mbs) continue;  // the two K groups fit inside one M block's span
          cudaMemset(dD, 0, D.size() * 4);
          k<<<1, 128, 40 * 1024>>>(dA, dB, dD, mbs, lbo, sbo, amaj, kgs);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("mbs %u lbo %u sbo %u: %s\n", mbs, lbo, sbo, cudaGetErrorString(e)); return 1; }
          cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
          double err = 0; for (size_t i = 0; i < D.size(); ++i) err = fmax(err, fabs(D[i] - R[i]));
          printf("a_major %d  M-block stride %5u  K-group stride %5u  LBO %5u  SBO %5u : max abs err %g%s\n", amaj,
                 mbs, kgs, lbo, sbo, err, err < 1e-3 ? "   <== OK" : "");
        }
  (void)opts;
  return 0;
}
