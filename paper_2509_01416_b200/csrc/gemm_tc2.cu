// gemm_tc2.cu — warp-specialised, TMA-fed tcgen05 GEMM (3xTF32) for K-contiguous operands with
// K <= 128 (the FNO inverse-DFT + W contraction, the FNO projection head, the DeepONet hidden
// layers and combine). Same contract and accuracy as gemm_tc.cu's non-split kernel:
//
//   C(b, m, n) = act( alpha * sum_k A(b, m, k) B(b, n, k) + bias[n] )   (or the fused row-dot)
//
// Roles (one persistent CTA per SM, 14 warps):
//   warp 0      TMA producer: 2-D tensor-map loads of the raw fp32 A (128 x 32) and B (N x 32)
//               chunks into a 128-byte-swizzled K-major stage (cp.async.bulk.tensor, mbarrier tx)
//   warps 2-5   converters: per stage, hi = x as loaded (read as tf32) and lo = rnd(x - trunc(x)) into the lo
//               buffer — an element-wise pass, so the swizzled layout is preserved
//   warp 1      MMA issuer: 4 k-steps x 3 tcgen05.mma.kind::tf32 (lo*hi, hi*lo, hi*hi) per chunk
//               into one of two TMEM accumulators, commits free the stage / publish the tile
//   warps 6-21  epilogue: tcgen05.ld of the finished accumulator (warp w reads TMEM lanes
//               32 (w % 4) .., one of four column quarters), bias / activation (compile-time) /
//               fp32-fp64 store or the fused row-dot; the other accumulator is meanwhile filled
//               by the next tile's MMAs
// Stages are recycled through full (TMA) -> conv (converters) -> empty (MMA commit) mbarriers,
// so global loads, the split, the tensor core and the epilogue all overlap.
#include <cuda.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "gemm.cuh"

namespace snop_ops {
namespace tc2 {

constexpr int TM = 128;
constexpr int KC = 32;  // fp32 per 128-byte swizzle row
constexpr int NWARPS = 14;
#ifndef SNOP_TC2_NCONV
#define SNOP_TC2_NCONV 4
#endif
constexpr int CONV0 = 2, NCONV = SNOP_TC2_NCONV, EPI0 = CONV0 + NCONV;
// epilogue warps: 4 per TMEM lane quarter (column quarters: 16 columns at N = 64, 32 at N = 128).
// The element-wise epilogue (bias, GELU, row-dot, staging) is the pipeline's bottleneck, so it gets
// 16 of the 22 warps (80 registers each, no spills); 8 epilogue warps measured 3-6% slower
// (N = 64: layer-0 inverse 455 -> 504 us, the 3-chunk inverse+W tiles unchanged at ~620 us).
#ifndef SNOP_TC2_NEPI64
#define SNOP_TC2_NEPI64 16
#endif
template <int N>
constexpr int nepi() { return N == 64 ? SNOP_TC2_NEPI64 : 16; }
template <int N>
constexpr int threads() { return (EPI0 + nepi<N>()) * 32; }

// BR ("B resident"): a batch-invariant, pre-split B operand with K <= 64 (the FNO projection
// weights) is loaded into shared memory once per CTA; the stages then carry only A, so the TMA
// streams 16 instead of 48 KB per K chunk and four stages fit.
#ifndef SNOP_TC2_S64
#define SNOP_TC2_S64 3
#endif
template <int N, bool BR = false>
constexpr int stages() { return BR ? 4 : (N == 64 ? SNOP_TC2_S64 : 3); }
constexpr int BR_CHUNKS = 2;
// N = 64 tiles are stored through shared memory by TMA (two 128 x 32 fp32 halves, 128-B swizzle)
template <int N>
#ifndef SNOP_TC2_CST
#define SNOP_TC2_CST 1
#endif
constexpr int cst_floats() { return (N == 64 && SNOP_TC2_CST) ? 2 * TM * N : 4; }  // double-buffered

template <int N, bool BR = false>
struct alignas(1024) Stage {
  float a_hi[TM * KC];  // 16 KB, 1024-B aligned (swizzle atom = 8 rows x 128 B)
  float a_lo[TM * KC];
  float b_hi[BR ? 4 : N * KC];
  float b_lo[BR ? 4 : N * KC];
};

template <int N, bool BR = false>
struct Smem {
  Stage<N, BR> st[stages<N, BR>()];
  alignas(1024) float bres[BR ? 2 * BR_CHUNKS * N * KC : 4];  // resident B: [hi c0, hi c1, lo c0, lo c1]
  uint64_t bres_full;
  alignas(1024) float cst[cst_floats<N>()];  // output tile staging for the TMA store (N = 64)
  uint64_t full[stages<N, BR>()], conv[stages<N, BR>()], empty[stages<N, BR>()];
  uint64_t acc_full[2], acc_empty[2];
  uint64_t stg_full[2], stg_free[2];  // TMA-store staging hand-off (decoupled epilogue)
  uint32_t tmem_base;
  alignas(16) float ep_bias[2][N];  // per accumulator: this tile's bias / row-dot weights / rank-2 columns
  float ep_rw[2][N];
  float ep_ra[2][N];
  float ep_rb[2][N];
};

// n / d for n < 2^31 by multiply-high (host-computed magic; q = (umulhi(n, m) + n) >> s): the tile
// decomposition runs in every warp for every tile, and the K = 64..96 contractions have ~3 K chunks
// per tile, so the two integer divisions were ~8% of the warp samples.
struct FastDiv {
  uint32_t m, s;
  void init(uint32_t d) {
    s = 0;
    while ((1ull << s) < d) ++s;
    m = (uint32_t)(((1ull << 32) * ((1ull << s) - d)) / d + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return (uint32_t)(((uint64_t)__umulhi(n, m) + n) >> s);
  }
};

struct Args {
  GemmArgs g;
  FastDiv div_n, div_mn;  // by n_tiles, by n_tiles * m_tiles
  int64_t a1_brows, a2_brows, b1_brows, b2_brows;  // batch stride in rows of each 2-D view
  int64_t m_tiles, n_tiles, total;
  int a1_pre, a2_pre, b1_pre, b2_pre;  // operand has a pre-split lo array (loaded, not converted)
  int tma_store;                       // N = 64, contiguous fp32 rows: epilogue stores by TMA
  int decouple;                        // mbarrier staging hand-off instead of per-tile named barriers
  int b1_mn;      // B segment 1 is N-contiguous (MN-major): loaded as 32 x 32 boxes (32B-atom swizzle)
  int64_t b1_bcol;  // its batch stride in elements along the contiguous (column) dimension
};

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(su32(b)), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}

// K-major, 128-byte swizzle: 8-row groups 1024 B apart (SBO), LBO unused (1), version 1, type 2.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// MN-major tf32 (the only valid MN-major tf32 layout, SWIZZLE_128B_BASE32B = type 1): 128-B rows of
// 32 MN elements per K index, 4-row atoms with the 32-B chunk index XOR (k % 4) (what TMA's
// SWIZZLE_128B_ATOM_32B writes), K groups of 4 rows SBO = 512 B apart, 32-element MN blocks LBO
// apart (tools/micro/umma_mn_test.cu).
__device__ __forceinline__ uint64_t mn32_desc(uint32_t saddr, uint32_t lbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)(512 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)1 << 61);
}
constexpr uint32_t kAMajorMN = 1u << 15;  // instruction descriptor: A is MN-major
constexpr uint32_t kBMajorMN = 1u << 16;  // instruction descriptor: B is MN-major
__host__ __device__ constexpr uint32_t idesc(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(
          d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b)) : "memory");
}
// The tensor core consumes an fp32 operand as tf32 by ignoring its 13 low mantissa bits, so the hi
// part of the 3xTF32 split is the raw operand already in shared memory (no rewrite) and only the lo
// part is written to the second buffer: lo = x - trunc_tf32(x) (exact), itself rounded to tf32 so
// the tensor core's truncation of it loses nothing.
__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
__device__ __forceinline__ float tf32_rnd(float x) { return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u); }
__device__ __forceinline__ float4 split_lo(float4 x) {
  return make_float4(tf32_rnd(x.x - tf32_trunc(x.x)), tf32_rnd(x.y - tf32_trunc(x.y)), tf32_rnd(x.z - tf32_trunc(x.z)),
                     tf32_rnd(x.w - tf32_trunc(x.w)));
}

template <int ACT>
__device__ __forceinline__ float act_c(float x) {
  if constexpr (ACT == ACT_RELU) return x > 0.f ? x : 0.f;
  else if constexpr (ACT == ACT_TANH) return tanhf(x);
  else if constexpr (ACT == ACT_GELU) return gelu_f(x);
  else return x;
}

template <int N, int ACT, bool BR = false>
__global__ void __launch_bounds__(threads<N>(), 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tA1, const __grid_constant__ CUtensorMap tA2,
                    const __grid_constant__ CUtensorMap tB1, const __grid_constant__ CUtensorMap tB2,
                    const __grid_constant__ CUtensorMap tA1l, const __grid_constant__ CUtensorMap tA2l,
                    const __grid_constant__ CUtensorMap tB1l, const __grid_constant__ CUtensorMap tB2l,
                    const __grid_constant__ CUtensorMap tC, const __grid_constant__ Args a) {
  constexpr int S = stages<N, BR>();
  constexpr uint32_t TCOLS = 2 * N;
  extern __shared__ __align__(1024) unsigned char raw[];
  // the 128-B swizzle atoms need 1024-B aligned stages: align the dynamic window explicitly
  const uint32_t pad = (1024u - (su32(raw) & 1023u)) & 1023u;
  auto& s = *reinterpret_cast<Smem<N, BR>*>(raw + pad);
  const GemmArgs& g = a.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nchunks = (g.K + KC - 1) / KC;

  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&s.tmem_base)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      bar_init(&s.full[i], 1);
      bar_init(&s.conv[i], NCONV);
      bar_init(&s.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      bar_init(&s.acc_full[i], 1);
      bar_init(&s.acc_empty[i], nepi<N>());
    }
    bar_init(&s.bres_full, 1);
    for (int i = 0; i < 2; ++i) {
      bar_init(&s.stg_full[i], nepi<N>());
      bar_init(&s.stg_free[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s.tmem_base;

  // tile -> (sample, row block, column block) in 32-bit arithmetic (the tile count is checked on
  // the host; the 64-bit divisions showed up at ~5-9% of the warp samples of these short-K kernels)
  const uint32_t n_t = (uint32_t)a.n_tiles, mn_t = (uint32_t)(a.n_tiles * a.m_tiles);
  auto tile_coords = [&](int64_t tile, int& b, int64_t& m0, int& n0) {
    const uint32_t t = (uint32_t)tile;
    const uint32_t bq = a.div_mn.div(t), rem = t - bq * mn_t;
    const uint32_t mt = a.div_n.div(rem), nt = rem - mt * n_t;
    b = (int)bq;
    m0 = (int64_t)mt * TM;
    n0 = (int)nt * N;
  };

  if (warp == 0) {
    // ---------------- TMA producer (one lane; the rest of the warp waits at the final barrier) --
    if (lane == 0) {
      uint32_t it = 0;
      if constexpr (BR) {  // resident B: hi and lo of every K chunk, once
        bar_expect_tx(&s.bres_full, (uint32_t)(2 * nchunks * N * KC * sizeof(float)));
        for (int c = 0; c < nchunks; ++c) {
          tma_2d(s.bres + c * N * KC, &tB1, c * KC, 0, &s.bres_full);
          tma_2d(s.bres + (BR_CHUNKS + c) * N * KC, &tB1l, c * KC, 0, &s.bres_full);
        }
      }
      for (int64_t tile = blockIdx.x; tile < a.total; tile += gridDim.x) {
        int b, n0;
        int64_t m0;
        tile_coords(tile, b, m0, n0);
        for (int c = 0; c < nchunks; ++c, ++it) {
          const int st = (int)(it % S);
          bar_wait(&s.empty[st], ((it / S) & 1) ^ 1);
          const int k0 = c * KC;
          const bool seg2 = g.ksplit > 0 && k0 >= g.ksplit;
          const int kk = seg2 ? k0 - g.ksplit : k0;
          const bool apre = seg2 ? a.a2_pre : a.a1_pre, bpre = seg2 ? a.b2_pre : a.b1_pre;
          const int bmult = BR ? 0 : (bpre ? 2 : 1);
          bar_expect_tx(&s.full[st], (uint32_t)(((apre ? 2 : 1) * TM + bmult * N) * KC * sizeof(float)));
          const int ar = (int)(b * (seg2 ? a.a2_brows : a.a1_brows) + m0);
          const int br = (int)(b * (seg2 ? a.b2_brows : a.b1_brows) + n0);
          tma_2d(s.st[st].a_hi, seg2 ? &tA2 : &tA1, kk, ar, &s.full[st]);
          if (apre) tma_2d(s.st[st].a_lo, seg2 ? &tA2l : &tA1l, kk, ar, &s.full[st]);
          if constexpr (!BR) {
            if (!seg2 && a.b1_mn) {  // N-contiguous B: boxes of [32 k][32 n] at 4 KB (MN blocks)
              const int col = (int)(b * a.b1_bcol + n0);
#pragma unroll
              for (int h = 0; h < N / 32; ++h) tma_2d(s.st[st].b_hi + h * 32 * KC, &tB1, col + 32 * h, kk, &s.full[st]);
            } else {
              tma_2d(s.st[st].b_hi, seg2 ? &tB2 : &tB1, kk, br, &s.full[st]);
              if (bpre) tma_2d(s.st[st].b_lo, seg2 ? &tB2l : &tB1l, kk, br, &s.full[st]);
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      uint32_t it = 0, tcount = 0;
      constexpr uint32_t id = idesc(N);
      for (int64_t tile = blockIdx.x; tile < a.total; tile += gridDim.x, ++tcount) {
        const uint32_t acc = tcount & 1;
        bar_wait(&s.acc_empty[acc], ((tcount >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + acc * N;
        if (BR && tcount == 0) bar_wait(&s.bres_full, 0);
        for (int c = 0; c < nchunks; ++c, ++it) {
          const int st = (int)(it % S);
          bar_wait(&s.conv[st], (it / S) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t ah = su32(s.st[st].a_hi), al = su32(s.st[st].a_lo);
          const uint32_t bh = BR ? su32(s.bres + c * N * KC) : su32(s.st[st].b_hi);
          const uint32_t bl = BR ? su32(s.bres + (BR_CHUNKS + c) * N * KC) : su32(s.st[st].b_lo);
          const bool bmn = !BR && a.b1_mn && !(g.ksplit > 0 && c * KC >= g.ksplit);
          if (bmn) {  // MN-major B: 8 k = 2 four-row groups = 1024 B per k-step; MN blocks 4 KB apart
#pragma unroll
            for (int ks = 0; ks < KC / 8; ++ks) {
              const uint32_t off = ks * 32, boff = ks * 1024;
              const uint32_t first = (c == 0 && ks == 0) ? 0u : 1u;
              mma(d, sw128_desc(al + off), mn32_desc(bh + boff, 4096), id | kBMajorMN, first);
              mma(d, sw128_desc(ah + off), mn32_desc(bl + boff, 4096), id | kBMajorMN, 1u);
              mma(d, sw128_desc(ah + off), mn32_desc(bh + boff, 4096), id | kBMajorMN, 1u);
            }
          } else {
#pragma unroll
            for (int ks = 0; ks < KC / 8; ++ks) {
              const uint32_t off = ks * 32;  // 8 tf32 = 32 B along K inside the swizzle row
              const uint32_t first = (c == 0 && ks == 0) ? 0u : 1u;
              mma(d, sw128_desc(al + off), sw128_desc(bh + off), id, first);  // small terms first
              mma(d, sw128_desc(ah + off), sw128_desc(bl + off), id, 1u);
              mma(d, sw128_desc(ah + off), sw128_desc(bh + off), id, 1u);
            }
          }
          commit(&s.empty[st]);
        }
        commit(&s.acc_full[acc]);
      }
    }
    __syncwarp();
  } else if (warp >= CONV0 && warp < CONV0 + NCONV) {
    // ---------------- converters: hi = x as loaded, lo = rnd(x - trunc(x)) ----------------
    const int ct = tid - CONV0 * 32;  // 0..32 NCONV - 1
    uint32_t it = 0;
    for (int64_t tile = blockIdx.x; tile < a.total; tile += gridDim.x) {
      for (int c = 0; c < nchunks; ++c, ++it) {
        const int st = (int)(it % S);
        const bool seg2 = g.ksplit > 0 && c * KC >= g.ksplit;
        const bool apre = seg2 ? a.a2_pre : a.a1_pre, bpre = seg2 ? a.b2_pre : a.b1_pre;
        bar_wait(&s.full[st], (it / S) & 1);
        if (!apre) {
          float4* ah = reinterpret_cast<float4*>(s.st[st].a_hi);
          float4* al = reinterpret_cast<float4*>(s.st[st].a_lo);
#pragma unroll
          for (int i = 0; i < TM * KC / 4 / (NCONV * 32); ++i) al[ct + i * NCONV * 32] = split_lo(ah[ct + i * NCONV * 32]);
        }
        if (!BR && !bpre) {
          float4* bh = reinterpret_cast<float4*>(s.st[st].b_hi);
          float4* bl = reinterpret_cast<float4*>(s.st[st].b_lo);
#pragma unroll
          for (int i = 0; i < N * KC / 4 / (NCONV * 32); ++i) bl[ct + i * NCONV * 32] = split_lo(bh[ct + i * NCONV * 32]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
        __syncwarp();
        if (lane == 0) bar_arrive(&s.conv[st]);
      }
    }
  } else if (warp >= EPI0) {
    // ---------------- epilogue ----------------
    constexpr int NEPI = nepi<N>();
    const int e = warp - EPI0;             // 0..NEPI-1
    const int et = tid - EPI0 * 32;        // 0..32 NEPI - 1
    const int q = warp & 3;                // TMEM lane quarter this warp may access
    constexpr int NH = N / (NEPI / 4);     // columns per epilogue warp (32)
    const int cbeg = (e >> 2) * NH;
    uint32_t tcount = 0;
    for (int64_t tile = blockIdx.x; tile < a.total; tile += gridDim.x, ++tcount) {
      const uint32_t acc = tcount & 1;
      int b, n0;
      int64_t m0;
      tile_coords(tile, b, m0, n0);
      // this tile's bias / row-dot weights (epilogue warps only; named barrier 1); with one column
      // tile they are the same for every tile, so each accumulator slot's copy is loaded once
      if (a.n_tiles != 1 || tcount < 2)
      for (int j = et; j < N; j += NEPI * 32) {
        const int gn = n0 + j;
        s.ep_bias[acc][j] = (g.bias && gn < g.N) ? g.bias[gn] : 0.f;
        s.ep_rw[acc][j] = (g.rowdot_w && gn < g.N) ? g.rowdot_w[gn] : 0.f;
        s.ep_ra[acc][j] = (g.r2_a && gn < g.N) ? g.r2_a[gn] : 0.f;
        s.ep_rb[acc][j] = (g.r2_b && gn < g.N) ? g.r2_b[gn] : 0.f;
      }
      // decoupled staging (a.decouple): the warps hand the staged tile to one storing thread by
      // mbarrier instead of two named barriers per tile, so they do not wait for each other
      const bool dec = N == 64 && a.tma_store && a.decouple;
      if (!dec || a.n_tiles != 1 || tcount < 2) {
        if (N == 64 && a.tma_store && et == 0 && !dec)  // the store two tiles back has read this buffer
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        asm volatile("bar.sync 1, %0;" ::"r"(NEPI * 32) : "memory");
      }
      bar_wait(&s.acc_full[acc], (tcount >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (dec && tcount >= 2) bar_wait(&s.stg_free[tcount & 1], ((tcount >> 1) & 1) ^ 1);
      const int64_t gm = m0 + q * 32 + lane;
      const int64_t row = (int64_t)b * g.scb + gm * g.scm;
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + acc * N + cbeg;
      float rpart = 0.f;
      const bool r2 = g.r2_a != nullptr;
      const float rs = (r2 && gm < g.M) ? g.r2_s[(int64_t)b * g.r2_sb + gm] : 0.f;
      const float rx = (r2 && gm < g.M) ? g.r2_x[gm] : 0.f;
#pragma unroll 1
      for (int c0 = 0; c0 < NH; c0 += 16) {
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr + (uint32_t)c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (gm >= g.M) continue;
        const int cc = cbeg + c0;  // column within the tile
        const bool full = n0 + cc + 16 <= g.N;
        float o[16];
        // bias / rank-2 terms read as float4 (16 consecutive columns); branches hoisted out of the
        // element loop
        const float4* bv = reinterpret_cast<const float4*>(&s.ep_bias[acc][cc]);
        if (r2) {
          const float4* av = reinterpret_cast<const float4*>(&s.ep_ra[acc][cc]);
          const float4* cv = reinterpret_cast<const float4*>(&s.ep_rb[acc][cc]);
#pragma unroll
          for (int j4 = 0; j4 < 4; ++j4) {
            const float4 b4 = bv[j4], a4 = av[j4], c4 = cv[j4];
            const float bb[4] = {b4.x, b4.y, b4.z, b4.w}, aa[4] = {a4.x, a4.y, a4.z, a4.w},
                        rr[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int j = 4 * j4 + u;
              const float x = fmaf(g.alpha, __uint_as_float(v[j]), bb[u]);
              o[j] = fmaf(aa[u], rs, fmaf(rr[u], rx, x));
            }
          }
        } else {
#pragma unroll
          for (int j4 = 0; j4 < 4; ++j4) {
            const float4 b4 = bv[j4];
            const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
            for (int u = 0; u < 4; u += 2)  // packed pairs (same rounding as fmaf per element)
              f2_upk(f2_fma(f2_pk(g.alpha, g.alpha), f2_pk(__uint_as_float(v[4 * j4 + u]), __uint_as_float(v[4 * j4 + u + 1])),
                            f2_pk(bb[u], bb[u + 1])),
                     o[4 * j4 + u], o[4 * j4 + u + 1]);
          }
        }
        if constexpr (ACT == ACT_GELU) {
#pragma unroll
          for (int j = 0; j < 16; j += 2) gelu2(o[j], o[j + 1]);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) o[j] = act_c<ACT>(o[j]);
        }
        if (g.rowdot_w) {
          if (full) {
            const float4* wv = reinterpret_cast<const float4*>(&s.ep_rw[acc][cc]);
#pragma unroll
            for (int j4 = 0; j4 < 4; ++j4) {
              const float4 w4 = wv[j4];
              rpart = fmaf(o[4 * j4], w4.x, rpart);
              rpart = fmaf(o[4 * j4 + 1], w4.y, rpart);
              rpart = fmaf(o[4 * j4 + 2], w4.z, rpart);
              rpart = fmaf(o[4 * j4 + 3], w4.w, rpart);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (n0 + cc + j < g.N) rpart = fmaf(o[j], s.ep_rw[acc][cc + j], rpart);
          }
        } else if (N == 64 && a.tma_store) {
          // 128-B swizzled staging: half (cc >> 5), row r, 16-B chunk (c >> 2) ^ (r & 7)
          const int r = q * 32 + lane, hcol = cc & 31;
          float* hbase = s.cst + (tcount & 1) * (TM * N) + (cc >> 5) * (TM * 32) + r * 32;
#pragma unroll
          for (int v4 = 0; v4 < 4; ++v4) {
            const int chunk = ((hcol >> 2) + v4) ^ (r & 7);
            *reinterpret_cast<float4*>(hbase + chunk * 4) =
                make_float4(o[4 * v4], o[4 * v4 + 1], o[4 * v4 + 2], o[4 * v4 + 3]);
          }
        } else if (full && g.scn == 1 && !g.Cd && ((row + n0 + cc) & 3) == 0) {
          float4* dst = reinterpret_cast<float4*>(g.C + row + n0 + cc);
#pragma unroll
          for (int v4 = 0; v4 < 4; ++v4) dst[v4] = make_float4(o[4 * v4], o[4 * v4 + 1], o[4 * v4 + 2], o[4 * v4 + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int gn = n0 + cc + j;
            if (gn >= g.N) continue;
            const int64_t off = row + (int64_t)gn * g.scn;
            if (g.Cd) g.Cd[off] = (double)o[j];
            else g.C[off] = o[j];
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) bar_arrive(&s.acc_empty[acc]);
      if (dec) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) bar_arrive(&s.stg_full[tcount & 1]);
        if (et == 0) {
          bar_wait(&s.stg_full[tcount & 1], (tcount >> 1) & 1);
          const int row0 = (int)(b * g.M + m0);
#pragma unroll
          for (int h = 0; h < 2; ++h)
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                             reinterpret_cast<uint64_t>(&tC)),
                         "r"(n0 + 32 * h), "r"(row0), "r"(su32(s.cst + (tcount & 1) * (TM * N) + h * TM * 32))
                         : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          bar_arrive(&s.stg_free[tcount & 1]);
        }
        __syncwarp();
      } else if (N == 64 && a.tma_store) {  // whole tile staged -> two TMA stores by one thread
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 3, %0;" ::"r"(NEPI * 32) : "memory");
        if (et == 0) {
          const int row0 = (int)(b * g.M + m0);
#pragma unroll
          for (int h = 0; h < 2; ++h)
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                             reinterpret_cast<uint64_t>(&tC)),
                         "r"(n0 + 32 * h), "r"(row0), "r"(su32(s.cst + (tcount & 1) * (TM * N) + h * TM * 32))
                         : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      if (g.rowdot_w) {  // the column groups of a row meet in shared memory (fixed order)
        __shared__ float rsum[3][128];
        const int gi = e >> 2;
        if (gi > 0 && gm < g.M) rsum[gi - 1][q * 32 + lane] = rpart;
        asm volatile("bar.sync 2, %0;" ::"r"(NEPI * 32) : "memory");
        if (gi == 0 && gm < g.M) {
          double tot = (double)rpart;
#pragma unroll
          for (int k = 0; k < NEPI / 4 - 1; ++k) tot += (double)rsum[k][q * 32 + lane];
          g.rowdot_out[row] = tot + (double)g.rowdot_b;
        }
        asm volatile("bar.sync 2, %0;" ::"r"(NEPI * 32) : "memory");
      }
    }
  }
  if (N == 64 && a.tma_store && warp == EPI0 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
}

// ---- host side ------------------------------------------------------------------------------
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeFn) nullptr;
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

// 2-D view [rows][cols] of fp32 with row stride `ld` elements, box [box_rows][32], 128-B swizzle.
bool make_map(CUtensorMap* m, const float* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  EncodeFn enc = encoder();
  if (!enc || !base || rows <= 0 || cols <= 0) return false;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld * 4) & 15)) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  const cuuint32_t box[2] = {(cuuint32_t)KC, (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int N, int ACT, bool BR = false>
cudaError_t launch(const Args& a, const CUtensorMap* maps, cudaStream_t st) {
  const size_t smem = sizeof(Smem<N, BR>) + 1024;  // + alignment slack
  static DeviceOnce once;
  int sms = 1;
  const cudaError_t e = device_once(once, &sms, [&] {
    return cudaFuncSetAttribute(gemm_tc2_kernel<N, ACT, BR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (e != cudaSuccess) return e;
  const int64_t grid = a.total < sms ? a.total : sms;
  gemm_tc2_kernel<N, ACT, BR><<<(unsigned)grid, threads<N>(), smem, st>>>(maps[0], maps[1], maps[2], maps[3], maps[4],
                                                                      maps[5], maps[6], maps[7], maps[8], a);
  return cudaGetLastError();
}


// ---- FNO forward truncated DFT on the tensor core -------------------------------------------
// Vh[b][c][m'] = sum_i V[b][i][c] F[m'][i] for C = 64 channels, 2M = 32 modes. One work unit =
// a sample pair: M = 128 rows (2 samples x 64 channels), N = 32 modes, K = all n cells in blocks
// of 128 (4 chunks of 32). V is channel-contiguous, an MN-major A operand: the TMA lands four
// 32-channel x 32-cell boxes per chunk in the SWIZZLE_128B_ATOM_32B layout, which is exactly the
// MN-major tf32 canonical layout, so the MMA reads them in place as A_hi and the converter warps
// only write the lo parts (3xTF32) into a buffer of the same layout (SNOP_DFT_MN = 1; 0 keeps the
// round-1 transpose into K-major hi / lo: 240 vs 216 us per layer). Each 128-cell block accumulates in TMEM (K = 128, as the other contractions);
// the epilogue adds the blocks' results in registers in block order and writes Vh once.
// Two rings: TMA landing stages (raw boxes + the pre-split F chunk, which the MMA reads in place;
// freed by the MMA commit) and converted K-major hi / lo A slots.
#ifndef SNOP_DFT_LAND
#define SNOP_DFT_LAND 6
#endif
#ifndef SNOP_DFT_CONV
#define SNOP_DFT_CONV 2
#endif
constexpr int DFT_LAND = SNOP_DFT_LAND, DFT_CONV = SNOP_DFT_CONV, DFT_NT = 32;
struct alignas(1024) DftTcLand {
  float a_raw[TM * KC];     // 4 boxes [32 cells][32 channels] (swizzled), as landed by TMA
  float b_hi[DFT_NT * KC];  // F chunk, K-major [32 modes][32 cells] (swizzled), pre-split hi / lo
  float b_lo[DFT_NT * KC];
};
static_assert(offsetof(DftTcLand, b_lo) == offsetof(DftTcLand, b_hi) + DFT_NT * KC * sizeof(float),
              "the N = 64 hi|lo MMA reads b_hi and b_lo as one 64-row K-major operand");
#ifndef SNOP_DFT_MN
#define SNOP_DFT_MN 1  // A (the activations) read MN-major in place; 0: transposed to K-major
#endif
struct alignas(1024) DftTcConv {
#if SNOP_DFT_MN
  float a_lo[TM * KC];  // lo parts of the landed boxes, same MN-major layout
#else
  float a_hi[TM * KC];  // K-major [128 rows][32 cells] (swizzled)
  float a_lo[TM * KC];
#endif
};
struct DftTcSmem {
  DftTcLand land[DFT_LAND];
  DftTcConv cv[DFT_CONV];
  uint64_t full[DFT_LAND], lempty[DFT_LAND], cfull[DFT_CONV], cempty[DFT_CONV];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
};
__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar))
      : "memory");
}
#ifndef SNOP_DFT_NCONV
#define SNOP_DFT_NCONV 8
#endif
constexpr int DFT_NCONV = SNOP_DFT_NCONV;
constexpr int DFT_THREADS = (2 + DFT_NCONV + 4) * 32;  // producer, MMA, converters, 4 epilogue warps

__global__ void __launch_bounds__(DFT_THREADS, 1)
    dft_tc_kernel(const __grid_constant__ CUtensorMap tV, const __grid_constant__ CUtensorMap tF,
                  const __grid_constant__ CUtensorMap tFl, float* __restrict__ Vh, int B, int n, int npairs) {
  extern __shared__ __align__(1024) unsigned char raw[];
  const uint32_t pad = (1024u - (su32(raw) & 1023u)) & 1023u;
  auto& s = *reinterpret_cast<DftTcSmem*>(raw + pad);
  constexpr int SL = DFT_LAND, SC = DFT_CONV;
  constexpr uint32_t TCOLS = 4 * DFT_NT;  // two accumulators x [hi*hi (+ lo*hi) | hi*lo] columns
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nkb = n / 128, nch = nkb * 4;  // K chunks per sample pair
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&s.tmem_base)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < SL; ++i) {
      bar_init(&s.full[i], 1);
      bar_init(&s.lempty[i], 1);  // released by the MMA commit (B is read in place)
    }
    for (int i = 0; i < SC; ++i) {
      bar_init(&s.cfull[i], DFT_NCONV);
      bar_init(&s.cempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      bar_init(&s.acc_full[i], 1);
      bar_init(&s.acc_empty[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s.tmem_base;
  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int sp = blockIdx.x; sp < npairs; sp += gridDim.x) {
        for (int c = 0; c < nch; ++c, ++it) {
          const int sl = (int)(it % SL);
          bar_wait(&s.lempty[sl], ((it / SL) & 1) ^ 1);
          bar_expect_tx(&s.full[sl], (uint32_t)((TM + 2 * DFT_NT) * KC * sizeof(float)));
          const int k0 = c * KC;
#pragma unroll
          for (int q = 0; q < 4; ++q) {  // box q = (sample 2 sp + q / 2, channel half q % 2)
            const int b = min(2 * sp + (q >> 1), B - 1);
            tma_3d(s.land[sl].a_raw + q * 32 * KC, &tV, 32 * (q & 1), k0, b, &s.full[sl]);
          }
          tma_2d(s.land[sl].b_hi, &tF, k0, 0, &s.full[sl]);
          tma_2d(s.land[sl].b_lo, &tFl, k0, 0, &s.full[sl]);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      uint32_t it = 0, tcount = 0;
      constexpr uint32_t id = idesc(DFT_NT), id2 = idesc(2 * DFT_NT);
      for (int sp = blockIdx.x; sp < npairs; sp += gridDim.x) {
        for (int kb = 0; kb < nkb; ++kb, ++tcount) {
          const uint32_t acc = tcount & 1;
          bar_wait(&s.acc_empty[acc], ((tcount >> 1) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t d = tmem + acc * 2 * DFT_NT;
          for (int c = 0; c < 4; ++c, ++it) {
            const int sc = (int)(it % SC), sl = (int)(it % SL);
            bar_wait(&s.cfull[sc], (it / SC) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t bh = su32(s.land[sl].b_hi), bl = su32(s.land[sl].b_lo);
#if SNOP_DFT_MN
            // A_hi = the landed boxes themselves (the tensor core truncates fp32 to tf32), MN-major:
            // 4 boxes = 4 MN blocks of 32 channels, 4 KB apart; a k-step of 8 cells = 1024 B
            const uint32_t ah = su32(s.land[sl].a_raw), al = su32(s.cv[sc].a_lo);
#pragma unroll
            for (int ks = 0; ks < KC / 8; ++ks) {
              const uint32_t off = ks * 32, aoff = ks * 1024;
              const uint32_t first = (c == 0 && ks == 0) ? 0u : 1u;
              mma(d, mn32_desc(ah + aoff, 4096), sw128_desc(bh + off), id2 | kAMajorMN, first);
              mma(d, mn32_desc(al + aoff, 4096), sw128_desc(bh + off), id | kAMajorMN, 1u);
            }
#else
            const uint32_t ah = su32(s.cv[sc].a_hi), al = su32(s.cv[sc].a_lo);
#pragma unroll
            for (int ks = 0; ks < KC / 8; ++ks) {
              const uint32_t off = ks * 32;
              const uint32_t first = (c == 0 && ks == 0) ? 0u : 1u;
              // b_hi / b_lo are adjacent: one N = 64 MMA reads A_hi once for hi*hi and hi*lo
              mma(d, sw128_desc(ah + off), sw128_desc(bh + off), id2, first);
              mma(d, sw128_desc(al + off), sw128_desc(bh + off), id, 1u);
            }
#endif
            commit(&s.cempty[sc]);
            commit(&s.lempty[sl]);
          }
          commit(&s.acc_full[acc]);
        }
      }
    }
    __syncwarp();
  } else if (warp < 2 + DFT_NCONV) {
    // converters: transpose the landed boxes into K-major hi / lo (3xTF32 split), split B
    const int ct = tid - 64;  // 0..32 DFT_NCONV - 1
    uint32_t it = 0;
    for (int sp = blockIdx.x; sp < npairs; sp += gridDim.x) {
      for (int c = 0; c < nch; ++c, ++it) {
        const int sl = (int)(it % SL), sc = (int)(it % SC);
        bar_wait(&s.full[sl], (it / SL) & 1);
        bar_wait(&s.cempty[sc], ((it / SC) & 1) ^ 1);  // the MMAs of chunk it - SC are done
        const float* ar = s.land[sl].a_raw;
#if SNOP_DFT_MN
        {  // lo = rnd_tf32(x - trunc_tf32(x)), element-wise in the landed layout (no transpose)
          const float4* a4 = reinterpret_cast<const float4*>(ar);
          float4* l4 = reinterpret_cast<float4*>(s.cv[sc].a_lo);
#pragma unroll
          for (int i = 0; i < TM * KC / 4 / (DFT_NCONV * 32); ++i) l4[ct + i * DFT_NCONV * 32] = split_lo(a4[ct + i * DFT_NCONV * 32]);
        }
#else
        float* ah = s.cv[sc].a_hi;
        float* al = s.cv[sc].a_lo;
        // task = (box q, 4-cell group kg, 4-channel group jc): four 16-B loads of the landed box,
        // a 4 x 4 register transpose, four 16-B stores each into K-major hi and lo. A 16-B access
        // is served eight lanes at a time and both swizzled layouts put a 16-B chunk's bank group
        // at (chunk index) only, so each 8-lane group takes kg = l and jc = (l ^ 4 (l & 1)) ^ g:
        // the load chunks jc ^ (4 kg + r) and the store chunks kg ^ (4 jc + i) are then both
        // permutations of 0..7 (no bank conflicts on either side of the transpose).
        for (int task = ct; task < 4 * 8 * 8; task += DFT_NCONV * 32) {
          const int l = task & 7, g = (task >> 3) & 7, q = task >> 6;
          const int kg = l, jc = (l ^ ((l & 1) << 2)) ^ g;
          float4 v[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int kk = 4 * kg + r;
            v[r] = *reinterpret_cast<const float4*>(ar + q * 1024 + kk * 32 + ((jc ^ (kk & 7)) << 2));
          }
          const float vv[4][4] = {{v[0].x, v[0].y, v[0].z, v[0].w}, {v[1].x, v[1].y, v[1].z, v[1].w},
                                  {v[2].x, v[2].y, v[2].z, v[2].w}, {v[3].x, v[3].y, v[3].z, v[3].w}};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int m = q * 32 + 4 * jc + i;  // row = (sample q / 2) * 64 + (half q % 2) * 32 + channel
            const int o = (m >> 3) * 256 + (m & 7) * 32 + ((kg ^ (m & 7)) << 2);
            const float4 h = make_float4(vv[0][i], vv[1][i], vv[2][i], vv[3][i]);
            *reinterpret_cast<float4*>(ah + o) = h;
            *reinterpret_cast<float4*>(al + o) = split_lo(h);
          }
        }
#endif
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) bar_arrive(&s.cfull[sc]);
      }
    }
  } else {
    const int q = warp & 3;  // TMEM lane quarter = rows 32 q .. 32 q + 31
    uint32_t tcount = 0;
    for (int sp = blockIdx.x; sp < npairs; sp += gridDim.x) {
      float sum[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) sum[j] = 0.f;
      for (int kb = 0; kb < nkb; ++kb, ++tcount) {
        const uint32_t acc = tcount & 1;
        bar_wait(&s.acc_full[acc], (tcount >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + acc * 2 * DFT_NT;
        uint32_t v[32], w[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
            "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
              "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
              "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
              "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
            "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]), "=r"(w[8]),
              "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15]), "=r"(w[16]),
              "=r"(w[17]), "=r"(w[18]), "=r"(w[19]), "=r"(w[20]), "=r"(w[21]), "=r"(w[22]), "=r"(w[23]), "=r"(w[24]),
              "=r"(w[25]), "=r"(w[26]), "=r"(w[27]), "=r"(w[28]), "=r"(w[29]), "=r"(w[30]), "=r"(w[31])
            : "r"(taddr + DFT_NT));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) bar_arrive(&s.acc_empty[acc]);
#pragma unroll
        for (int j = 0; j < 32; ++j) sum[j] += __uint_as_float(v[j]) + __uint_as_float(w[j]);
      }
      const int r = q * 32 + lane, b = 2 * sp + (r >> 6);
      if (b < B) {  // mode-major Vh[m'][b][c]: a warp's 32 channels are one contiguous 128-B row
#pragma unroll
        for (int j = 0; j < DFT_NT; ++j) Vh[((size_t)j * B + b) * 64 + (r & 63)] = sum[j];
      }
    }
  }
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
}
}  // namespace tc2

// Returns true (and launches) when the contraction fits this engine: K-contiguous operands,
// K <= 128 in whole 32-wide chunks per segment, N <= 128, no batch folding, beta = 0, aligned
// strides. Otherwise false and the caller uses gemm_tc.
bool gemm_tc2(const GemmArgs& g, cudaStream_t st, int64_t mfold, cudaError_t* err) {
  using namespace tc2;
  *err = cudaSuccess;
  // B segment 1 may be N-contiguous (sbn == 1, MN-major): N a multiple of 32, K-chunks whole
  const bool b1mn = g.sbn == 1 && g.sbk != 1 && g.N % 32 == 0 && !g.B_lo;
  if (mfold > 0 || g.beta != 0.f || g.K > 128 || g.N > 128 || g.sak != 1 || (g.sbk != 1 && !b1mn)) return false;
  if (g.ksplit > 0 && (g.ksplit % KC != 0 || g.sak2 != 1 || g.sbk2 != 1)) return false;
  if (g.rowdot_w && g.N > 128) return false;
  const int K1 = g.ksplit > 0 ? g.ksplit : g.K, K2 = g.ksplit > 0 ? g.K - g.ksplit : 0;
  auto brows = [](int64_t sb, int64_t sr, int64_t* out) {
    if (sb == 0) { *out = 0; return true; }
    if (sr <= 0 || sb % sr != 0) return false;
    *out = sb / sr;
    return true;
  };
  Args a{};
  a.g = g;
  if (!brows(g.sab, g.sam, &a.a1_brows) || !brows(g.sbb, g.sbn, &a.b1_brows)) return false;
  if (g.ksplit > 0 && (!brows(g.sab2, g.sam2, &a.a2_brows) || !brows(g.sbb2, g.sbn2, &a.b2_brows))) return false;
  const int NT = g.N <= 64 ? 64 : 128;
  CUtensorMap maps[9];  // A1 A2 B1 B2, their pre-split lo parts (copies of the hi maps when absent), C
  std::memset(maps, 0, sizeof(maps));
  const int64_t rowsA1 = (g.batch - 1) * a.a1_brows + g.M, rowsB1 = (g.batch - 1) * a.b1_brows + g.N;
  a.b1_mn = b1mn ? 1 : 0;
  a.b1_bcol = b1mn ? g.sbb : 0;
  if (!make_map(&maps[0], g.A, rowsA1, K1, g.sam, TM)) return false;
  if (b1mn) {  // [K rows][batch * (column stride)] fp32, 32 x 32 boxes in the 32B-atom swizzle
    EncodeFn enc = encoder();
    const cuuint64_t dims[2] = {(cuuint64_t)((g.batch - 1) * g.sbb + g.N), (cuuint64_t)K1};
    const cuuint64_t strides[1] = {(cuuint64_t)(g.sbk * 4)};
    const cuuint32_t box[2] = {32, (cuuint32_t)KC};
    const cuuint32_t es[2] = {1, 1};
    if (!enc || (reinterpret_cast<uintptr_t>(g.B) & 15) || ((g.sbk * 4) & 15) ||
        enc(&maps[2], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(g.B), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  } else if (!make_map(&maps[2], g.B, rowsB1, K1, g.sbn, NT)) {
    return false;
  }
  a.a1_pre = g.A_lo && make_map(&maps[4], g.A_lo, rowsA1, K1, g.sam, TM);
  a.b1_pre = g.B_lo && make_map(&maps[6], g.B_lo, rowsB1, K1, g.sbn, NT);
  if (g.ksplit > 0) {
    const int64_t rowsA2 = (g.batch - 1) * a.a2_brows + g.M, rowsB2 = (g.batch - 1) * a.b2_brows + g.N;
    if (!make_map(&maps[1], g.A2, rowsA2, K2, g.sam2, TM) || !make_map(&maps[3], g.B2, rowsB2, K2, g.sbn2, NT))
      return false;
    a.a2_pre = g.A2_lo && make_map(&maps[5], g.A2_lo, rowsA2, K2, g.sam2, TM);
    a.b2_pre = g.B2_lo && make_map(&maps[7], g.B2_lo, rowsB2, K2, g.sbn2, NT);
  } else {
    maps[1] = maps[0];
    maps[3] = maps[2];
    maps[5] = maps[4];
    maps[7] = maps[6];
    a.a2_pre = a.a1_pre;
    a.b2_pre = a.b1_pre;
  }
  if (!a.a1_pre) maps[4] = maps[0];
  if (!a.b1_pre) maps[6] = maps[2];
  if (!a.a2_pre) maps[5] = maps[1];
  if (!a.b2_pre) maps[7] = maps[3];
  // TMA-store epilogue: N = 64 fp32 output, unit column stride, whole 128-row tiles per sample and
  // samples contiguous (row b*M + m), no row-dot; C viewed as [batch*M][N] with row stride scm
  a.tma_store = 0;
  maps[8] = maps[0];
  if (NT == 64 && g.N == 64 && g.C && !g.Cd && !g.rowdot_w && g.scn == 1 && g.M % TM == 0 &&
      (g.batch == 1 || g.scb == (int64_t)g.M * g.scm) && SNOP_TC2_CST) {
    EncodeFn enc = encoder();
    const cuuint64_t dims[2] = {(cuuint64_t)g.N, (cuuint64_t)((int64_t)g.batch * g.M)};
    const cuuint64_t strides[1] = {(cuuint64_t)(g.scm * 4)};
    const cuuint32_t box[2] = {32, (cuuint32_t)TM};
    const cuuint32_t es[2] = {1, 1};
    if (enc && !(reinterpret_cast<uintptr_t>(g.C) & 15) && !((g.scm * 4) & 15) &&
        enc(&maps[8], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g.C, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
            CUDA_SUCCESS)
      a.tma_store = 1;
  }
  a.m_tiles = (g.M + TM - 1) / TM;
  a.n_tiles = (g.N + NT - 1) / NT;
  a.total = a.m_tiles * a.n_tiles * g.batch;
  if (a.total == 0) return true;
  if (a.total >= ((int64_t)1 << 31)) return false;  // 32-bit tile arithmetic in the kernel
  // single-K-chunk tiles (the FNO layer-0 inverse with its rank-2 epilogue) are epilogue-bound and
  // gain from the decoupled hand-off (496 -> 456 us); the 3-chunk inverse+W tiles measured 611 vs
  // 620 us with it, so they keep the named barriers
  a.decouple = a.tma_store && g.K <= KC;
  a.div_n.init((uint32_t)a.n_tiles);
  a.div_mn.init((uint32_t)(a.n_tiles * a.m_tiles));
  // resident B (see stages()): N = 128 tile, one column tile, batch-invariant pre-split B, K <= 64
  const bool bres = NT == 128 && a.n_tiles == 1 && g.ksplit == 0 && g.sbb == 0 && a.b1_pre &&
                    (g.K + KC - 1) / KC <= BR_CHUNKS;
  switch (g.act) {
    case ACT_RELU: *err = NT == 64 ? launch<64, ACT_RELU>(a, maps, st) : launch<128, ACT_RELU>(a, maps, st); break;
    case ACT_TANH: *err = NT == 64 ? launch<64, ACT_TANH>(a, maps, st) : launch<128, ACT_TANH>(a, maps, st); break;
    case ACT_GELU:
      *err = NT == 64 ? launch<64, ACT_GELU>(a, maps, st)
                      : (bres ? launch<128, ACT_GELU, true>(a, maps, st) : launch<128, ACT_GELU>(a, maps, st));
      break;
    default: *err = NT == 64 ? launch<64, ACT_NONE>(a, maps, st) : launch<128, ACT_NONE>(a, maps, st); break;
  }
  return true;
}


// FNO forward truncated DFT on the tensor core (dft_tc_kernel): Vh [B][64][32] from V [B][n][64].
// Returns false (nothing launched) when the shape does not fit (C = 64, 2M = 32, n % 128 == 0).
bool fno_dft_tc(const float* V, const float* F, const float* F_lo, float* Vh, int B, int n, cudaStream_t st,
                cudaError_t* err) {
  using namespace tc2;
  *err = cudaSuccess;
  if (n % 128 != 0 || B < 1) return false;
  EncodeFn enc = encoder();
  if (!enc) return false;
  CUtensorMap mv, mf, mfl;
  if (!F_lo) return false;
  const cuuint64_t dv[3] = {64, (cuuint64_t)n, (cuuint64_t)B};
  const cuuint64_t sv[2] = {64 * 4, (cuuint64_t)n * 64 * 4};
  const cuuint32_t bv[3] = {32, 32, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  if (enc(&mv, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(V), dv, sv, bv, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          SNOP_DFT_MN ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  if (!make_map(&mf, F, 32, n, n, 32) || !make_map(&mfl, F_lo, 32, n, n, 32)) return false;
  const int npairs = (B + 1) / 2;
  const size_t smem = sizeof(DftTcSmem) + 1024;
  static DeviceOnce once;
  int sms = 1;
  *err = device_once(once, &sms, [&] {
    return cudaFuncSetAttribute(dft_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (*err != cudaSuccess) return true;
  const int grid = npairs < sms ? npairs : sms;
  dft_tc_kernel<<<grid, DFT_THREADS, smem, st>>>(mv, mf, mfl, Vh, B, n, npairs);
  *err = cudaGetLastError();
  return true;
}
}  // namespace snop_ops
