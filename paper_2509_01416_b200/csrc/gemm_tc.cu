// gemm_tc.cu — tcgen05 (5th-gen tensor core) GEMM for the neural-operator contractions, sm_100a.
//
//   C(b, m, n) = act( alpha * sum_k A(b, m, k) B(b, n, k) + beta * C(b, m, n) + bias[n] )
//
// fp32 operands, fp32-class accuracy through the 3xTF32 split: every operand x = hi + lo with
// hi = x rounded to TF32 and lo = x - hi (exact in fp32), and D = A_hi B_hi + A_hi B_lo + A_lo B_hi
// accumulated in TMEM by tcgen05.mma.kind::tf32 (plain TF32 would miss the 1e-5 operator
// tolerance by two orders of magnitude). One CTA = 128 threads = one 128 x NTILE output tile:
//   * all threads stage a 128 x 32 A chunk and an NTILE x 32 B chunk from global memory (generic
//     strides, so the FNO's per-sample / transposed operands need no copies), split hi/lo and store
//     them in the UMMA no-swizzle K-major core-matrix layout (8 rows x 16 B per core matrix);
//   * one elected thread issues 4 k-steps x 3 tcgen05.mma (M=128, N=NTILE, K=8) per chunk and
//     commits them to the chunk buffer's mbarrier; staging of chunk c+1 overlaps the MMAs of c
//     (double-buffered shared memory);
//   * the epilogue reads the fp32 accumulator with tcgen05.ld (each warp its 32 TMEM lanes) and
//     applies alpha / beta / bias / activation, writing fp32 or fp64.
#include <cstdint>
#include <cstdio>

#include "gemm.cuh"

namespace snop_ops {

namespace tc {

constexpr int TM = 128;  // rows per tile (cta_group::1 M = 128: TMEM lane i = row i)
constexpr int KC = 32;   // K elements per staged chunk (4 MMA k-steps of 8)
constexpr int THREADS = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major, no-swizzle core-matrix layout: element (r, k) of a [rows][KC] fp32 tile.
// Core matrix = 8 rows x 4 fp32 (16 B per row, 128 B contiguous); core matrices adjacent in K
// are LBO = 128 B apart, 8-row groups are SBO = (KC/4) * 128 B apart.
__device__ __forceinline__ int core_off(int r, int k) {
  return ((r >> 3) * (KC / 4) + (k >> 2)) * 32 + (r & 7) * 4 + (k & 3);  // in floats
}
constexpr uint32_t LBO_BYTES = 128;
constexpr uint32_t SBO_BYTES = (KC / 4) * 128;

__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  // base_offset = 0, lbo_mode = 0, layout_type = 0 (SWIZZLE_NONE)
  return d;
}

// Instruction descriptor, kind::tf32: D fp32, A/B TF32, both K-major, M = 128, N = n.
__host__ __device__ constexpr uint32_t make_idesc(int n) {
  return (1u << 4)                           // c_format = F32
         | (2u << 7)                         // a_format = TF32
         | (2u << 10)                        // b_format = TF32
         | ((uint32_t)(n >> 3) << 17)        // N >> 3
         | ((uint32_t)(TM >> 4) << 24);      // M >> 4
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t u = __float_as_uint(x);
  u = (u + 0x1000u) & 0xFFFFE000u;  // round to nearest (ties away) at the TF32 mantissa width
  return __uint_as_float(u);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// Shared-memory chunk buffers: the non-split kernels use ONE stage (48 KB at N = 64 -> four
// CTAs per SM; the register prefetch of the next chunk still overlaps the MMAs), the split
// (long-K) kernels keep two stages (their register sums leave room for two CTAs per SM only).
template <bool SPLIT>
constexpr int stages() { return SPLIT ? 2 : 1; }

template <int N, int STAGES>
struct Smem {
  float a_hi[STAGES][TM * KC];
  float a_lo[STAGES][TM * KC];
  float b_hi[STAGES][N * KC];
  float b_lo[STAGES][N * KC];
  uint64_t bar[2];     // chunk buffers: MMAs reading the buffer have completed
  uint64_t accbar[2];  // split mode: all MMAs of the chunk accumulating into TMEM slot s are done
  uint32_t tmem_base;
  float ep_bias[N];    // this tile's bias[n0 .. n0 + N) (0 beyond N / without bias)
  float ep_rw[N];      // this tile's row-dot weights (fused FNO projection)
};

// Long-K contractions (K > SPLIT_K: DeepONet branch K = 2000, FNO forward DFT K = 1024) use split
// accumulation: every KC = 32-wide chunk accumulates in one of two TMEM accumulators, which is
// drained into fp32 registers while the tensor core works on the next chunk. This bounds the
// accumulation length inside the tensor core (its fp32 accumulation rounding grows with K), and
// these chunks also add the lo*lo product (4xTF32), so long-K results match fp32 FFMA accuracy.
constexpr int DR = 1;
constexpr int SPLIT_K = 4 * KC;

// One operand's staging for a chunk: ROWS x KC fp32 = ROWS * KC / 4 float4 groups; thread tid
// handles groups tid + i * THREADS, group -> (row = g % ROWS, kq = g / ROWS): consecutive lanes
// take consecutive rows, so the float4 stores into the core-matrix layout are bank-conflict free
// (8 lanes fill one 128 B core matrix) and MN-contiguous operands load coalesced. Because
// THREADS is a multiple of ROWS, every group of a thread lies in the same row (row = tid % ROWS):
// the row's base pointers are resolved once per tile (RowPtr) and a chunk only adds k offsets.
template <int ROWS>
struct Stage {
  static constexpr int G = ROWS * KC / 4 / THREADS;
  float4 v[G];
};

struct RowPtr {
  const float* p1;  // row base in the first K segment (nullptr: row out of range)
  const float* p2;  // row base in the second K segment (ksplit > 0)
  int64_t sk1, sk2;
};

template <int ROWS, bool IS_A>
__device__ __forceinline__ RowPtr row_ptr(const GemmArgs& g, int b, int64_t row0, int64_t mfold, int tid) {
  RowPtr rp;
  const int64_t gr = row0 + (tid % ROWS);
  const int64_t nrows = IS_A ? (int64_t)g.M : (int64_t)g.N;
  if (gr >= nrows) {
    rp.p1 = rp.p2 = nullptr;
    rp.sk1 = rp.sk2 = 0;
    return rp;
  }
  if (IS_A) {
    int64_t r1, r2;
    if (mfold > 0) {
      const int64_t q = gr / mfold, r = gr - q * mfold;
      r1 = q * g.sab + r * g.sam;
      r2 = q * g.sab2 + r * g.sam2;
    } else {
      r1 = (int64_t)b * g.sab + gr * g.sam;
      r2 = (int64_t)b * g.sab2 + gr * g.sam2;
    }
    rp.p1 = g.A + r1;
    rp.p2 = g.ksplit > 0 ? g.A2 + r2 : nullptr;
    rp.sk1 = g.sak;
    rp.sk2 = g.sak2;
  } else {
    rp.p1 = g.B + (int64_t)b * g.sbb + gr * g.sbn;
    rp.p2 = g.ksplit > 0 ? g.B2 + (int64_t)b * g.sbb2 + gr * g.sbn2 : nullptr;
    rp.sk1 = g.sbk;
    rp.sk2 = g.sbk2;
  }
  return rp;
}

template <int ROWS>
__device__ __forceinline__ void load_chunk(Stage<ROWS>& st, const GemmArgs& g, const RowPtr& rp, int k0, int tid) {
  const bool seg2 = g.ksplit > 0 && k0 >= g.ksplit;  // ksplit is a multiple of KC: whole chunk
  const float* base = seg2 ? rp.p2 : rp.p1;
  const int64_t sk = seg2 ? rp.sk2 : rp.sk1;
  const int kofs = seg2 ? k0 - g.ksplit : k0;
  const bool vec = base && sk == 1 && k0 + KC <= g.K &&
                   ((reinterpret_cast<uintptr_t>(base + kofs) & 15) == 0);
#pragma unroll
  for (int i = 0; i < Stage<ROWS>::G; ++i) {
    const int kq = (tid + i * THREADS) / ROWS;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (vec) {
      v = __ldg(reinterpret_cast<const float4*>(base + kofs + kq * 4));
    } else if (base) {
      const int kg = k0 + kq * 4;
      const float* p = base + (int64_t)(kofs + kq * 4) * sk;
      if (k0 + KC <= g.K) {  // interior chunk: no per-element bounds checks
        v.x = __ldg(p);
        v.y = __ldg(p + sk);
        v.z = __ldg(p + 2 * sk);
        v.w = __ldg(p + 3 * sk);
      } else {
        if (kg < g.K) v.x = __ldg(p);
        if (kg + 1 < g.K) v.y = __ldg(p + sk);
        if (kg + 2 < g.K) v.z = __ldg(p + 2 * sk);
        if (kg + 3 < g.K) v.w = __ldg(p + 3 * sk);
      }
    }
    st.v[i] = v;
  }
}

template <int ROWS>
__device__ __forceinline__ void store_chunk(const Stage<ROWS>& st, float* hi, float* lo, int tid) {
#pragma unroll
  for (int i = 0; i < Stage<ROWS>::G; ++i) {
    const int grp = tid + i * THREADS;
    const int r = grp % ROWS, kq = grp / ROWS;
    const float4 v = st.v[i];
    const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
    const float4 l = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
    const int o = core_off(r, kq * 4);
    *reinterpret_cast<float4*>(hi + o) = h;
    *reinterpret_cast<float4*>(lo + o) = l;
  }
}

template <int N, bool SPLIT>
__global__ void __launch_bounds__(THREADS, (N <= 64 ? (SPLIT ? 2 : 4) : 1))
    gemm_tc_kernel(const GemmArgs g, int64_t mfold, int64_t m_tiles, int64_t n_tiles, int64_t n_total) {
  constexpr int STAGES = stages<SPLIT>();
  extern __shared__ __align__(1024) unsigned char raw[];
  auto& s = *reinterpret_cast<Smem<N, STAGES>*>(raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr uint32_t NACC = SPLIT ? 2 : 1;
  constexpr uint32_t TCOLS = (N * NACC) <= 32 ? 32 : (N * NACC) <= 64 ? 64 : (N * NACC) <= 128 ? 128 : 256;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s.tmem_base)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&s.bar[0], 1);
    mbar_init(&s.bar[1], 1);
    mbar_init(&s.accbar[0], 1);
    mbar_init(&s.accbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s.tmem_base;
  const uint32_t tlane = tmem + ((uint32_t)(warp * 32) << 16);  // this warp's TMEM lanes

  const int nchunks = (g.K + KC - 1) / KC;
  uint32_t phase[2] = {0u, 0u}, aphase[2] = {0u, 0u};
  int64_t cg = 0;  // chunk counter across the tiles of this persistent CTA (buffer parity)
  constexpr uint32_t idesc = make_idesc(N);
  float sum[SPLIT ? N : 1];
  auto drain = [&](int slot) {
    mbar_wait(&s.accbar[slot], aphase[slot]);
    aphase[slot] ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(tlane + (uint32_t)(slot * N + c0)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if constexpr (SPLIT) {
#pragma unroll
        for (int j = 0; j < 16; ++j) sum[c0 + j] += __uint_as_float(v[j]);
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  };

  Stage<TM> sa;
  Stage<N> sb;
  // persistent loop over output tiles (n fastest, then m, then batch)
  for (int64_t tile = blockIdx.x; tile < n_total; tile += gridDim.x) {
    const int nt = (int)(tile % n_tiles);
    const int64_t mt = (tile / n_tiles) % m_tiles;
    const int b = (int)(tile / (n_tiles * m_tiles));
    const int64_t m0 = mt * TM;
    const int n0 = nt * N;
    if constexpr (SPLIT) {
#pragma unroll
      for (int j = 0; j < N; ++j) sum[j] = 0.f;
    }
    const RowPtr ra = row_ptr<TM, true>(g, b, m0, mfold, tid);
    const RowPtr rb = row_ptr<N, false>(g, b, n0, 0, tid);
    for (int j = tid; j < N; j += THREADS) {  // visible to the epilogue through the chunk barriers
      const int gn = n0 + j;
      s.ep_bias[j] = (g.bias && gn < g.N) ? g.bias[gn] : 0.f;
      s.ep_rw[j] = (g.rowdot_w && gn < g.N) ? g.rowdot_w[gn] : 0.f;
    }
    load_chunk<TM>(sa, g, ra, 0, tid);
    load_chunk<N>(sb, g, rb, 0, tid);
    int last_buf = 0;
    for (int c = 0; c < nchunks; ++c, ++cg) {
      const int buf = (int)(cg % STAGES);
      if (cg >= STAGES) {  // buffer reuse: wait for the MMAs issued on it STAGES chunks ago
        mbar_wait(&s.bar[buf], phase[buf]);
        phase[buf] ^= 1u;
      }
      store_chunk<TM>(sa, s.a_hi[buf], s.a_lo[buf], tid);
      store_chunk<N>(sb, s.b_hi[buf], s.b_lo[buf], tid);
      if (c + 1 < nchunks) {  // prefetch the next chunk: global latency overlaps this chunk's MMAs
        load_chunk<TM>(sa, g, ra, (c + 1) * KC, tid);
        load_chunk<N>(sb, g, rb, (c + 1) * KC, tid);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> async proxy
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int slot = SPLIT ? (c & 1) : 0;
      if (tid == 0) {
        const uint32_t ah = smem_u32(s.a_hi[buf]), al = smem_u32(s.a_lo[buf]);
        const uint32_t bh = smem_u32(s.b_hi[buf]), bl = smem_u32(s.b_lo[buf]);
        const uint32_t td = tmem + (uint32_t)(slot * N);
#pragma unroll
        for (int ks = 0; ks < KC / 8; ++ks) {
          const uint32_t off = ks * 2 * 128;  // two core matrices along K per k-step
          const uint64_t dah = make_sdesc(ah + off, LBO_BYTES, SBO_BYTES);
          const uint64_t dal = make_sdesc(al + off, LBO_BYTES, SBO_BYTES);
          const uint64_t dbh = make_sdesc(bh + off, LBO_BYTES, SBO_BYTES);
          const uint64_t dbl = make_sdesc(bl + off, LBO_BYTES, SBO_BYTES);
          const uint32_t first = (SPLIT ? ks == 0 : (c == 0 && ks == 0)) ? 0u : 1u;
          if (SPLIT) mma_tf32(td, dal, dbl, idesc, first);  // 4xTF32 on the long-K path
          mma_tf32(td, dal, dbh, idesc, SPLIT ? 1u : first);  // small terms first
          mma_tf32(td, dah, dbl, idesc, 1u);
          mma_tf32(td, dah, dbh, idesc, 1u);
        }
        mma_commit(&s.bar[buf]);
        if (SPLIT) mma_commit(&s.accbar[slot]);
      }
      __syncwarp();
      if constexpr (SPLIT) {
        if (c > 0) drain((c - 1) & 1);
      }
      last_buf = buf;
    }
    if constexpr (SPLIT) {
      drain((nchunks - 1) & 1);
    } else {
      // the tile's last commit covers all its MMAs; consume that completion so the buffer
      // parity bookkeeping stays exact across tiles
      mbar_wait(&s.bar[last_buf], phase[last_buf]);
      phase[last_buf] ^= 1u;
      // the other buffer's last commit (if any this tile) completed before; consume it too
      if (STAGES == 2 && nchunks >= 2) {
        const int ob = last_buf ^ 1;
        mbar_wait(&s.bar[ob], phase[ob]);
        phase[ob] ^= 1u;
      }
      cg = 0;  // both buffers drained: restart parity at the next tile
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    if constexpr (SPLIT) {
      // drain() consumed the accumulator barriers; the chunk-buffer barriers still hold up to two
      // pending completions — consume them before reusing the buffers on the next tile
      const int lb = (int)((cg - 1) % STAGES);
      mbar_wait(&s.bar[lb], phase[lb]);
      phase[lb] ^= 1u;
      if (STAGES == 2 && nchunks >= 2) {
        mbar_wait(&s.bar[lb ^ 1], phase[lb ^ 1]);
        phase[lb ^ 1] ^= 1u;
      }
      cg = 0;
    }

    // epilogue: warp w owns TMEM lanes (rows) 32w..32w+31
    const int64_t gm = m0 + warp * 32 + lane;
    const int64_t row = mfold > 0 ? (gm / mfold) * g.scb + (gm % mfold) * g.scm : (int64_t)b * g.scb + gm * g.scm;
    double rdot = 0.0;
#pragma unroll
    for (int c0 = 0; c0 < N; c0 += 16) {
      float x16[16];
      if constexpr (SPLIT) {
#pragma unroll
        for (int j = 0; j < 16; ++j) x16[j] = sum[c0 + j];
      } else {
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(tlane + (uint32_t)c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) x16[j] = __uint_as_float(v[j]);
      }
      if (gm < g.M) {
        const bool full = (n0 + c0 + 16 <= g.N);
        if (g.rowdot_w) {
          float part = 0.f;  // 16 products in fp32, then one fp64 accumulate per 16 columns
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (!full && n0 + c0 + j >= g.N) continue;
            const float x = fmaf(g.alpha, x16[j], s.ep_bias[c0 + j]);
            part = fmaf(act_f(x, g.act), s.ep_rw[c0 + j], part);
          }
          rdot += (double)part;
        } else if (full && g.scn == 1 && !g.Cd && ((row + n0 + c0) & 3) == 0 &&
                   ((reinterpret_cast<uintptr_t>(g.C) & 15) == 0)) {
          // vectorised path: 16 contiguous fp32 of this row -> 4 x 16 B
          float4* dst = reinterpret_cast<float4*>(g.C + row + n0 + c0);
#pragma unroll
          for (int v4 = 0; v4 < 4; ++v4) {
            float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
            if (g.beta != 0.f) o = dst[v4];
            float* op = reinterpret_cast<float*>(&o);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int j = v4 * 4 + e;
              float x = g.alpha * x16[j] + (g.beta != 0.f ? g.beta * op[e] : 0.f);
              x += s.ep_bias[c0 + j];
              op[e] = act_f(x, g.act);
            }
            dst[v4] = o;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int gn = n0 + c0 + j;
            if (gn >= g.N) continue;
            const int64_t off = row + (int64_t)gn * g.scn;
            float x = g.alpha * x16[j];
            if (g.beta != 0.f) x += g.beta * g.C[off];
            x += s.ep_bias[c0 + j];
            x = act_f(x, g.act);
            if (g.Cd) g.Cd[off] = (double)x;
            else g.C[off] = x;
          }
        }
      }
    }
    if (g.rowdot_w && gm < g.M) {
      // N split over at most two 64-wide tiles: two addends onto a zeroed output commute exactly
      // in IEEE arithmetic (0 + a + b == 0 + b + a), so the atomic accumulation is deterministic
      const double part = rdot + (nt == 0 ? (double)g.rowdot_b : 0.0);
      if (n_tiles == 1) g.rowdot_out[row] = part;
      else atomicAdd(&g.rowdot_out[row], part);
    }
    // all warps finished reading TMEM before the next tile's first MMA overwrites it
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
}

template <int N, bool SPLIT>
cudaError_t launch(const GemmArgs& g, int64_t mfold, cudaStream_t st) {
  const size_t smem = sizeof(Smem<N, stages<SPLIT>()>);
  static DeviceOnce once;
  int sms = 1;
  const cudaError_t e = device_once(once, &sms, [&] {
    return cudaFuncSetAttribute(gemm_tc_kernel<N, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (e != cudaSuccess) return e;
  const int64_t m_tiles = (g.M + TM - 1) / TM;
  const int64_t n_tiles = (g.N + N - 1) / N;
  const int64_t total = m_tiles * n_tiles * (mfold > 0 ? 1 : g.batch);
  const int per_sm = N <= 64 ? (SPLIT ? 2 : 4) : 1;
  const int64_t grid = total < (int64_t)sms * per_sm ? total : (int64_t)sms * per_sm;
  gemm_tc_kernel<N, SPLIT><<<(unsigned)grid, THREADS, smem, st>>>(g, mfold, m_tiles, n_tiles, total);
  return cudaGetLastError();
}

}  // namespace tc

// Tensor-core GEMM. mfold > 0 folds the batch into M: row r of the GEMM is row (r % mfold) of
// batch (r / mfold), i.e. A row offset (r / mfold) * sab + (r % mfold) * sam, C row offset
// (r / mfold) * scb + (r % mfold) * scm (used for the FNO forward DFT over B x C rows).
cudaError_t gemm_tc(const GemmArgs& g, cudaStream_t st, int64_t mfold) {
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return cudaSuccess;
  if (g.r2_a) return cudaErrorInvalidValue;  // rank-2 epilogue: TMA engine only
  if (g.ksplit > 0 && g.ksplit % tc::KC != 0) return cudaErrorInvalidValue;  // segment = whole chunks
  const bool split = g.K > tc::SPLIT_K;  // long K: chunk-wise drained accumulation
  if (g.rowdot_w) {  // row-dot epilogue: N <= 128 as one or two 64-wide tiles (caller zeroes out)
    if (g.N > 128 || split) return cudaErrorInvalidValue;
    return tc::launch<64, false>(g, mfold, st);
  }
  if (g.N <= 32) return split ? tc::launch<32, true>(g, mfold, st) : tc::launch<32, false>(g, mfold, st);
  return split ? tc::launch<64, true>(g, mfold, st) : tc::launch<64, false>(g, mfold, st);
}

}  // namespace snop_ops

// Test hook (C linkage, not part of the public C-ABI): runs one GEMM on device pointers with both
// engines so tests can pin the tensor-core path against the FFMA path.
extern "C" int snop_internal_gemm_test(int engine, int M, int N, int K, int batch, const float* A, long long sam,
                                       long long sak, long long sab, const float* B, long long sbn, long long sbk,
                                       long long sbb, float* C, long long scm, long long scn, long long scb,
                                       const float* bias, float alpha, float beta, int act, long long mfold) {
  snop_ops::GemmArgs g{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.batch = batch;
  g.A = A;
  g.sam = sam;
  g.sak = sak;
  g.sab = sab;
  g.B = B;
  g.sbn = sbn;
  g.sbk = sbk;
  g.sbb = sbb;
  g.C = C;
  g.scm = scm;
  g.scn = scn;
  g.scb = scb;
  g.bias = bias;
  g.alpha = alpha;
  g.beta = beta;
  g.act = act;
  g.ksplit = 0;
  cudaError_t e = cudaSuccess;
  if (engine == 2) {  // TMA-fed warp-specialised engine; -1 when the shape does not fit it
    if (!snop_ops::gemm_tc2(g, 0, mfold, &e)) return -1;
  } else {
    e = engine == 1 ? snop_ops::gemm_tc(g, 0, mfold) : snop_ops::gemm_f32(g, 0);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return (int)e;
}
