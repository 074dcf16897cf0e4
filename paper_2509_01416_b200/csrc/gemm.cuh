// gemm.cuh — strided, batched fp32 GEMM used by the neural-operator forwards:
//   C(b, m, n) = act( alpha * sum_k A(b, m, k) B(b, n, k) + beta * C(b, m, n) + bias[n] )
// with arbitrary element strides for every operand (so the FNO's per-sample DFT, inverse DFT
// and channel mixing need no transposes). fp32 FFMA accumulation (exact-fp32 class numerics).
// The tcgen05 engine (gemm_tc.cu) replaces this for the large contractions; this kernel stays
// the fallback for tiny/odd shapes and the cross-check in tests.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <mutex>

namespace snop_ops {

// One-time per-device launch setup (kernel attributes) and the device's SM count, thread-safe: a
// second context on another device in the same process gets its own entry.
constexpr int kMaxDevices = 64;
struct DeviceOnce {
  std::once_flag flag[kMaxDevices];
  cudaError_t err[kMaxDevices] = {};
  int sms[kMaxDevices] = {};
};
template <class F>
inline cudaError_t device_once(DeviceOnce& d, int* sms, F&& setup) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  std::call_once(d.flag[dev], [&] {
    d.err[dev] = setup();
    if (cudaDeviceGetAttribute(&d.sms[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) d.sms[dev] = 1;
  });
  *sms = d.sms[dev] > 0 ? d.sms[dev] : 1;
  return d.err[dev];
}

enum Act : int { ACT_RELU = 0, ACT_TANH = 1, ACT_GELU = 2, ACT_NONE = 3 };

// GELU(x) = x Phi(x) = 0.5 x (1 + erf(x / sqrt 2)) (exact-erf form). Default: erfc
// from A&S 7.1.28 (SNOP_GELU_AS28, one MUFU, below). Alternative (SNOP_GELU_AS28 = 0): erf from
// Abramowitz & Stegun 7.1.26: erf(z) = 1 - t (a1 + a2 t + ... + a5 t^4) exp(-z^2), t = 1/(1 + p z),
// |error| <= 1.5e-7 (<= 5e-7 absolute on GELU in fp32 arithmetic). The reciprocal and the
// exponential are the raw flush-to-zero MUFU ops (rcp.approx.ftz, ex2.approx.ftz: __fdividef /
// __expf add denormal-range fix-ups, 6 + 9 instructions at the source line in ncu; a flushed
// exp(-z^2) < 2^-126 changes nothing at fp32), and the sign is folded algebraically (below), so
// no copysign or |.|: ~13 instructions, 2 MUFU, |error| <= 3.4e-7 absolute on GELU (fp32, swept
// over [-12, 12]). The epilogues of the FNO GEMMs evaluate it ~1.6e9 times per C5 forward
// (the projection is issue-bound on it).
__device__ __forceinline__ float rcp_ftz(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_ftz(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// A&S coefficients a_i / sqrt 2, negated (so the last step is a plain fma; -(a b) = (-a) b exactly)
#define SNOP_GELU_C0 (-7.505269764e-01f)
#define SNOP_GELU_C1 (1.027533652e+00f)
#define SNOP_GELU_C2 (-1.005091295e+00f)
#define SNOP_GELU_C3 (2.011695713e-01f)
#define SNOP_GELU_C4 (-1.801917326e-01f)
#ifndef SNOP_GELU_AS28
#define SNOP_GELU_AS28 1
#endif
#if SNOP_GELU_AS28
// A&S 7.1.28: erf(y) = 1 - (1 + a1 y + ... + a6 y^6)^-16, |error| <= 3e-7; with y = |x|/sqrt 2 the
// factors 1/sqrt 2^i are folded into the coefficients, so erfc(|x|/sqrt 2) = r^16 with
// r = 1 / poly(|x|): ONE MUFU (the reciprocal) per GELU instead of two (reciprocal and exp2) -
// the epilogues of the FNO GEMMs are bound by the MUFU rate (16 per SM per clock). |error| <=
// 7.5e-7 absolute on GELU in fp32 (swept over [-12, 12], 1-ulp reciprocal included).
#define SNOP_GELU_B1 (4.986734697e-02f)
#define SNOP_GELU_B2 (2.114100615e-02f)
#define SNOP_GELU_B3 (3.277626324e-03f)
#define SNOP_GELU_B4 (3.800357500e-05f)
#define SNOP_GELU_B5 (4.889063564e-05f)
#define SNOP_GELU_B6 (5.382975000e-06f)
__device__ __forceinline__ float gelu_f(float x) {
  // GELU = max(x, 0) - (|x| / 2) erfc(|x| / sqrt 2)
  const float y = fabsf(x);
  const float p = fmaf(fmaf(fmaf(fmaf(fmaf(fmaf(SNOP_GELU_B6, y, SNOP_GELU_B5), y, SNOP_GELU_B4), y, SNOP_GELU_B3), y,
                                SNOP_GELU_B2), y, SNOP_GELU_B1), y, 1.0f);
  float r = rcp_ftz(p);
  r *= r;
  r *= r;
  r *= r;
  r *= r;
  return fmaf(-0.5f * y, r, fmaxf(x, 0.0f));
}
#else
__device__ __forceinline__ float gelu_f(float x) {
  // GELU = x/2 + |x|/2 erf(z) = max(x, 0) - (|x|/2) t P(t) e^{-z^2}, z = |x|/sqrt 2, and
  // |x|/2 = z / sqrt 2: the factor 1/sqrt 2 is folded into the A&S coefficients (a_i / sqrt 2).
  const float z = fabsf(x) * 0.70710678118654752440f;
  const float t = rcp_ftz(fmaf(0.3275911f, z, 1.0f));
  const float p = fmaf(fmaf(fmaf(fmaf(SNOP_GELU_C0, t, SNOP_GELU_C1), t, SNOP_GELU_C2), t, SNOP_GELU_C3), t, SNOP_GELU_C4) * t;
  const float e = ex2_ftz((z * z) * -1.44269504088896340736f);  // exp(-z^2)
  return fmaf(z, p * e, fmaxf(x, 0.0f));
}

#endif

// Two GELUs with packed FP32 (fma.rn.f32x2 / mul.rn.f32x2 -> FFMA2 / FMUL2): the same operations
// in the same order per element as gelu_f (bit-identical results) in ~9 instead of ~13 issue slots
// per element; the FNO projection epilogue is issue-bound on GELU.
__device__ __forceinline__ unsigned long long f2_pk(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_upk(unsigned long long r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ unsigned long long f2_fma(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
#if SNOP_GELU_AS28
__device__ __forceinline__ void gelu2(float& xa, float& xb) {
  const unsigned long long y = f2_pk(fabsf(xa), fabsf(xb));
  unsigned long long p = f2_fma(f2_pk(SNOP_GELU_B6, SNOP_GELU_B6), y, f2_pk(SNOP_GELU_B5, SNOP_GELU_B5));
  p = f2_fma(p, y, f2_pk(SNOP_GELU_B4, SNOP_GELU_B4));
  p = f2_fma(p, y, f2_pk(SNOP_GELU_B3, SNOP_GELU_B3));
  p = f2_fma(p, y, f2_pk(SNOP_GELU_B2, SNOP_GELU_B2));
  p = f2_fma(p, y, f2_pk(SNOP_GELU_B1, SNOP_GELU_B1));
  p = f2_fma(p, y, f2_pk(1.0f, 1.0f));
  float pa, pb;
  f2_upk(p, pa, pb);
  unsigned long long r = f2_pk(rcp_ftz(pa), rcp_ftz(pb));
  r = f2_mul(r, r);
  r = f2_mul(r, r);
  r = f2_mul(r, r);
  r = f2_mul(r, r);
  f2_upk(f2_fma(f2_mul(y, f2_pk(-0.5f, -0.5f)), r, f2_pk(fmaxf(xa, 0.0f), fmaxf(xb, 0.0f))), xa, xb);
}
#else
__device__ __forceinline__ void gelu2(float& xa, float& xb) {
  const unsigned long long z = f2_mul(f2_pk(fabsf(xa), fabsf(xb)), f2_pk(0.70710678118654752440f, 0.70710678118654752440f));
  float da, db;
  f2_upk(f2_fma(f2_pk(0.3275911f, 0.3275911f), z, f2_pk(1.0f, 1.0f)), da, db);
  const unsigned long long t = f2_pk(rcp_ftz(da), rcp_ftz(db));
  unsigned long long p = f2_fma(f2_pk(SNOP_GELU_C0, SNOP_GELU_C0), t, f2_pk(SNOP_GELU_C1, SNOP_GELU_C1));
  p = f2_fma(p, t, f2_pk(SNOP_GELU_C2, SNOP_GELU_C2));
  p = f2_fma(p, t, f2_pk(SNOP_GELU_C3, SNOP_GELU_C3));
  p = f2_fma(p, t, f2_pk(SNOP_GELU_C4, SNOP_GELU_C4));
  p = f2_mul(p, t);
  float ga, gb;
  f2_upk(f2_mul(f2_mul(z, z), f2_pk(-1.44269504088896340736f, -1.44269504088896340736f)), ga, gb);
  const unsigned long long e = f2_pk(ex2_ftz(ga), ex2_ftz(gb));
  f2_upk(f2_fma(z, f2_mul(p, e), f2_pk(fmaxf(xa, 0.0f), fmaxf(xb, 0.0f))), xa, xb);
}

#endif

__device__ __forceinline__ float act_f(float x, int act) {
  switch (act) {
    case ACT_RELU: return x > 0.f ? x : 0.f;
    case ACT_TANH: return tanhf(x);
    case ACT_GELU: return gelu_f(x);
    default: return x;
  }
}

struct GemmArgs {
  int M, N, K, batch;
  const float* A;
  int64_t sam, sak, sab;
  const float* B;
  int64_t sbn, sbk, sbb;
  float* C;          // fp32 output (or nullptr when Cd is used)
  double* Cd;        // optional fp64 output (same strides)
  int64_t scm, scn, scb;
  const float* bias; // [N] or nullptr
  float alpha, beta; // beta applies to the existing fp32 C
  int act;
  // optional second K segment: for k >= ksplit, A/B elements come from A2/B2 at k - ksplit
  // (fuses e.g. the FNO inverse DFT [G | V] x [U | W]^T into one contraction). ksplit = 0: none.
  int ksplit;
  const float* A2;
  int64_t sam2, sak2, sab2;
  const float* B2;
  int64_t sbn2, sbk2, sbb2;
  // optional row-dot epilogue (tensor-core engine; requires N <= 128): instead of storing C,
  // rowdot_out[row] = sum_n act(alpha*acc + bias[n]) * rowdot_w[n] + rowdot_b  (fp64 output),
  // row = b * scb + m * scm. Fuses the FNO projection 64 -> hidden -> 1.
  const float* rowdot_w;
  float rowdot_b;
  double* rowdot_out;
  // optional rank-2 epilogue term (TMA engine only): + r2_a[n] * r2_s[b * r2_sb + m] + r2_b[n] * r2_x[m]
  // (the FNO's affine lift folded through layer 0's W path)
  const float* r2_a;
  const float* r2_b;
  const float* r2_s;
  int64_t r2_sb;
  const float* r2_x;
  // optional pre-split lo parts of constant operands (TMA engine only): lo = rnd_tf32(x - trunc_tf32(x))
  // with the same layout/strides as A / B / A2 / B2; the engine then loads lo instead of splitting
  const float* A_lo;
  const float* B_lo;
  const float* A2_lo;
  const float* B2_lo;
};

// host-side 3xTF32 lo part of a constant operand (matches the engine's in-kernel split)
inline float tf32_lo_host(float x) {
  uint32_t u;
  __builtin_memcpy(&u, &x, 4);
  uint32_t t = u & 0xFFFFE000u;
  float h;
  __builtin_memcpy(&h, &t, 4);
  float d = x - h;
  __builtin_memcpy(&u, &d, 4);
  u = (u + 0x1000u) & 0xFFFFE000u;
  __builtin_memcpy(&d, &u, 4);
  return d;
}

__device__ __forceinline__ float gemm_a(const GemmArgs& a, int b, int64_t m, int k) {
  if (a.ksplit > 0 && k >= a.ksplit)
    return a.A2[(int64_t)b * a.sab2 + m * a.sam2 + (int64_t)(k - a.ksplit) * a.sak2];
  return a.A[(int64_t)b * a.sab + m * a.sam + (int64_t)k * a.sak];
}
__device__ __forceinline__ float gemm_b(const GemmArgs& a, int b, int64_t n, int k) {
  if (a.ksplit > 0 && k >= a.ksplit)
    return a.B2[(int64_t)b * a.sbb2 + n * a.sbn2 + (int64_t)(k - a.ksplit) * a.sbk2];
  return a.B[(int64_t)b * a.sbb + n * a.sbn + (int64_t)k * a.sbk];
}

constexpr int GBM = 64, GBN = 64, GBK = 16, GTHREADS = 256;

static __global__ void __launch_bounds__(GTHREADS) gemm_f32_kernel(const GemmArgs a) {
  __shared__ float As[GBK][GBM + 4];
  __shared__ float Bs[GBK][GBN + 4];
  const int b = blockIdx.z;
  const int m0 = blockIdx.x * GBM, n0 = blockIdx.y * GBN;  // M on x (2^31 limit)
  const int tid = threadIdx.x;
  const int tm = (tid / 16) * 4, tn = (tid % 16) * 4;
  float acc[4][4] = {};
  const bool a_kfast = a.sak == 1, b_kfast = a.sbk == 1;
  for (int k0 = 0; k0 < a.K; k0 += GBK) {
#pragma unroll
    for (int r = 0; r < (GBM * GBK) / GTHREADS; ++r) {
      const int e = tid + r * GTHREADS;
      const int mm = a_kfast ? e / GBK : e % GBM, kk = a_kfast ? e % GBK : e / GBM;
      const int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < a.M && gk < a.K) ? gemm_a(a, b, gm, gk) : 0.f;
      const int nn = b_kfast ? e / GBK : e % GBN, kb = b_kfast ? e % GBK : e / GBN;
      const int gn = n0 + nn, gkb = k0 + kb;
      Bs[kb][nn] = (gn < a.N && gkb < a.K) ? gemm_b(a, b, gn, gkb) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GBK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][tm + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tn + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + tm + i;
    if (gm >= a.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tn + j;
      if (gn >= a.N) continue;
      const int64_t off = (int64_t)b * a.scb + (int64_t)gm * a.scm + (int64_t)gn * a.scn;
      float v = a.alpha * acc[i][j];
      if (a.beta != 0.f) v += a.beta * a.C[off];
      if (a.bias) v += a.bias[gn];
      v = act_f(v, a.act);
      if (a.Cd) a.Cd[off] = (double)v;
      else a.C[off] = v;
    }
  }
}

// Tensor-core (tcgen05, 3xTF32) engine, gemm_tc.cu. mfold > 0 folds the batch into M.
cudaError_t gemm_tc(const GemmArgs& g, cudaStream_t st, int64_t mfold = 0);
// Warp-specialised TMA-fed engine (gemm_tc2.cu) for K-contiguous operands with K <= 128: returns
// false when the contraction does not fit it (the caller then uses gemm_tc).
bool gemm_tc2(const GemmArgs& g, cudaStream_t st, int64_t mfold, cudaError_t* err);
// FNO forward truncated DFT on the tensor core (C = 64, 2M = 32, n % 128 == 0): V [B][n][64] ->
// Vh MODE-MAJOR [32][B][64] (the layout fno_mix64<true> stages with coalesced rows).
bool fno_dft_tc(const float* V, const float* F, const float* F_lo, float* Vh, int B, int n, cudaStream_t st,
                cudaError_t* err);

static inline cudaError_t gemm_f32(const GemmArgs& a, cudaStream_t s) {
  if (a.M <= 0 || a.N <= 0 || a.batch <= 0) return cudaSuccess;
  dim3 grid((a.M + GBM - 1) / GBM, (a.N + GBN - 1) / GBN, a.batch);
  gemm_f32_kernel<<<grid, GTHREADS, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace snop_ops
