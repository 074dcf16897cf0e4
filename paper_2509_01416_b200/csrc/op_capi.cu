// op_capi.cu — SolutionOperators on the device and the MD-PNOP drivers
// built on them: recast_fixed_point and precondition_fixed_source
// (SPEC.md:413-421). Every dense contraction (DeepONet branch/trunk/combine, FNO truncated DFT,
// inverse DFT + W path, projection) goes through one GEMM entry point (gemm.cuh / the tcgen05
// engine); the elementwise parts (lift, spectral mixing, recast, row projection, fixed-point
// bookkeeping) are small fused kernels here. Neural operators compute in fp32; the API is fp64.
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#define SNOP_PHASE_SYM g_phase_cycles_op
#include "gemm.cuh"
#include "model_io.h"
#include "snop_internal.h"

using namespace snop_impl;
using namespace snop_ops;

struct snop_op {
  int kind = 0;  // 0 DeepONet, 1 FNO, 2 exact model-based solve at p*
  snop_ctx* ctx = nullptr;
  snop_grid grid{};
  double tstar = 1.0, sstar = 0.5;
  int act = ACT_TANH;
  // DeepONet
  std::vector<int> bsizes, tsizes;
  std::vector<float*> bW, bb;  // device, per branch layer
  float* trunk_out = nullptr;  // [Nc][p] trunk evaluated at the cell centres (once)
  float* bias0_vec = nullptr;  // [Nc] filled with bias0 (or nullptr)
  bool has_bias0 = false;
  float bias0 = 0.f;
  std::vector<float> host_params;  // as created (save_model); DeepONet: branch then trunk
  // FNO
  int width = 64, modes = 16, layers = 4, hidden = 128;
  float *lift_W = nullptr, *lift_b = nullptr, *xc = nullptr;
  std::vector<float*> Rr, Ri, W, b;
  float *P1W = nullptr, *P1b = nullptr, *P2W = nullptr, *P2b = nullptr;
  float p2b_host = 0.f;
  // layer 0 folded through the affine lift: U0 = S^ (x) P + Q, W-path rank-2 terms
  float *l0_P = nullptr, *l0_Q = nullptr;         // [2][M][C] (re, im)
  float *l0_A = nullptr, *l0_B = nullptr, *l0_C = nullptr;  // [C]
  float *F = nullptr, *Ginv = nullptr;  // forward [2M][n] and inverse [n][2M] truncated DFT
  float* FT = nullptr;                  // forward DFT transposed, [n][2M] (fno_dft64)
  // pre-split 3xTF32 lo parts of the constant GEMM operands (TMA engine loads them, no conversion)
  float *Ginv_lo = nullptr, *P1W_lo = nullptr, *F_lo = nullptr;
  // spectral mixing as tensor-core GEMMs (per layer): the per-mode real forms of R, K-major,
  // [4][M][C][C] = {Rr^T, -Ri^T (U_re), Ri^T, Rr^T (U_im)} with [o][c] rows, and their lo parts
  std::vector<float*> mixB, mixB_lo;
  // exact operator
  int order = 16;
  snop_solver_config cfg{};
  double *cst = nullptr, *css = nullptr;
  size_t cst_n = 0;
  // identity of this operator for cached device-loop graphs: a process-unique serial, and a
  // generation bumped when its own device buffers are reallocated
  uint64_t serial = next_serial();
  uint64_t gen = 0;
  static uint64_t next_serial() {
    static std::atomic<uint64_t> n{1};
    return n++;
  }
  std::vector<void*> owned;
  ~snop_op() {
    for (void* p : owned) cudaFree(p);
    if (cst) cudaFree(cst);
    if (css) cudaFree(css);
  }
  float* upload_lo(const float* h, size_t n) {
    std::vector<float> lo(n);
    for (size_t i = 0; i < n; ++i) lo[i] = tf32_lo_host(h[i]);
    return upload(lo.data(), n);
  }
  template <class T>
  T* upload(const T* h, size_t n) {
    T* d = nullptr;
    if (cudaMalloc(&d, n * sizeof(T)) != cudaSuccess) return nullptr;
    owned.push_back(d);
    if (h && cudaMemcpy(d, h, n * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
    return d;
  }
};

namespace {

#define SNOP_TRY(expr)             \
  do {                             \
    const snop_status _s = (expr); \
    if (_s != SNOP_OK) return _s;  \
  } while (0)

snop_status invalid(const std::string& m) {
  set_error(m);
  return SNOP_INVALID_ARGUMENT;
}
snop_status cuda_status(const char* what, cudaError_t e) {
  if (e == cudaSuccess) return SNOP_OK;
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return SNOP_CUDA_ERROR;
}

// ---- small fused kernels -------------------------------------------------------------------
__global__ void cast_f64_to_f32(size_t n, const double* __restrict__ in, float* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = (float)in[i];
}

__global__ void fill_f64(size_t n, double v, double* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = v;
}

// FNO lift: v[b][i][c] = Wl[c][0] S[b][i] + Wl[c][1] x_i + bl[c]
__global__ void fno_lift(int B, int n, int C, const double* __restrict__ S, const float* __restrict__ xc,
                         const float* __restrict__ Wl, const float* __restrict__ bl, float* __restrict__ V) {
  const size_t total = (size_t)B * n * C;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % C);
    const size_t row = e / C;
    const int i = (int)(row % n);
    const float s = (float)S[row];
    V[e] = fmaf(Wl[2 * c], s, fmaf(Wl[2 * c + 1], xc[i], bl[c]));
  }
}

// FNO spectral mixing: U[b][o][m] + i U[b][o][M+m] =
//   sum_c (Rr[m][c][o] + i Ri[m][c][o]) (Vh[b][c][m] + i Vh[b][c][M+m]).
// Real form per mode: [Ur | Ui] = [Vr | Vi] . [[Rr, Ri], [-Ri, Rr]], a (samples x 2C) x (2C x 2C)
// product. Block = (mode m, MIX_S samples): the 2C x 2C mode matrix and the samples' (transposed)
// spectra are staged in shared memory, each thread accumulates a 4-sample x 8-output register tile
// (three 16-byte shared loads per 32 FFMA). C = 64 (the FNO width) is the tuned shape; other widths
// use the generic loop below.
constexpr int MIX_S = 64;
// MM: Vh is mode-major [2M][B][C] (written so by the tensor-core forward DFT): the staging loads
// are then contiguous channel rows (consecutive threads -> consecutive channels) instead of one
// float per 128-B [b][c][2M] row, and Vt gets a padded pitch for the transposed stores.
template <bool MM>
__global__ void __launch_bounds__(256) fno_mix64(int B, int M, const float* __restrict__ Vh,
                                                 const float* __restrict__ Rr, const float* __restrict__ Ri,
                                                 float* __restrict__ U) {
  constexpr int C = 64, C2 = 128, VP = MM ? MIX_S + 4 : MIX_S;
  extern __shared__ __align__(16) float smx[];
  float* Mx = smx;             // [2C][2C]
  float* Vt = smx + C2 * C2;   // [2C][VP]: Vt[k][s]
  const int m = blockIdx.y, b0 = blockIdx.x * MIX_S, t = threadIdx.x;
  const float* rr = Rr + (size_t)m * C * C;
  const float* ri = Ri + (size_t)m * C * C;
  // all global loads of the staging issued before any shared-memory store (independent requests
  // in flight instead of one L2 round trip per loop trip)
  constexpr int NR = C * C / 256, NV = MIX_S * C / 256;
  float ra[NR], rb[NR], va[NV], vb[NV];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    ra[r] = rr[t + 256 * r];
    rb[r] = ri[t + 256 * r];
  }
#pragma unroll
  for (int r = 0; r < NV; ++r) {
    if constexpr (MM) {  // consecutive threads -> consecutive channels (coalesced rows)
      const int e = t + 256 * r, c = e & (C - 1), b = b0 + (e >> 6);
      const size_t bb = (size_t)(b < B ? b : B - 1);
      va[r] = Vh[((size_t)m * B + bb) * C + c];
      vb[r] = Vh[((size_t)(M + m) * B + bb) * C + c];
    } else {  // consecutive threads -> consecutive samples (conflict-free stores)
      const int e = t + 256 * r, c = e / MIX_S, b = b0 + (e - c * MIX_S);
      const float* v = Vh + ((size_t)(b < B ? b : B - 1) * C + c) * 2 * M;
      va[r] = v[m];
      vb[r] = v[M + m];
    }
  }
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int e = t + 256 * r, c = e / C, o = e - c * C;
    Mx[c * C2 + o] = ra[r];
    Mx[c * C2 + C + o] = rb[r];
    Mx[(C + c) * C2 + o] = -rb[r];
    Mx[(C + c) * C2 + C + o] = ra[r];
  }
#pragma unroll
  for (int r = 0; r < NV; ++r) {
    const int e = t + 256 * r;
    const int c = MM ? (e & (C - 1)) : e / MIX_S, sidx = MM ? (e >> 6) : e - c * MIX_S;
    Vt[c * VP + sidx] = va[r];
    Vt[(C + c) * VP + sidx] = vb[r];
  }
  __syncthreads();
  const int sg = t & 15, og = t >> 4;  // samples 4 sg .. 4 sg + 3, outputs 8 og .. 8 og + 7
  float acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
#pragma unroll 4
  for (int k = 0; k < C2; ++k) {
    const float4 v = *reinterpret_cast<const float4*>(Vt + k * VP + 4 * sg);
    const float4 w0 = *reinterpret_cast<const float4*>(Mx + k * C2 + 8 * og);
    const float4 w1 = *reinterpret_cast<const float4*>(Mx + k * C2 + 8 * og + 4);
    const float vv[4] = {v.x, v.y, v.z, v.w};
    const float ww[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(vv[i], ww[j], acc[i][j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int b = b0 + 4 * sg + i;
    if (b >= B) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int q = 8 * og + j;  // 0..63: Ur[o = q]; 64..127: Ui[o = q - 64]
      const int o = q & (C - 1);
      U[((size_t)b * C + o) * 2 * M + (q < C ? m : M + m)] = acc[i][j];
    }
  }
}

__global__ void fno_mix(int B, int C, int M, const float* __restrict__ Vh, const float* __restrict__ Rr,
                        const float* __restrict__ Ri, float* __restrict__ U) {
  extern __shared__ float sR[];  // [2][C][C]
  const int m = blockIdx.y;
  for (int e = threadIdx.x; e < C * C; e += blockDim.x) {
    sR[e] = Rr[(size_t)m * C * C + e];
    sR[C * C + e] = Ri[(size_t)m * C * C + e];
  }
  __syncthreads();
  const int o = threadIdx.x % C, sub = threadIdx.x / C, per = blockDim.x / C;
  for (int b = blockIdx.x * per + sub; b < B; b += gridDim.x * per) {
    const float* vh = Vh + (size_t)b * C * 2 * M;
    float re = 0.f, im = 0.f;
    for (int c = 0; c < C; ++c) {
      const float vr = vh[c * 2 * M + m], vi = vh[c * 2 * M + M + m];
      const float a = sR[c * C + o], bb = sR[C * C + c * C + o];
      re = fmaf(a, vr, fmaf(-bb, vi, re));
      im = fmaf(a, vi, fmaf(bb, vr, im));
    }
    U[(size_t)b * C * 2 * M + (size_t)o * 2 * M + m] = re;
    U[(size_t)b * C * 2 * M + (size_t)o * 2 * M + M + m] = im;
  }
}

// Forward truncated DFT of the FNO activations in exact fp32 (C = 64 channels, 2M = 32 rows):
//   Vh[b][c][m'] = sum_i V[b][i][c] FT[i][m'].
// Block = 8 warps = 8 samples; lane l of warp w accumulates an 8-channel x 8-mode block (channel
// block l & 7, mode block l >> 3) over all cells, in cell order. Rows stream through a 3-stage
// shared-memory ring fed by cp.async.bulk (one contiguous 4 KB copy per sample and 2 KB of FT per
// 16-row chunk) with mbarrier transaction counts; operands are read as broadcast float4 (8 distinct
// addresses per warp), so the loop is FFMA-bound: 64 FFMA per 4 LDS.128 (ncu: FMA pipe 64%, issue
// 72%; 420 us per C5 layer against 487 us for the 3xTF32 tensor-core GEMM with per-thread staging).
#ifndef SNOP_DFT_ROWS
#define SNOP_DFT_ROWS 16
#define SNOP_DFT_ST 3
#endif
constexpr int DFT_ROWS = SNOP_DFT_ROWS, DFT_ST = SNOP_DFT_ST, DFT_S = 8;
struct DftStage {
  float v[DFT_S][DFT_ROWS * 64];
  float ft[DFT_ROWS * 32];
};
__device__ __forceinline__ uint32_t sa32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__global__ void __launch_bounds__(32 * DFT_S) fno_dft64(int B, int n, const float* __restrict__ V,
                                                 const float* __restrict__ FT, float* __restrict__ Vh) {
  extern __shared__ __align__(128) unsigned char dft_raw[];
  DftStage* st = reinterpret_cast<DftStage*>(dft_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(dft_raw + DFT_ST * sizeof(DftStage));
  uint64_t* empty = full + DFT_ST;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b0 = blockIdx.x * DFT_S;
  const int nchunks = n / DFT_ROWS;
  constexpr uint32_t kBytes = DFT_S * DFT_ROWS * 64 * 4 + DFT_ROWS * 32 * 4;
  if (threadIdx.x == 0) {
    for (int s = 0; s < DFT_ST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa32(&empty[s])), "r"(DFT_S));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int c) {
    const int s = c % DFT_ST;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa32(&full[s])), "r"(kBytes)
                 : "memory");
    for (int q = 0; q < DFT_S; ++q) {
      const int b = min(b0 + q, B - 1);
      const float* src = V + ((size_t)b * n + (size_t)c * DFT_ROWS) * 64;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              sa32(st[s].v[q])),
          "l"(src), "r"(DFT_ROWS * 64 * 4), "r"(sa32(&full[s]))
          : "memory");
    }
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            sa32(st[s].ft)),
        "l"(FT + (size_t)c * DFT_ROWS * 32), "r"(DFT_ROWS * 32 * 4), "r"(sa32(&full[s]))
        : "memory");
  };
  auto wait = [&](uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(sa32(bar)), "r"(parity)
          : "memory");
  };
  if (threadIdx.x == 0)
    for (int c = 0; c < DFT_ST && c < nchunks; ++c) issue(c);
  const int cb = lane & 7, mb = lane >> 3;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  for (int c = 0; c < nchunks; ++c) {
    const int s = c % DFT_ST;
    wait(&full[s], (uint32_t)((c / DFT_ST) & 1));
    const float* v = st[s].v[w] + cb * 8;
    const float* f = st[s].ft + mb * 8;
#pragma unroll 4
    for (int r = 0; r < DFT_ROWS; ++r) {
      const float4 v0 = *reinterpret_cast<const float4*>(v + r * 64);
      const float4 v1 = *reinterpret_cast<const float4*>(v + r * 64 + 4);
      const float4 f0 = *reinterpret_cast<const float4*>(f + r * 32);
      const float4 f1 = *reinterpret_cast<const float4*>(f + r * 32 + 4);
      const float vv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
      const float ff[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(vv[i], ff[j], acc[i][j]);
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa32(&empty[s])) : "memory");
    if (threadIdx.x == 0 && c + DFT_ST < nchunks) {
      wait(&empty[s], (uint32_t)((c / DFT_ST) & 1));
      issue(c + DFT_ST);
    }
  }
  const int b = b0 + w;
  if (b < B) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float4* dst = reinterpret_cast<float4*>(Vh + ((size_t)b * 64 + cb * 8 + i) * 32 + mb * 8);
      dst[0] = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
      dst[1] = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    }
  }
}

// Layer-0 spectral mixing from the source spectrum (affine-lift folding): U[b][o][m] + i U[b][o][M+m]
// = (Sh[b][m] + i Sh[b][M+m]) (P[m][o] + i P[M+m][o]) + Q[m][o] + i Q[M+m][o].
// MN: U written mode-major U'[m'][b][o] (consecutive threads -> consecutive channels: coalesced)
// for the inverse GEMM's MN-major B operand; otherwise [b][o][m'].
template <bool MN>
__global__ void fno_mix_l0(int B, int C, int M, const float* __restrict__ Sh, const float* __restrict__ P,
                           const float* __restrict__ Q, float* __restrict__ U) {
  const size_t total = (size_t)B * C * M;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    int m, o;
    size_t b;
    if constexpr (MN) {  // e = (m * B + b) * C + o
      o = (int)(e % C);
      const size_t mb = e / C;
      b = mb % B;
      m = (int)(mb / B);
    } else {
      m = (int)(e % M);
      const size_t bo = e / M;
      o = (int)(bo % C);
      b = bo / C;
    }
    const float sr = Sh[b * 2 * M + m], si = Sh[b * 2 * M + M + m];
    const float pr = P[(size_t)m * C + o], pi = P[(size_t)(M + m) * C + o];
    const float ur = fmaf(sr, pr, fmaf(-si, pi, Q[(size_t)m * C + o]));
    const float ui = fmaf(sr, pi, fmaf(si, pr, Q[(size_t)(M + m) * C + o]));
    if constexpr (MN) {
      U[((size_t)m * B + b) * C + o] = ur;
      U[((size_t)(M + m) * B + b) * C + o] = ui;
    } else {
      U[(b * C + o) * 2 * M + m] = ur;
      U[(b * C + o) * 2 * M + M + m] = ui;
    }
  }
}

// Projection second stage: out[r] = sum_k h[r][k] P2[k] + b2 (fp64 output). One warp per row.
__global__ void rowdot(size_t rows, int H, const float* __restrict__ h, const float* __restrict__ P2,
                       const float* __restrict__ b2, double* __restrict__ out) {
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) / 32;
  for (size_t r = warp; r < rows; r += nwarps) {
    float s = 0.f;
    for (int k = lane; k < H; k += 32) s = fmaf(h[r * H + k], P2[k], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[r] = (double)(s + b2[0]);
  }
}

// recast fixed-point bookkeeping, one CTA per instance: relative change,
// divergence guard (non-finite or > 1e6 x initial max-norm -> restore phi0), freeze when done.
__global__ void recast_update(int n, int norm, double tol, const int* __restrict__ it_done, const double* __restrict__ nx,
                              double* __restrict__ phi, const double* __restrict__ phi0,
                              const double* __restrict__ norm0, uint8_t* __restrict__ active,
                              int32_t* __restrict__ iters, int32_t* __restrict__ status, int* __restrict__ n_active) {
  const int b = blockIdx.x;
  if (!active[b]) return;
  const int it = *it_done + 1;
  const double* x = nx + (size_t)b * n;
  double* p = phi + (size_t)b * n;
  double num = 0.0, den = 0.0, mx = 0.0;
  int finite = 1;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = x[i], d = v - p[i];
    finite &= isfinite(v) ? 1 : 0;
    mx = fmax(mx, fabs(v));
    if (norm == 0) {
      num = fmax(num, fabs(d));
      den = fmax(den, fabs(v));
    } else {
      num = fma(d, d, num);
      den = fma(v, v, den);
    }
  }
  __shared__ double sh[3][32];
  __shared__ int shf[32];
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    finite &= __shfl_xor_sync(0xffffffffu, finite, o);
    if (norm == 0) {
      num = fmax(num, __shfl_xor_sync(0xffffffffu, num, o));
      den = fmax(den, __shfl_xor_sync(0xffffffffu, den, o));
    } else {
      num += __shfl_xor_sync(0xffffffffu, num, o);
      den += __shfl_xor_sync(0xffffffffu, den, o);
    }
  }
  const int w = threadIdx.x / 32, nw = blockDim.x / 32;
  if ((threadIdx.x & 31) == 0) {
    sh[0][w] = num;
    sh[1][w] = den;
    sh[2][w] = mx;
    shf[w] = finite;
  }
  __syncthreads();
  num = sh[0][0];
  den = sh[1][0];
  mx = sh[2][0];
  finite = shf[0];
  for (int u = 1; u < nw; ++u) {
    if (norm == 0) {
      num = fmax(num, sh[0][u]);
      den = fmax(den, sh[1][u]);
    } else {
      num += sh[0][u];
      den += sh[1][u];
    }
    mx = fmax(mx, sh[2][u]);
    finite &= shf[u];
  }
  __syncthreads();
  const double n0 = norm0[b];
  const bool diverged = !finite || (n0 > 0.0 && mx > 1e6 * n0);
  double rel;
  if (norm == 1) {
    num = sqrt(num);
    den = sqrt(den);
  }
  rel = den > 0.0 ? num / den : (num > 0.0 ? INFINITY : 0.0);
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = diverged ? phi0[(size_t)b * n + i] : x[i];
  if (threadIdx.x == 0) {
    iters[b] = it;
    if (diverged) {
      status[b] = SNOP_RECAST_DIVERGED;
      active[b] = 0;
    } else if (rel < tol) {
      status[b] = SNOP_RECAST_CONVERGED;
      active[b] = 0;
    } else {
      atomicAdd(n_active, 1);
    }
  }
}

// Loop control of a device-looped iteration (WHILE conditional graph node): counts the iteration
// and continues while any instance is active and the cap is not reached.
__global__ void loop_ctl(cudaGraphConditionalHandle h, int* __restrict__ it_done, const int* __restrict__ n_active,
                         int max_it, int n_body, unsigned long long* __restrict__ launches) {
  const int it = *it_done + 1;
  *it_done = it;
  *launches += (unsigned long long)n_body;  // this pass's kernels (loop bodies run one at a time)
  cudaGraphSetConditional(h, (*n_active > 0 && it < max_it) ? 1u : 0u);
}

__global__ void loop_arm(cudaGraphConditionalHandle h) { cudaGraphSetConditional(h, 1u); }

__global__ void fill_i32(int n, int32_t v, int32_t* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = v;
}

__global__ void maxabs_rows(int n, const double* __restrict__ x, double* __restrict__ out) {
  const int b = blockIdx.x;
  double mx = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) mx = fmax(mx, fabs(x[(size_t)b * n + i]));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  __shared__ double sh[32];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x / 32] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = sh[0];
    for (int u = 1; u < (int)(blockDim.x / 32); ++u) r = fmax(r, sh[u]);
    out[b] = r;
  }
}

unsigned grid_for(const Ctx& c, size_t n, int threads = 256) {
  size_t blocks = (n + threads - 1) / threads;
  const size_t cap = (size_t)c.sm_count * 16;
  if (blocks > cap) blocks = cap;
  return (unsigned)(blocks ? blocks : 1);
}

// Dense contractions run on the tcgen05 3xTF32 engines (gemm_tc2.cu, gemm_tc.cu);
// ctx.opt.gemm_engine = 2 selects the FFMA engine (cross-check only), 1 the tcgen05 engine v1 only.
bool use_tc(const Ctx& ctx) { return ctx.opt.gemm_engine != 2; }

snop_status gemm(Ctx& ctx, const GemmArgs& a, int64_t mfold = 0) {
  ctx.launches++;
  if (use_tc(ctx)) {
    cudaError_t e = cudaSuccess;
    if (ctx.opt.gemm_engine == 0 && gemm_tc2(a, ctx.stream, mfold, &e)) return cuda_status("gemm_tc2", e);
    return cuda_status("gemm_tc", gemm_tc(a, ctx.stream, mfold));
  }
  if (mfold > 0) return invalid("batch-folded GEMM requires the tensor-core engine");
  return cuda_status("gemm", gemm_f32(a, ctx.stream));
}

GemmArgs rowmajor(int M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C, int ldc,
                  const float* bias, int act) {
  GemmArgs g{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.batch = 1;
  g.A = A;
  g.sam = lda;
  g.sak = 1;
  g.B = B;
  g.sbn = ldb;
  g.sbk = 1;
  g.C = C;
  g.scm = ldc;
  g.scn = 1;
  g.bias = bias;
  g.alpha = 1.f;
  g.beta = 0.f;
  g.act = act;
  return g;
}

// DenseNetwork forward over `rows` inputs: hidden layers activated, output linear.
snop_status dense_forward(Ctx& ctx, int rows, const std::vector<int>& sizes, const std::vector<float*>& W,
                          const std::vector<float*>& bvec, int act, const float* in, float* buf0, float* buf1,
                          float** out) {
  const float* cur = in;
  float* bufs[2] = {buf0, buf1};
  const int L = (int)sizes.size() - 1;
  for (int l = 0; l < L; ++l) {
    float* dst = bufs[l & 1];
    SNOP_TRY(gemm(ctx, rowmajor(rows, sizes[l + 1], sizes[l], cur, sizes[l], W[l], sizes[l], dst, sizes[l + 1],
                                bvec[l], l + 1 < L ? act : ACT_NONE)));
    cur = dst;
  }
  *out = const_cast<float*>(cur);
  return SNOP_OK;
}

// predict: in/out fp64 device arrays [B][Nc].
snop_status op_predict_dev(Ctx& ctx, snop_op& op, int B, const double* in, double* out,
                           const uint8_t* active = nullptr) {
  const int n = op.grid.n_cells;
  const size_t rowsN = (size_t)B * n;
  if (op.kind == 2) {  // exact operator: model-based solve at p*
    if (op.cst_n < rowsN) {
      if (op.cst) cudaFree(op.cst);
      if (op.css) cudaFree(op.css);
      op.cst = op.css = nullptr;
      ++op.gen;
      if (cudaMalloc(&op.cst, rowsN * sizeof(double)) != cudaSuccess ||
          cudaMalloc(&op.css, rowsN * sizeof(double)) != cudaSuccess)
        return cuda_status("cudaMalloc exact-op materials", cudaErrorMemoryAllocation);
      op.cst_n = rowsN;
    }
    // filled on every call: a device loop may capture this call into a graph that is discarded
    // and captured again, so a fill done only on allocation could be lost
    fill_f64<<<grid_for(ctx, rowsN), 256, 0, ctx.stream>>>(rowsN, op.tstar, op.cst);
    fill_f64<<<grid_for(ctx, rowsN), 256, 0, ctx.stream>>>(rowsN, op.sstar, op.css);
    ctx.launches += 2;
    int32_t* it = static_cast<int32_t*>(ctx.slot(40, (size_t)B * sizeof(int32_t)));
    uint8_t* cv = static_cast<uint8_t*>(ctx.slot(41, (size_t)B));
    // (active: a device loop's frozen instances are skipped; the neural operators run whole batches)
    return launch_source_iteration(ctx, op.grid, op.order, B, op.cst, op.css, nullptr, in, op.cfg, nullptr, out,
                                   nullptr, it, cv, nullptr, nullptr, active);
  }
  float* X = static_cast<float*>(ctx.slot(42, rowsN * sizeof(float)));
  if (!X) return cuda_status("workspace", cudaErrorMemoryAllocation);
  if (op.kind == 0) {
    cast_f64_to_f32<<<grid_for(ctx, rowsN), 256, 0, ctx.stream>>>(rowsN, in, X);
    ctx.launches++;
    int maxw = 0;
    for (int s : op.bsizes) maxw = std::max(maxw, s);
    float* b0 = static_cast<float*>(ctx.slot(43, (size_t)B * maxw * sizeof(float)));
    float* b1 = static_cast<float*>(ctx.slot(44, (size_t)B * maxw * sizeof(float)));
    float* br = nullptr;
    SNOP_TRY(dense_forward(ctx, B, op.bsizes, op.bW, op.bb, op.act, X, b0, b1, &br));
    const int p = op.bsizes.back();
    GemmArgs g = rowmajor(B, n, p, br, p, op.trunk_out, p, nullptr, n, op.bias0_vec, ACT_NONE);
    g.Cd = out;
    return gemm(ctx, g);
  }
  // FNO
  const int C = op.width, M = op.modes, H = op.hidden;
  const size_t vsz = rowsN * C;
  float* V = static_cast<float*>(ctx.slot(45, vsz * sizeof(float)));
  float* Vn = static_cast<float*>(ctx.slot(46, vsz * sizeof(float)));
  float* Vh = static_cast<float*>(ctx.slot(47, (size_t)B * C * 2 * M * sizeof(float)));
  float* U = static_cast<float*>(ctx.slot(48, (size_t)B * C * 2 * M * sizeof(float)));
  if (!V || !Vn || !Vh || !U) return cuda_status("FNO workspace", cudaErrorMemoryAllocation);
  const bool tc_fused = use_tc(ctx) && (2 * M) % 32 == 0;
  // layer 0 without materialising the lifted field (TMA engine with the rank-2 epilogue)
  const bool l0 = tc_fused && op.layers >= 1 && op.l0_P && 2 * M <= 128 && C <= 128 && ctx.opt.gemm_engine == 0;
  if (l0) {
    cast_f64_to_f32<<<grid_for(ctx, rowsN), 256, 0, ctx.stream>>>(rowsN, in, X);
    ctx.launches++;
    // source spectrum S^[b][m'] = sum_i S[b][i] F[m'][i]  (B x 2M x n)
    GemmArgs fs = rowmajor(B, 2 * M, n, X, n, op.F, n, Vh, 2 * M, nullptr, ACT_NONE);
    SNOP_TRY(gemm(ctx, fs));
    const bool l0mn = C % 32 == 0;  // the engine's MN-major B needs whole 32-column boxes
    if (l0mn) fno_mix_l0<true><<<grid_for(ctx, (size_t)B * C * M), 256, 0, ctx.stream>>>(B, C, M, Vh, op.l0_P, op.l0_Q, U);
    else fno_mix_l0<false><<<grid_for(ctx, (size_t)B * C * M), 256, 0, ctx.stream>>>(B, C, M, Vh, op.l0_P, op.l0_Q, U);
    ctx.launches++;
    GemmArgs iv{};
    iv.M = n; iv.N = C; iv.K = 2 * M; iv.batch = B;
    iv.A = op.Ginv; iv.sam = 2 * M; iv.sak = 1; iv.sab = 0;
    iv.A_lo = op.Ginv_lo;
    if (l0mn) {  // U' mode-major (MN-major B)
      iv.B = U; iv.sbn = 1; iv.sbk = (int64_t)B * C; iv.sbb = C;
    } else {
      iv.B = U; iv.sbn = 2 * M; iv.sbk = 1; iv.sbb = (int64_t)C * 2 * M;
    }
    iv.C = V; iv.scm = C; iv.scn = 1; iv.scb = (int64_t)n * C;
    iv.bias = op.l0_C; iv.alpha = 1.f; iv.act = op.act;
    iv.r2_a = op.l0_A; iv.r2_b = op.l0_B; iv.r2_s = X; iv.r2_sb = n; iv.r2_x = op.xc;
    SNOP_TRY(gemm(ctx, iv));
  } else {
    fno_lift<<<grid_for(ctx, vsz), 256, 0, ctx.stream>>>(B, n, C, in, op.xc, op.lift_W, op.lift_b, V);
    ctx.launches++;
  }
  for (int l = l0 ? 1 : 0; l < op.layers; ++l) {
    bool u_mn = false;  // U written mode-major [2M][B][C] by the tensor-core mixing
    // forward truncated DFT: Vh[b][c][m'] = sum_i V[b][i][c] F[m'][i]. Tensor-core engine: one
    // GEMM over all B*C rows (batch folded into M); FFMA engine: batched per sample.
    GemmArgs f{};
    f.M = C; f.N = 2 * M; f.K = n; f.batch = B;
    f.A = V; f.sam = 1; f.sak = C; f.sab = (int64_t)n * C;
    f.B = op.F; f.sbn = n; f.sbk = 1; f.sbb = 0;
    f.C = Vh; f.scm = 2 * M; f.scn = 1; f.scb = (int64_t)C * 2 * M;
    f.alpha = 1.f; f.act = ACT_NONE;
    bool tc_done = false;
    if (C == 64 && 2 * M == 32 && n % 128 == 0 && use_tc(ctx) && ctx.opt.fno_dft == 0) {
      cudaError_t e = cudaSuccess;
      if (fno_dft_tc(V, op.F, op.F_lo, Vh, B, n, ctx.stream, &e)) {
        SNOP_TRY(cuda_status("fno_dft_tc", e));
        ctx.launches++;
        tc_done = true;
      }
    }
    if (tc_done) {
    } else if (C == 64 && 2 * M == 32 && n % DFT_ROWS == 0 && op.FT) {
      const size_t sm = DFT_ST * sizeof(DftStage) + 2 * DFT_ST * sizeof(uint64_t);
      cudaFuncSetAttribute(fno_dft64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      fno_dft64<<<(B + DFT_S - 1) / DFT_S, 32 * DFT_S, sm, ctx.stream>>>(B, n, V, op.FT, Vh);
      ctx.launches++;
      SNOP_TRY(cuda_status("fno_dft64", cudaGetLastError()));
    } else if (use_tc(ctx)) {
      f.M = B * C;
      f.batch = 1;
      SNOP_TRY(gemm(ctx, f, C));
    } else {
      SNOP_TRY(gemm(ctx, f));
    }
    // complex channel mixing per retained mode
    if (tc_done && use_tc(ctx) && ctx.opt.fno_mix == 0) {
      // on the tensor core: per mode m, U_re = [V_re | V_im] . [Rr ; -Ri] and U_im = [V_re | V_im] .
      // [Ri ; Rr] - two mode-batched 3xTF32 GEMMs (samples x C outputs x 2C, the mode-major spectra
      // Vh [2M][B][C] read as two K segments) writing U' [2M][B][C] (mode-major, channel rows
      // contiguous: whole-tile TMA stores); the inverse GEMM then reads U' as an N-contiguous
      // (MN-major) B operand
      const size_t MCC = (size_t)M * C * C;
      for (int part = 0; part < 2; ++part) {
        GemmArgs mx{};
        mx.M = B; mx.N = C; mx.K = 2 * C; mx.batch = M;
        mx.A = Vh; mx.sam = C; mx.sak = 1; mx.sab = (int64_t)B * C;
        mx.ksplit = C;
        mx.A2 = Vh + (size_t)M * B * C; mx.sam2 = C; mx.sak2 = 1; mx.sab2 = (int64_t)B * C;
        mx.B = op.mixB[l] + (2 * part) * MCC; mx.sbn = C; mx.sbk = 1; mx.sbb = (int64_t)C * C;
        mx.B2 = op.mixB[l] + (2 * part + 1) * MCC; mx.sbn2 = C; mx.sbk2 = 1; mx.sbb2 = (int64_t)C * C;
        mx.B_lo = op.mixB_lo[l] + (2 * part) * MCC;
        mx.B2_lo = op.mixB_lo[l] + (2 * part + 1) * MCC;
        mx.C = U + (size_t)part * M * B * C; mx.scb = (int64_t)B * C; mx.scm = C; mx.scn = 1;
        mx.alpha = 1.f; mx.act = ACT_NONE;
        SNOP_TRY(gemm(ctx, mx));
      }
      u_mn = true;
    } else if (C == 64 && tc_done) {  // the tensor-core DFT wrote Vh mode-major
      const size_t sm = (size_t)(128 * 128 + 128 * (MIX_S + 4)) * sizeof(float);
      cudaFuncSetAttribute(fno_mix64<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      fno_mix64<true><<<dim3((B + MIX_S - 1) / MIX_S, M), 256, sm, ctx.stream>>>(B, M, Vh, op.Rr[l], op.Ri[l], U);
    } else if (C == 64) {
      const size_t sm = (size_t)(128 * 128 + 128 * MIX_S) * sizeof(float);
      cudaFuncSetAttribute(fno_mix64<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      fno_mix64<false><<<dim3((B + MIX_S - 1) / MIX_S, M), 256, sm, ctx.stream>>>(B, M, Vh, op.Rr[l], op.Ri[l], U);
    } else {
      fno_mix<<<dim3((B + 3) / 4 < 1024 ? (B + 3) / 4 : 1024, M), 4 * C, 2 * C * C * sizeof(float), ctx.stream>>>(
          B, C, M, Vh, op.Rr[l], op.Ri[l], U);
    }
    if (!(tc_done && use_tc(ctx) && ctx.opt.fno_mix == 0)) ctx.launches++;
    if (tc_fused) {
      // inverse truncated DFT + W path + bias + activation as ONE contraction per sample:
      // Vn[b][i][o] = act( [Ginv | V_b](i, :) . [U_b | W](o, :) + b[o] ),  K = 2M + C
      GemmArgs iv{};
      iv.M = n; iv.N = C; iv.K = 2 * M + C; iv.batch = B;
      iv.A = op.Ginv; iv.sam = 2 * M; iv.sak = 1; iv.sab = 0;
      if (u_mn) {  // U' [2M][B][C]: element (b, o, m') at m' B C + b C + o
        iv.B = U; iv.sbn = 1; iv.sbk = (int64_t)B * C; iv.sbb = C;
      } else {
        iv.B = U; iv.sbn = 2 * M; iv.sbk = 1; iv.sbb = (int64_t)C * 2 * M;
      }
      iv.ksplit = 2 * M;
      iv.A2 = V; iv.sam2 = C; iv.sak2 = 1; iv.sab2 = (int64_t)n * C;
      iv.B2 = op.W[l]; iv.sbn2 = C; iv.sbk2 = 1; iv.sbb2 = 0;
      // (pre-split lo parts measured slower here: the extra lo tiles are re-read for every output
      // tile and the K = 96 pipeline is not converter-bound; they pay off for layer 0 and the
      // projection only)
      iv.C = Vn; iv.scm = C; iv.scn = 1; iv.scb = (int64_t)n * C;
      iv.bias = op.b[l]; iv.alpha = 1.f; iv.act = op.act;
      SNOP_TRY(gemm(ctx, iv));
    } else {
      // inverse truncated DFT per sample: Vn[b][i][o] = sum_m' Ginv[i][m'] U[b][o][m']
      GemmArgs iv{};
      iv.M = n; iv.N = C; iv.K = 2 * M; iv.batch = B;
      iv.A = op.Ginv; iv.sam = 2 * M; iv.sak = 1; iv.sab = 0;
      if (u_mn) {
        iv.B = U; iv.sbn = 1; iv.sbk = (int64_t)B * C; iv.sbb = C;
      } else {
        iv.B = U; iv.sbn = 2 * M; iv.sbk = 1; iv.sbb = (int64_t)C * 2 * M;
      }
      iv.C = Vn; iv.scm = C; iv.scn = 1; iv.scb = (int64_t)n * C;
      iv.alpha = 1.f; iv.act = ACT_NONE;
      SNOP_TRY(gemm(ctx, iv));
      // + W path + bias, activation (accumulating epilogue)
      GemmArgs wp = rowmajor((int)rowsN, C, C, V, C, op.W[l], C, Vn, C, op.b[l], op.act);
      wp.beta = 1.f;
      SNOP_TRY(gemm(ctx, wp));
    }
    std::swap(V, Vn);
  }
  // projection 64 -> hidden (act) -> 1. Tensor-core engine: one GEMM whose epilogue does the
  // second layer as a row-dot (no hidden tensor in HBM); FFMA engine: chunked GEMM + rowdot.
  if (use_tc(ctx) && H <= 128) {
    GemmArgs pj = rowmajor((int)rowsN, H, C, V, C, op.P1W, C, nullptr, 1, op.P1b, op.act);
    pj.B_lo = op.P1W_lo;
    pj.scm = 1;
    pj.rowdot_w = op.P2W;
    pj.rowdot_out = out;
    pj.rowdot_b = op.p2b_host;
    if (H > 64) SNOP_TRY(cuda_status("zero", cudaMemsetAsync(out, 0, rowsN * sizeof(double), ctx.stream)));
    SNOP_TRY(gemm(ctx, pj));
  } else {
    const size_t chunk = (size_t)1 << 18;
    float* h = static_cast<float*>(ctx.slot(49, chunk * H * sizeof(float)));
    if (!h) return cuda_status("FNO projection workspace", cudaErrorMemoryAllocation);
    for (size_t r0 = 0; r0 < rowsN; r0 += chunk) {
      const int rows = (int)std::min(chunk, rowsN - r0);
      SNOP_TRY(gemm(ctx, rowmajor(rows, H, C, V + r0 * C, C, op.P1W, C, h, H, op.P1b, op.act)));
      rowdot<<<grid_for(ctx, (size_t)rows * 32), 256, 0, ctx.stream>>>(rows, H, h, op.P2W, op.P2b, out + r0);
      ctx.launches++;
    }
  }
  return cuda_status("FNO forward", cudaGetLastError());
}

snop_status drain(Ctx& ctx) {
  int flags = 0;
  cudaError_t e = cudaMemcpyAsync(&flags, ctx.d_flags, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx.stream);
  if (e != cudaSuccess) return cuda_status("synchronize", e);
  ctx.settle_loops();
  if (flags) cudaMemsetAsync(ctx.d_flags, 0, sizeof(int), ctx.stream);
  if (flags & FLAG_BAD_SIGMA_T) return invalid("nonpositive sigma_t in at least one instance");
  if (flags & FLAG_DEGENERATE) {
    set_error("zero fission integral in at least one instance");
    return SNOP_DEGENERATE_PROBLEM;
  }
  if (flags & FLAG_NONFINITE) {
    set_error("non-finite values produced");
    return SNOP_NUMERICAL_ERROR;
  }
  return SNOP_OK;
}

// Runs `body` (which enqueues one iteration on ctx.stream and ends with loop_ctl on the handle it
// is given) as the body of a WHILE conditional node of a CUDA graph: the iteration loop runs on
// the device with no host round trip per iteration. Top level: the executable is cached on the
// context under `key` (every pointer and scalar the body captures, plus the workspace
// generation), so repeated calls with the same buffers relaunch it directly. Nested (ctx.stream is
// being captured by an enclosing device loop): the conditional node is added to the enclosing
// body graph and this body is captured into it through the context's side stream.
// The body returns its kernel count through `n_body` for loop_ctl's launch accounting.
template <class Body>
snop_status device_loop(Ctx& ctx, std::vector<uint64_t> key, Body&& body) {
  if (!ctx.d_loop_launches) {
    if (cudaMalloc(&ctx.d_loop_launches, sizeof(unsigned long long)) != cudaSuccess)
      return cuda_status("cudaMalloc", cudaErrorMemoryAllocation);
    cudaMemsetAsync(ctx.d_loop_launches, 0, sizeof(unsigned long long), ctx.stream);
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  SNOP_TRY(cuda_status("capture status", cudaStreamIsCapturing(ctx.stream, &cs)));
  const bool nested = cs == cudaStreamCaptureStatusActive;
  // capture `body` into the body graph of a new WHILE node of graph g (after deps)
  auto build = [&](cudaGraph_t g, const cudaGraphNode_t* deps, size_t ndeps, cudaStream_t cap,
                   cudaGraphNode_t* node_out, cudaGraphConditionalHandle h) -> snop_status {
    cudaError_t e = cudaSuccess;
    cudaGraphNodeParams np{};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    if (e == cudaSuccess) e = cudaGraphAddNode(node_out, g, deps, ndeps, &np);
    if (e != cudaSuccess) return cuda_status("device loop node", e);
    const cudaStream_t outer = ctx.stream;
    ctx.stream = cap;
    e = cudaStreamBeginCaptureToGraph(cap, np.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                      cudaStreamCaptureModeRelaxed);
    snop_status bs = SNOP_OK;
    if (e == cudaSuccess) {
      const int64_t l0 = ctx.launches;
      bs = body(h);
      ctx.launches = l0;  // captured, not launched: counted on the device per pass
      cudaGraph_t out = nullptr;
      e = cudaStreamEndCapture(cap, &out);
    }
    ctx.stream = outer;
    if (bs != SNOP_OK) return bs;
    return cuda_status("device loop capture", e);
  };
  if (nested) {
    if (!ctx.side && cudaStreamCreateWithFlags(&ctx.side, cudaStreamNonBlocking) != cudaSuccess)
      return cuda_status("side stream", cudaErrorUnknown);
    cudaGraph_t g = nullptr;
    SNOP_TRY(cuda_status("capture info", cudaStreamGetCaptureInfo(ctx.stream, &cs, nullptr, &g, nullptr, nullptr)));
    // A nested handle's default value is applied only when the top-level graph is launched, so
    // every pass of the enclosing body re-arms it explicitly before the loop node.
    cudaGraphConditionalHandle h{};
    SNOP_TRY(cuda_status("conditional handle", cudaGraphConditionalHandleCreate(&h, g, 1, 0)));
    loop_arm<<<1, 1, 0, ctx.stream>>>(h);
    ctx.launches++;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    SNOP_TRY(cuda_status("capture info", cudaStreamGetCaptureInfo(ctx.stream, &cs, nullptr, &g, &deps, &ndeps)));
    std::vector<cudaGraphNode_t> dv(deps, deps + ndeps);  // (the returned array is invalidated below)
    cudaGraphNode_t node;
    SNOP_TRY(build(g, dv.data(), dv.size(), ctx.side, &node, h));
    return cuda_status("capture dependencies",
                       cudaStreamUpdateCaptureDependencies(ctx.stream, &node, 1, cudaStreamSetCaptureDependencies));
  }
  key.push_back(ctx.slot_gen);
  {  // execution options select kernels inside the body: a graph captured under others is stale
    const int32_t* o = reinterpret_cast<const int32_t*>(&ctx.opt);
    for (size_t i = 0; i < sizeof(ctx.opt) / sizeof(int32_t); ++i) key.push_back((uint64_t)(uint32_t)o[i]);
  }
  Ctx::LoopGraph* lg = nullptr;
  for (auto& g : ctx.graphs)
    if (g.key == key) lg = &g;
  if (!lg) {
    if (ctx.graphs.size() >= 8) {  // evict the oldest (it may still be running: wait first)
      cudaStreamSynchronize(ctx.stream);
      cudaGraphExecDestroy(ctx.graphs.front().exec);
      ctx.graphs.erase(ctx.graphs.begin());
    }
    // A body may size workspaces on first use while it is captured; nodes captured before a
    // reallocation would hold stale pointers, so such a graph is discarded and captured again.
    cudaGraph_t g = nullptr;
    snop_status bs = SNOP_OK;
    for (int attempt = 0; attempt < 3; ++attempt) {
      const uint64_t gen0 = ctx.slot_gen;
      SNOP_TRY(cuda_status("device loop graph", cudaGraphCreate(&g, 0)));
      cudaGraphNode_t node;
      cudaGraphConditionalHandle h{};
      SNOP_TRY(cuda_status("conditional handle", cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault)));
      bs = build(g, nullptr, 0, ctx.stream, &node, h);
      if (bs == SNOP_OK && ctx.slot_gen == gen0) break;
      cudaGraphDestroy(g);
      g = nullptr;
      cudaGetLastError();  // a capture broken by an allocation leaves a sticky-free error state
    }
    if (!g) return bs != SNOP_OK ? bs : cuda_status("device loop capture", cudaErrorStreamCaptureInvalidated);
    key[key.size() - 1 - sizeof(ctx.opt) / sizeof(int32_t)] = ctx.slot_gen;
    cudaGraphExec_t ex = nullptr;
    const cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_status("device loop instantiate", e);
    ctx.graphs.push_back({key, ex});
    lg = &ctx.graphs.back();
  }
  return cuda_status("device loop launch", cudaGraphLaunch(lg->exec, ctx.stream));
}

snop_status recast_fp_dev(Ctx& ctx, snop_op& op, int B, const double* S, const double* st, const double* ss,
                          double tol, int max_it, int norm, const double* init, double* phi, int32_t* iters,
                          int32_t* status, const uint8_t* outer_active = nullptr) {
  const int n = op.grid.n_cells;
  const size_t N = (size_t)B * n;
  double* phi0 = static_cast<double*>(ctx.slot(50, N * sizeof(double)));
  double* s = static_cast<double*>(ctx.slot(51, N * sizeof(double)));
  double* nx = static_cast<double*>(ctx.slot(52, N * sizeof(double)));
  double* norm0 = static_cast<double*>(ctx.slot(53, (size_t)B * sizeof(double)));
  uint8_t* active = static_cast<uint8_t*>(ctx.slot(54, (size_t)B));
  int* n_active = static_cast<int*>(ctx.slot(55, 2 * sizeof(int)));
  if (!phi0 || !s || !nx || !norm0 || !active || !n_active) return cuda_status("workspace", cudaErrorMemoryAllocation);
  int* it_done = n_active + 1;
  if (init) SNOP_TRY(cuda_status("copy", cudaMemcpyAsync(phi0, init, N * sizeof(double), cudaMemcpyDeviceToDevice, ctx.stream)));
  else SNOP_TRY(op_predict_dev(ctx, op, B, S, phi0));  // Eq. 9 with zero initial guess
  maxabs_rows<<<B, 256, 0, ctx.stream>>>(n, phi0, norm0);
  ctx.launches++;
  SNOP_TRY(cuda_status("copy", cudaMemcpyAsync(phi, phi0, N * sizeof(double), cudaMemcpyDeviceToDevice, ctx.stream)));
  if (outer_active)  // instances an enclosing loop has frozen do not iterate
    cudaMemcpyAsync(active, outer_active, (size_t)B, cudaMemcpyDeviceToDevice, ctx.stream);
  else
    cudaMemsetAsync(active, 1, (size_t)B, ctx.stream);
  cudaMemsetAsync(iters, 0, (size_t)B * sizeof(int32_t), ctx.stream);
  cudaMemsetAsync(it_done, 0, sizeof(int), ctx.stream);
  fill_i32<<<grid_for(ctx, (size_t)B), 256, 0, ctx.stream>>>(B, SNOP_RECAST_MAXED, status);
  ctx.launches++;
  if (max_it < 1) return cuda_status("recast fixed point", cudaGetLastError());
  // One iteration per pass of the device loop: recast source, operator
  // forward, per-instance update/freeze, loop control.
  auto body = [&](cudaGraphConditionalHandle h) -> snop_status {
    const int64_t l0 = ctx.launches;
    SNOP_TRY(launch_recast(ctx, N, S, phi, st, ss, op.tstar, op.sstar, s));
    SNOP_TRY(op_predict_dev(ctx, op, B, s, nx, active));
    cudaMemsetAsync(n_active, 0, sizeof(int), ctx.stream);
    recast_update<<<B, 256, 0, ctx.stream>>>(n, norm, tol, it_done, nx, phi, phi0, norm0, active, iters, status,
                                             n_active);
    const int nb = (int)(ctx.launches - l0) + 2;
    loop_ctl<<<1, 1, 0, ctx.stream>>>(h, it_done, n_active, max_it, nb, ctx.d_loop_launches);
    return cuda_status("recast iteration", cudaGetLastError());
  };
  uint64_t tolbits;
  std::memcpy(&tolbits, &tol, sizeof tolbits);
  const std::vector<uint64_t> key = {1, (uint64_t)(uintptr_t)&op, op.serial, (uint64_t)B, (uint64_t)(uintptr_t)S,
                                     (uint64_t)(uintptr_t)st, (uint64_t)(uintptr_t)ss, (uint64_t)(uintptr_t)phi,
                                     (uint64_t)(uintptr_t)iters, (uint64_t)(uintptr_t)status, tolbits,
                                     (uint64_t)max_it, (uint64_t)norm, op.gen, (uint64_t)(uintptr_t)outer_active};
  return device_loop(ctx, key, body);
}

snop_status check_op(snop_ctx* ctx, snop_op* op) {
  if (!ctx || !op) return invalid("ctx/op is NULL");
  if (op->ctx != ctx) return invalid("operator was created on another context");
  return SNOP_OK;
}

template <class T>
snop_status stage(Ctx& ctx, size_t slot, const T* h, size_t n, T** d) {
  if (!h) {
    *d = nullptr;
    return SNOP_OK;
  }
  *d = static_cast<T*>(ctx.slot(slot, n * sizeof(T)));
  if (!*d) return cuda_status("cudaMalloc", cudaErrorMemoryAllocation);
  return cuda_status("H2D", cudaMemcpyAsync(*d, h, n * sizeof(T), cudaMemcpyHostToDevice, ctx.stream));
}

template <class T>
snop_status unstage(Ctx& ctx, T* h, const T* d, size_t n) {
  if (!h) return SNOP_OK;
  return cuda_status("D2H", cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, ctx.stream));
}

bool valid_act(int a) { return a == ACT_RELU || a == ACT_TANH || a == ACT_GELU; }


// ---- SP / CP hybrid eigenvalue solve (paper Eqs. A5-A8) -----------------------
// Stage 1 is a power iteration whose within-group solve is the operator: SP = recast fixed point
// warm-started from the current group flux (Eq. A5); CP = that prediction refined by a
// model-based source iteration (Eqs. A7-A8). Stage 2 is the fused model-based power iteration
// (K2) started from (k_NO, phi_NO), or from the cold start where stage 1 diverged.
// The outer loop is host-orchestrated because the operator is a multi-kernel pipeline; the
// per-instance bookkeeping (fission density, group source, k update, convergence, freeze) is in
// the one-CTA-per-instance kernels below.
constexpr int HY_THREADS = 256;

__device__ double hy_block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x / 32] = v;
  __syncthreads();
  double r = 0.0;
  for (int u = 0; u < HY_THREADS / 32; ++u) r += sh[u];
  return r;
}

__device__ double hy_block_max(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x / 32] = v;
  __syncthreads();
  double r = 0.0;
  for (int u = 0; u < HY_THREADS / 32; ++u) r = fmax(r, sh[u]);
  return r;
}

// dx * sum_i sum_g nuSf_g,i phi_g,i for instance b
__device__ double hy_fission_integral(int G, int Nc, double dx, const double* nsf, const double* phi, double* sh) {
  double s = 0.0;
  for (int i = threadIdx.x; i < Nc; i += HY_THREADS) {
    double f = 0.0;
    for (int g = 0; g < G; ++g) f = fma(nsf[(size_t)g * Nc + i], phi[(size_t)g * Nc + i], f);
    s += f;
  }
  return hy_block_sum(s, sh) * dx;
}

__global__ void __launch_bounds__(HY_THREADS) hy_init(int G, int Nc, double dx, const double* __restrict__ st,
                                                      const double* __restrict__ nsf, double* __restrict__ phi,
                                                      double* __restrict__ k, uint8_t* __restrict__ active,
                                                      uint8_t* __restrict__ fb, uint8_t* __restrict__ div,
                                                      int32_t* __restrict__ outer, int64_t* __restrict__ inner,
                                                      int* __restrict__ flags) {
  __shared__ double sh[HY_THREADS / 32];
  const int b = blockIdx.x;
  const size_t GN = (size_t)G * Nc;
  double* p = phi + b * GN;
  int bad = 0;
  for (size_t i = threadIdx.x; i < GN; i += HY_THREADS) {
    p[i] = 1.0;
    bad |= !(st[b * GN + i] > 0.0);
  }
  bad = __syncthreads_or(bad);
  const double F = hy_fission_integral(G, Nc, dx, nsf + b * GN, p, sh);
  const bool ok = !bad && F != 0.0 && isfinite(F);
  if (ok)
    for (size_t i = threadIdx.x; i < GN; i += HY_THREADS) p[i] /= F;
  if (threadIdx.x == 0) {
    if (bad) atomicOr(flags, FLAG_BAD_SIGMA_T);
    k[b] = 1.0;
    active[b] = ok ? 1 : 0;
    fb[b] = ok ? 0 : 1;
    div[b] = 0;
    outer[b] = 0;
    inner[b] = 0;
  }
}

// old = phi; fiss_i = sum_g nuSf_g,i phi_g,i (frozen for the Gauss-Seidel pass)
__global__ void hy_outer_begin(int G, int Nc, const double* __restrict__ nsf, const double* __restrict__ phi,
                               double* __restrict__ old, double* __restrict__ fiss, const uint8_t* __restrict__ active) {
  const int b = blockIdx.x;
  if (!active[b]) return;
  const size_t GN = (size_t)G * Nc;
  for (int i = threadIdx.x; i < Nc; i += blockDim.x) {
    double f = 0.0;
    for (int g = 0; g < G; ++g) {
      const double v = phi[b * GN + (size_t)g * Nc + i];
      old[b * GN + (size_t)g * Nc + i] = v;
      f = fma(nsf[b * GN + (size_t)g * Nc + i], v, f);
    }
    fiss[(size_t)b * Nc + i] = f;
  }
}

// Group-g inputs, gathered contiguous [B][Nc]: q_ext = chi_g fiss / k + sum_{g'!=g} Ss0(g'->g) phi_g',
// Sigma_t,g, Sigma_s0(g->g), Sigma_s1,g and the warm-start flux phi_g.
__global__ void hy_group_in(int g, int G, int Nc, const double* __restrict__ chi, const double* __restrict__ k,
                            const double* __restrict__ st, const double* __restrict__ ss0,
                            const double* __restrict__ ss1, const double* __restrict__ phi,
                            const double* __restrict__ fiss, double* __restrict__ qext, double* __restrict__ stg,
                            double* __restrict__ ssg, double* __restrict__ s1g, double* __restrict__ phig) {
  const int b = blockIdx.x;
  const size_t GN = (size_t)G * Nc;
  const double chig = chi[(size_t)b * G + g] / k[b];
  for (int i = threadIdx.x; i < Nc; i += blockDim.x) {
    const size_t o = (size_t)b * Nc + i;
    double q = chig * fiss[o];
    for (int gp = 0; gp < G; ++gp)
      if (gp != g) q = fma(ss0[b * GN * G + ((size_t)gp * G + g) * Nc + i], phi[b * GN + (size_t)gp * Nc + i], q);
    qext[o] = q;
    stg[o] = st[b * GN + (size_t)g * Nc + i];
    ssg[o] = ss0[b * GN * G + ((size_t)g * G + g) * Nc + i];
    if (ss1) s1g[o] = ss1[b * GN + (size_t)g * Nc + i];
    phig[o] = phi[b * GN + (size_t)g * Nc + i];
  }
}

__global__ void hy_group_out(int g, int G, int Nc, const double* __restrict__ phig, double* __restrict__ phi,
                             const uint8_t* __restrict__ active, const int32_t* __restrict__ it_a,
                             const int32_t* __restrict__ it_b, const int32_t* __restrict__ rstatus,
                             int64_t* __restrict__ inner, uint8_t* __restrict__ div) {
  const int b = blockIdx.x;
  if (!active[b]) return;
  const size_t GN = (size_t)G * Nc;
  for (int i = threadIdx.x; i < Nc; i += blockDim.x) phi[b * GN + (size_t)g * Nc + i] = phig[(size_t)b * Nc + i];
  if (threadIdx.x == 0) {
    inner[b] += it_a[b] + (it_b ? it_b[b] : 0);
    if (rstatus[b] == SNOP_RECAST_DIVERGED) div[b] = 1;
  }
}

// k_new = k F1 (old flux had unit fission integral), phi /= F1, convergence on dk and dphi.
__global__ void __launch_bounds__(HY_THREADS) hy_outer_end(int G, int Nc, double dx, const int* __restrict__ outer_done,
                                                           double tol_k,
                                                           double tol_phi, int norm, const double* __restrict__ nsf,
                                                           double* __restrict__ phi, const double* __restrict__ old,
                                                           double* __restrict__ k, uint8_t* __restrict__ active,
                                                           uint8_t* __restrict__ fb, int32_t* __restrict__ outer,
                                                           int* __restrict__ n_active) {
  __shared__ double sh[HY_THREADS / 32];
  const int b = blockIdx.x;
  if (!active[b]) return;
  const int outer_it = *outer_done + 1;  // this outer iteration (the device loop counts them)
  const size_t GN = (size_t)G * Nc;
  double* p = phi + b * GN;
  const double F1 = hy_fission_integral(G, Nc, dx, nsf + b * GN, p, sh);
  if (!(F1 != 0.0) || !isfinite(F1)) {  // degenerate stage 1 -> cold-start fallback
    if (threadIdx.x == 0) {
      active[b] = 0;
      fb[b] = 1;
      outer[b] = outer_it;
    }
    return;
  }
  const double kb = k[b], k_new = kb * F1;
  double num = 0.0, den = 0.0;
  for (size_t i = threadIdx.x; i < GN; i += HY_THREADS) {
    const double pn = p[i] / F1;
    p[i] = pn;
    const double d = pn - old[b * GN + i];
    if (norm == 0) {
      num = fmax(num, fabs(d));
      den = fmax(den, fabs(pn));
    } else {
      num = fma(d, d, num);
      den = fma(pn, pn, den);
    }
  }
  if (norm == 0) {
    num = hy_block_max(num, sh);
    den = hy_block_max(den, sh);
  } else {
    num = hy_block_sum(num, sh);
    den = hy_block_sum(den, sh);
  }
  if (threadIdx.x == 0) {
    const double dphi = snop_dev::rel_change(num, den, norm);
    const double dk = fabs(k_new - kb) / fabs(k_new);
    k[b] = k_new;
    outer[b] = outer_it;
    if (dk < tol_k && dphi < tol_phi) active[b] = 0;
    else atomicAdd(n_active, 1);
  }
}

// Stage-2 start: (k_NO, phi_NO), or the flat cold start where stage 1 diverged.
__global__ void hy_stage2_init(int G, int Nc, double* __restrict__ phi, const double* __restrict__ k1,
                               double* __restrict__ k0, uint8_t* __restrict__ fb, const uint8_t* __restrict__ div) {
  const int b = blockIdx.x;
  const double kb = k1[b];
  const bool f = fb[b] || div[b] || !isfinite(kb) || !(kb > 0.0);
  if (f) {
    const size_t GN = (size_t)G * Nc;
    for (size_t i = threadIdx.x; i < GN; i += blockDim.x) phi[b * GN + i] = 1.0;
  }
  if (threadIdx.x == 0) {
    fb[b] = f ? 1 : 0;
    k0[b] = f ? 1.0 : kb;
  }
}

struct HybridOut {
  double *k, *phi, *k1;
  int32_t *outer1, *outer2;
  int64_t *inner1, *inner2;
  uint8_t *conv, *fb;
};

// Result of a stage-1-only run (power iteration with the operator as inner solver): the stage-1
// flux and eigenvalue, converged = the dual test was met, fb = diverged or degenerate.
__global__ void hy_stage1_out(int G, int Nc, const double* __restrict__ phi1, double* __restrict__ phi,
                              const double* __restrict__ k1, double* __restrict__ k, const uint8_t* __restrict__ active,
                              uint8_t* __restrict__ fb, const uint8_t* __restrict__ div, uint8_t* __restrict__ conv) {
  const int b = blockIdx.x;
  const size_t GN = (size_t)G * Nc;
  for (size_t i = threadIdx.x; i < GN; i += blockDim.x) phi[b * GN + i] = phi1[b * GN + i];
  if (threadIdx.x == 0) {
    const bool f = fb[b] || div[b];
    if (k != k1) k[b] = k1[b];
    fb[b] = f ? 1 : 0;
    conv[b] = (!f && !active[b]) ? 1 : 0;
  }
}

snop_status hybrid_eigen_dev(Ctx& ctx, snop_op& op, int algorithm, int order, int B, int G, const double* st,
                             const double* ss0, const double* ss1, const double* nsf, const double* chi,
                             const snop_solver_config& cfg, double rtol, int rmax, const HybridOut& o,
                             bool stage1_only = false) {
  const int Nc = op.grid.n_cells;
  const size_t N = (size_t)B * Nc, GNB = N * G;
  const double dx = op.grid.length_cm / Nc;
  auto dslot = [&](int i, size_t n) { return static_cast<double*>(ctx.slot(i, n * sizeof(double))); };
  double *phi1 = dslot(80, GNB), *old = dslot(81, GNB), *fiss = dslot(82, N), *qext = dslot(83, N);
  double *stg = dslot(84, N), *ssg = dslot(85, N), *s1g = ss1 ? dslot(86, N) : nullptr, *phig = dslot(87, N);
  double *pred = dslot(88, N), *refined = dslot(89, N), *k0 = dslot(90, B);
  uint8_t* active = static_cast<uint8_t*>(ctx.slot(91, (size_t)B));
  uint8_t* div = static_cast<uint8_t*>(ctx.slot(92, (size_t)B));
  int32_t* rit = static_cast<int32_t*>(ctx.slot(93, (size_t)B * sizeof(int32_t)));
  int32_t* rst = static_cast<int32_t*>(ctx.slot(94, (size_t)B * sizeof(int32_t)));
  int32_t* sit = static_cast<int32_t*>(ctx.slot(95, (size_t)B * sizeof(int32_t)));
  uint8_t* scv = static_cast<uint8_t*>(ctx.slot(96, (size_t)B));
  int* n_active = static_cast<int*>(ctx.slot(97, sizeof(int)));
  double* pi_old = dslot(98, GNB);
  if (!phi1 || !old || !fiss || !qext || !stg || !ssg || (ss1 && !s1g) || !phig || !pred || !refined || !k0 ||
      !active || !div || !rit || !rst || !sit || !scv || !n_active || !pi_old)
    return cuda_status("workspace", cudaErrorMemoryAllocation);
  cudaStream_t s = ctx.stream;
  hy_init<<<B, HY_THREADS, 0, s>>>(G, Nc, dx, st, nsf, phi1, o.k1, active, o.fb, div, o.outer1, o.inner1,
                                   ctx.d_flags);
  ctx.launches++;
  // Stage 1: the outer loop runs on the device (WHILE conditional node); each group's recast fixed
  // point is a nested device loop. Instances whose stage 1 has finished are frozen (skipped).
  int* outer_done = static_cast<int*>(ctx.slot(99, sizeof(int)));
  if (!outer_done) return cuda_status("workspace", cudaErrorMemoryAllocation);
  cudaMemsetAsync(outer_done, 0, sizeof(int), s);
  auto body = [&](cudaGraphConditionalHandle h) -> snop_status {
    const cudaStream_t cs = ctx.stream;  // (the capture stream of this body)
    const int64_t l0 = ctx.launches;
    hy_outer_begin<<<B, HY_THREADS, 0, cs>>>(G, Nc, nsf, phi1, old, fiss, active);
    ctx.launches++;
    for (int g = 0; g < G; ++g) {
      hy_group_in<<<B, HY_THREADS, 0, cs>>>(g, G, Nc, chi, o.k1, st, ss0, ss1, phi1, fiss, qext, stg, ssg, s1g, phig);
      ctx.launches++;
      SNOP_TRY(recast_fp_dev(ctx, op, B, qext, stg, ssg, rtol, rmax, cfg.norm, phig, pred, rit, rst, active));
      const double* result = pred;
      if (algorithm == 1) {  // (instances whose stage 1 has finished are skipped)
        SNOP_TRY(launch_source_iteration(ctx, op.grid, order, B, stg, ssg, s1g, qext, cfg, pred, refined, nullptr,
                                         sit, scv, nullptr, nullptr, active));
        result = refined;
      }
      hy_group_out<<<B, HY_THREADS, 0, cs>>>(g, G, Nc, result, phi1, active, rit, algorithm == 1 ? sit : nullptr,
                                             rst, o.inner1, div);
      ctx.launches++;
    }
    cudaMemsetAsync(n_active, 0, sizeof(int), cs);
    hy_outer_end<<<B, HY_THREADS, 0, cs>>>(G, Nc, dx, outer_done, cfg.tolerance_k, cfg.tolerance_phi, cfg.norm,
                                           nsf, phi1, old, o.k1, active, o.fb, o.outer1, n_active);
    const int nb = (int)(ctx.launches - l0) + 2;
    loop_ctl<<<1, 1, 0, cs>>>(h, outer_done, n_active, cfg.max_outer, nb, ctx.d_loop_launches);
    return cuda_status("hybrid stage 1", cudaGetLastError());
  };
  uint64_t bits[4];
  std::memcpy(&bits[0], &rtol, 8);
  std::memcpy(&bits[1], &cfg.tolerance, 8);
  std::memcpy(&bits[2], &cfg.tolerance_k, 8);
  std::memcpy(&bits[3], &cfg.tolerance_phi, 8);
  const std::vector<uint64_t> key = {2, (uint64_t)(uintptr_t)&op, op.serial, op.gen, (uint64_t)algorithm,
                                     (uint64_t)order, (uint64_t)B, (uint64_t)G, (uint64_t)(uintptr_t)st,
                                     (uint64_t)(uintptr_t)ss0, (uint64_t)(uintptr_t)ss1, (uint64_t)(uintptr_t)nsf,
                                     (uint64_t)(uintptr_t)chi, (uint64_t)(uintptr_t)o.k1,
                                     (uint64_t)(uintptr_t)o.fb, (uint64_t)(uintptr_t)o.outer1,
                                     (uint64_t)(uintptr_t)o.inner1, bits[0], bits[1], bits[2], bits[3],
                                     (uint64_t)rmax, (uint64_t)cfg.max_outer, (uint64_t)cfg.max_inner,
                                     (uint64_t)cfg.norm, (uint64_t)cfg.bc_left, (uint64_t)cfg.bc_right};
  SNOP_TRY(device_loop(ctx, key, body));
  if (stage1_only) {
    hy_stage1_out<<<B, HY_THREADS, 0, s>>>(G, Nc, phi1, o.phi, o.k1, o.k, active, o.fb, div, o.conv);
    ctx.launches++;
    return cuda_status("hybrid stage 1 output", cudaGetLastError());
  }
  hy_stage2_init<<<B, HY_THREADS, 0, s>>>(G, Nc, phi1, o.k1, k0, o.fb, div);
  ctx.launches++;
  return launch_power_iteration(ctx, op.grid, order, B, G, st, ss0, ss1, nsf, chi, cfg, k0, phi1, o.k, o.phi,
                                pi_old, o.outer2, o.inner2, o.conv);
}


// ---- power iteration for slabs beyond the resident kernels ------------------
// The fused K2 kernel keeps an instance in one CTA's (or cluster's) shared memory; above 16384
// cells the outer loop runs instead as a device loop (WHILE graph) over the same bookkeeping the
// hybrid stage 1 uses - fission density, group sources (Gauss-Seidel, newest flux, upscatter),
// warm-started inner solves on the streaming K1, k update, renormalisation, dual test - with
// K2's validation and error semantics.
__global__ void __launch_bounds__(HY_THREADS) pi_big_init(int G, int Nc, double dx, const double* __restrict__ st,
                                                          const double* __restrict__ nsf, const double* __restrict__ k0,
                                                          const double* __restrict__ phi0, double* __restrict__ phi,
                                                          double* __restrict__ k, uint8_t* __restrict__ active,
                                                          uint8_t* __restrict__ conv, int32_t* __restrict__ outer,
                                                          int64_t* __restrict__ inner, int* __restrict__ flags) {
  __shared__ double sh[HY_THREADS / 32];
  const int b = blockIdx.x;
  const size_t GN = (size_t)G * Nc;
  double* p = phi + b * GN;
  int bad = 0;
  for (size_t i = threadIdx.x; i < GN; i += HY_THREADS) {
    p[i] = phi0 ? phi0[b * GN + i] : 1.0;
    bad |= !(st[b * GN + i] > 0.0);
  }
  const double kb = k0 ? k0[b] : 1.0;
  bad = __syncthreads_or(bad) || !(kb > 0.0);
  const double F = bad ? 1.0 : hy_fission_integral(G, Nc, dx, nsf + b * GN, p, sh);
  const bool degen = !bad && (!(F != 0.0) || !isfinite(F));
  if (!bad && !degen)
    for (size_t i = threadIdx.x; i < GN; i += HY_THREADS) p[i] /= F;
  if (threadIdx.x == 0) {
    if (bad) atomicOr(flags, FLAG_BAD_SIGMA_T);
    if (degen) atomicOr(flags, FLAG_DEGENERATE);
    k[b] = (bad || degen) ? __longlong_as_double(0x7ff8000000000000ll) : kb;
    active[b] = (bad || degen) ? 0 : 1;
    conv[b] = 0;
    outer[b] = 0;
    inner[b] = 0;
  }
}

__global__ void pi_big_group_out(int g, int G, int Nc, const double* __restrict__ phig, double* __restrict__ phi,
                                 const uint8_t* __restrict__ active, const int32_t* __restrict__ it,
                                 int64_t* __restrict__ inner) {
  const int b = blockIdx.x;
  if (!active[b]) return;
  const size_t GN = (size_t)G * Nc;
  for (int i = threadIdx.x; i < Nc; i += blockDim.x) phi[b * GN + (size_t)g * Nc + i] = phig[(size_t)b * Nc + i];
  if (threadIdx.x == 0) inner[b] += it[b];
}

__global__ void __launch_bounds__(HY_THREADS) pi_big_outer_end(int G, int Nc, double dx, const int* __restrict__ outer_done,
                                                               double tol_k, double tol_phi, int norm,
                                                               const double* __restrict__ nsf, double* __restrict__ phi,
                                                               const double* __restrict__ old, double* __restrict__ k,
                                                               uint8_t* __restrict__ active, uint8_t* __restrict__ conv,
                                                               int32_t* __restrict__ outer, int* __restrict__ n_active,
                                                               int* __restrict__ flags) {
  __shared__ double sh[HY_THREADS / 32];
  const int b = blockIdx.x;
  if (!active[b]) return;
  const int outer_it = *outer_done + 1;
  const size_t GN = (size_t)G * Nc;
  double* p = phi + b * GN;
  const double F1 = hy_fission_integral(G, Nc, dx, nsf + b * GN, p, sh);
  if (!(F1 != 0.0) || !isfinite(F1)) {  // zero fission integral -> degenerate
    if (threadIdx.x == 0) {
      atomicOr(flags, FLAG_DEGENERATE);
      k[b] = __longlong_as_double(0x7ff8000000000000ll);
      active[b] = 0;
      outer[b] = outer_it;
    }
    return;
  }
  const double kb = k[b], k_new = kb * F1;
  double num = 0.0, den = 0.0;
  for (size_t i = threadIdx.x; i < GN; i += HY_THREADS) {
    const double pn = p[i] / F1;
    p[i] = pn;
    const double d = pn - old[b * GN + i];
    if (norm == 0) {
      num = fmax(num, fabs(d));
      den = fmax(den, fabs(pn));
    } else {
      num = fma(d, d, num);
      den = fma(pn, pn, den);
    }
  }
  if (norm == 0) {
    num = hy_block_max(num, sh);
    den = hy_block_max(den, sh);
  } else {
    num = hy_block_sum(num, sh);
    den = hy_block_sum(den, sh);
  }
  if (threadIdx.x == 0) {
    const double dphi = snop_dev::rel_change(num, den, norm);
    const double dk = fabs(k_new - kb) / fabs(k_new);
    k[b] = k_new;
    outer[b] = outer_it;
    if (dk < tol_k && dphi < tol_phi) {
      active[b] = 0;
      conv[b] = 1;
    } else {
      atomicAdd(n_active, 1);
    }
  }
}

}  // namespace

namespace snop_impl {
snop_status launch_power_iteration_big(Ctx& ctx, const snop_grid& grid, int order, int B, int G, const double* st,
                                       const double* ss0, const double* ss1, const double* nsf, const double* chi,
                                       const snop_solver_config& cfg, const double* k0, const double* phi0, double* k,
                                       double* phi, int32_t* outer, int64_t* inner, uint8_t* conv) {
  if (B == 0) return SNOP_OK;
  const int Nc = grid.n_cells;
  const size_t N = (size_t)B * Nc, GNB = N * G;
  const double dx = grid.length_cm / Nc;
  auto dslot = [&](int i, size_t n) { return static_cast<double*>(ctx.slot(i, n * sizeof(double))); };
  double *old = dslot(100, GNB), *fiss = dslot(101, N), *qext = dslot(102, N), *stg = dslot(103, N);
  double *ssg = dslot(104, N), *s1g = ss1 ? dslot(105, N) : nullptr, *phig = dslot(106, N), *solved = dslot(107, N);
  uint8_t* active = static_cast<uint8_t*>(ctx.slot(108, (size_t)B));
  int32_t* sit = static_cast<int32_t*>(ctx.slot(109, (size_t)B * sizeof(int32_t)));
  uint8_t* scv = static_cast<uint8_t*>(ctx.slot(110, (size_t)B));
  int* cnt = static_cast<int*>(ctx.slot(111, 2 * sizeof(int)));
  if (!old || !fiss || !qext || !stg || !ssg || (ss1 && !s1g) || !phig || !solved || !active || !sit || !scv || !cnt)
    return cuda_status("workspace", cudaErrorMemoryAllocation);
  int *n_active = cnt, *outer_done = cnt + 1;
  // chi is per instance [B][G]; the gather kernels read it as such
  pi_big_init<<<B, HY_THREADS, 0, ctx.stream>>>(G, Nc, dx, st, nsf, k0, phi0, phi, k, active, conv, outer, inner,
                                               ctx.d_flags);
  ctx.launches++;
  cudaMemsetAsync(outer_done, 0, sizeof(int), ctx.stream);
  snop_solver_config icfg = cfg;  // inner solves: the flux tolerance, warm-started
  auto body = [&](cudaGraphConditionalHandle h) -> snop_status {
    const cudaStream_t cs = ctx.stream;
    const int64_t l0 = ctx.launches;
    hy_outer_begin<<<B, HY_THREADS, 0, cs>>>(G, Nc, nsf, phi, old, fiss, active);
    ctx.launches++;
    for (int g = 0; g < G; ++g) {
      hy_group_in<<<B, HY_THREADS, 0, cs>>>(g, G, Nc, chi, k, st, ss0, ss1, phi, fiss, qext, stg, ssg, s1g, phig);
      ctx.launches++;
      SNOP_TRY(launch_source_iteration(ctx, grid, order, B, stg, ssg, s1g, qext, icfg, phig, solved, nullptr, sit,
                                       scv, nullptr, nullptr, active));
      pi_big_group_out<<<B, HY_THREADS, 0, cs>>>(g, G, Nc, solved, phi, active, sit, inner);
      ctx.launches++;
    }
    cudaMemsetAsync(n_active, 0, sizeof(int), cs);
    pi_big_outer_end<<<B, HY_THREADS, 0, cs>>>(G, Nc, dx, outer_done, cfg.tolerance_k, cfg.tolerance_phi, cfg.norm,
                                               nsf, phi, old, k, active, conv, outer, n_active, ctx.d_flags);
    const int nb = (int)(ctx.launches - l0) + 2;
    loop_ctl<<<1, 1, 0, cs>>>(h, outer_done, n_active, cfg.max_outer, nb, ctx.d_loop_launches);
    return cuda_status("power iteration (streaming)", cudaGetLastError());
  };
  uint64_t bits[3];
  std::memcpy(&bits[0], &cfg.tolerance, 8);
  std::memcpy(&bits[1], &cfg.tolerance_k, 8);
  std::memcpy(&bits[2], &cfg.tolerance_phi, 8);
  const std::vector<uint64_t> key = {3, (uint64_t)order, (uint64_t)B, (uint64_t)G, (uint64_t)Nc,
                                     (uint64_t)(uintptr_t)st, (uint64_t)(uintptr_t)ss0, (uint64_t)(uintptr_t)ss1,
                                     (uint64_t)(uintptr_t)nsf, (uint64_t)(uintptr_t)chi, (uint64_t)(uintptr_t)k,
                                     (uint64_t)(uintptr_t)phi, (uint64_t)(uintptr_t)outer,
                                     (uint64_t)(uintptr_t)inner, (uint64_t)(uintptr_t)conv, bits[0], bits[1],
                                     bits[2], (uint64_t)cfg.max_outer, (uint64_t)cfg.max_inner, (uint64_t)cfg.norm,
                                     (uint64_t)cfg.bc_left, (uint64_t)cfg.bc_right,
                                     (uint64_t)std::llround(grid.length_cm * 1e12)};
  return device_loop(ctx, key, body);
}
}  // namespace snop_impl

extern "C" {


snop_status snop_deeponet_create(snop_ctx* ctx, const snop_grid* grid, double tstar, double sstar, int32_t act,
                                 int32_t nb, const int32_t* bs, const float* bp, int32_t nt, const int32_t* ts,
                                 const float* tp, int32_t has_bias0, float bias0, snop_op** out) {
  if (!out) return invalid("out is NULL");
  *out = nullptr;
  if (!ctx || !grid || !bs || !bp || !ts || !tp) return invalid("NULL argument");
  if (grid->n_cells < 1 || !(grid->length_cm > 0)) return invalid("bad grid");
  if (!valid_act(act)) return invalid("activation must be relu(0), tanh(1) or gelu(2)");
  if (nb < 2 || nt < 2) return invalid("networks need >= 2 layer sizes");
  if (bs[0] != grid->n_cells) return invalid("branch input width must equal n_cells (SPEC.md:321)");
  if (ts[0] != 1) return invalid("trunk input width must be 1 (position)");
  if (bs[nb - 1] != ts[nt - 1]) return invalid("branch/trunk output widths differ (SPEC.md:303)");
  for (int i = 0; i < nb; ++i) if (bs[i] < 1) return invalid("bad branch size");
  for (int i = 0; i < nt; ++i) if (ts[i] < 1) return invalid("bad trunk size");
  cudaSetDevice(ctx->device);
  auto* op = new snop_op;
  op->kind = 0;
  op->ctx = ctx;
  op->grid = *grid;
  op->tstar = tstar;
  op->sstar = sstar;
  op->act = act;
  op->bsizes.assign(bs, bs + nb);
  op->tsizes.assign(ts, ts + nt);
  op->has_bias0 = has_bias0 != 0;
  op->bias0 = bias0;
  {
    const size_t nbp = dense_param_count(std::vector<int32_t>(bs, bs + nb));
    const size_t ntp = dense_param_count(std::vector<int32_t>(ts, ts + nt));
    op->host_params.assign(bp, bp + nbp);
    op->host_params.insert(op->host_params.end(), tp, tp + ntp);
  }
  size_t off = 0;
  for (int l = 0; l + 1 < nb; ++l) {
    const size_t nw = (size_t)bs[l] * bs[l + 1];
    op->bW.push_back(op->upload(bp + off, nw));
    off += nw;
    op->bb.push_back(op->upload(bp + off, (size_t)bs[l + 1]));
    off += bs[l + 1];
  }
  std::vector<float*> tW, tb;
  off = 0;
  for (int l = 0; l + 1 < nt; ++l) {
    const size_t nw = (size_t)ts[l] * ts[l + 1];
    tW.push_back(op->upload(tp + off, nw));
    off += nw;
    tb.push_back(op->upload(tp + off, (size_t)ts[l + 1]));
    off += ts[l + 1];
  }
  // trunk evaluated once at the cell centres (fp32 inputs, as the oracle)
  const int n = grid->n_cells, p = ts[nt - 1];
  std::vector<float> xs(n);
  for (int i = 0; i < n; ++i) xs[i] = (float)((i + 0.5) * (grid->length_cm / n));
  float* xd = op->upload(xs.data(), n);
  int maxw = 0;
  for (int s : op->tsizes) maxw = std::max(maxw, s);
  float* t0 = op->upload<float>(nullptr, (size_t)n * maxw);
  float* t1 = op->upload<float>(nullptr, (size_t)n * maxw);
  op->trunk_out = op->upload<float>(nullptr, (size_t)n * p);
  if (has_bias0) {
    std::vector<float> bv(n, bias0);
    op->bias0_vec = op->upload(bv.data(), n);
  }
  float* res = nullptr;
  snop_status st = dense_forward(*ctx, n, op->tsizes, tW, tb, act, xd, t0, t1, &res);
  if (st == SNOP_OK)
    st = cuda_status("trunk copy", cudaMemcpyAsync(op->trunk_out, res, (size_t)n * p * sizeof(float),
                                                   cudaMemcpyDeviceToDevice, ctx->stream));
  if (st == SNOP_OK) st = cuda_status("trunk", cudaStreamSynchronize(ctx->stream));
  for (float* w : op->bW) if (!w) st = cuda_status("upload", cudaErrorMemoryAllocation);
  if (st != SNOP_OK) {
    delete op;
    return st;
  }
  *out = op;
  return SNOP_OK;
}

snop_status snop_fno_create(snop_ctx* ctx, const snop_grid* grid, double tstar, double sstar, int32_t act,
                            int32_t width, int32_t modes, int32_t layers, int32_t hidden, const float* p,
                            snop_op** out) {
  if (!out) return invalid("out is NULL");
  *out = nullptr;
  if (!ctx || !grid || !p) return invalid("NULL argument");
  const int n = grid->n_cells;
  if (n < 2 || !(grid->length_cm > 0)) return invalid("bad grid");
  if (!valid_act(act)) return invalid("activation must be relu(0), tanh(1) or gelu(2)");
  if (width < 1 || width > 256 || layers < 0 || hidden < 1 || modes < 1)
    return invalid("bad FNO architecture");
  if (modes > n / 2 + 1) return invalid("modes must be <= floor(n_cells/2)+1 (SPEC.md:309)");
  cudaSetDevice(ctx->device);
  auto* op = new snop_op;
  op->kind = 1;
  op->ctx = ctx;
  op->grid = *grid;
  op->tstar = tstar;
  op->sstar = sstar;
  op->act = act;
  op->width = width;
  op->modes = modes;
  op->layers = layers;
  op->hidden = hidden;
  op->host_params.assign(p, p + fno_param_count(width, modes, layers, hidden));
  const size_t C = width, M = modes;
  op->lift_W = op->upload(p, C * 2);
  p += C * 2;
  op->lift_b = op->upload(p, C);
  p += C;
  for (int l = 0; l < layers; ++l) {
    op->Rr.push_back(op->upload(p, M * C * C));
    op->Ri.push_back(op->upload(p + M * C * C, M * C * C));
    {  // U_re = V_re Rr - V_im Ri, U_im = V_re Ri + V_im Rr per mode, as B operands [o][c]
      const float *rr = p, *ri = p + M * C * C;
      std::vector<float> mb(4 * M * C * C);
      for (size_t m = 0; m < M; ++m)
        for (size_t c = 0; c < C; ++c)
          for (size_t o = 0; o < C; ++o) {
            const size_t src = (m * C + c) * C + o, dst = (m * C + o) * C + c;
            mb[0 * M * C * C + dst] = rr[src];
            mb[1 * M * C * C + dst] = -ri[src];
            mb[2 * M * C * C + dst] = ri[src];
            mb[3 * M * C * C + dst] = rr[src];
          }
      op->mixB.push_back(op->upload(mb.data(), mb.size()));
      op->mixB_lo.push_back(op->upload_lo(mb.data(), mb.size()));
    }
    p += 2 * M * C * C;
    op->W.push_back(op->upload(p, C * C));
    p += C * C;
    op->b.push_back(op->upload(p, C));
    p += C;
  }
  op->P1W = op->upload(p, (size_t)hidden * C);
  op->P1W_lo = op->upload_lo(p, (size_t)hidden * C);
  p += (size_t)hidden * C;
  op->P1b = op->upload(p, hidden);
  p += hidden;
  op->P2W = op->upload(p, hidden);
  p += hidden;
  op->p2b_host = p[0];
  op->P2b = op->upload(p, 1);
  // truncated real DFT matrices (exact index reduction), SURVEY §9 #9 conventions
  std::vector<float> F(2 * M * n), G((size_t)n * 2 * M), xs(n);
  const double two_pi = 6.283185307179586476925286766559;
  for (size_t m = 0; m < M; ++m)
    for (int i = 0; i < n; ++i) {
      const double ang = two_pi * (double)((m * (size_t)i) % (size_t)n) / n;
      F[m * n + i] = (float)std::cos(ang);
      F[(M + m) * n + i] = (float)-std::sin(ang);
      const bool nyq = 2 * m == (size_t)n;
      const double wr = (m == 0 || nyq) ? 1.0 : 2.0;
      const double wi = (m == 0 || nyq) ? 0.0 : 2.0;
      G[(size_t)i * 2 * M + m] = (float)(wr * std::cos(ang) / n);
      G[(size_t)i * 2 * M + M + m] = (float)(-wi * std::sin(ang) / n);
    }
  for (int i = 0; i < n; ++i) xs[i] = (float)((i + 0.5) * (grid->length_cm / n));
  op->F = op->upload(F.data(), F.size());
  op->Ginv = op->upload(G.data(), G.size());
  op->Ginv_lo = op->upload_lo(G.data(), G.size());
  op->F_lo = op->upload_lo(F.data(), F.size());
  {
    std::vector<float> FTh((size_t)n * 2 * M);
    for (size_t m = 0; m < 2 * M; ++m)
      for (int i = 0; i < n; ++i) FTh[(size_t)i * 2 * M + m] = F[m * n + i];
    op->FT = op->upload(FTh.data(), FTh.size());
  }
  op->xc = op->upload(xs.data(), n);
  if (layers >= 1) {
    // Layer 0 acts on V = lift(S, x) = Wl0 S + Wl1 x + bl, which is affine in the source, so its
    // forward DFT is Wl0 S^ + Wl1 x^ + bl 1^ and (by linearity) its spectral mixing is
    // U0 = S^ P + Q and its W path is Aw S + Bw x + Cw. Constants in fp64 from the fp32 parameters.
    const float* hp = op->host_params.data();
    const float *Wl = hp, *bl = hp + 2 * C, *R0r = bl + C, *R0i = R0r + M * C * C;
    const float *W0 = R0i + M * C * C, *b0 = W0 + C * C;
    std::vector<double> xh(2 * M, 0.0), oh(2 * M, 0.0);
    for (size_t m = 0; m < 2 * M; ++m)
      for (int i = 0; i < n; ++i) {
        xh[m] += (double)F[m * n + i] * (double)xs[i];
        oh[m] += (double)F[m * n + i];
      }
    std::vector<float> P(2 * M * C), Q(2 * M * C), Aw(C), Bw(C), Cw(C);
    for (size_t m = 0; m < M; ++m)
      for (size_t o = 0; o < C; ++o) {
        double pr = 0, pi = 0, qr = 0, qi = 0;
        for (size_t c = 0; c < C; ++c) {
          const double rr = R0r[(m * C + c) * C + o], ri = R0i[(m * C + c) * C + o];
          const double w0 = Wl[2 * c], w1 = Wl[2 * c + 1], bc = bl[c];
          const double zr = w1 * xh[m] + bc * oh[m], zi = w1 * xh[M + m] + bc * oh[M + m];
          pr += rr * w0;
          pi += ri * w0;
          qr += rr * zr - ri * zi;
          qi += rr * zi + ri * zr;
        }
        P[m * C + o] = (float)pr;
        P[(M + m) * C + o] = (float)pi;
        Q[m * C + o] = (float)qr;
        Q[(M + m) * C + o] = (float)qi;
      }
    for (size_t o = 0; o < C; ++o) {
      double a = 0, bb = 0, cc = b0[o];
      for (size_t c = 0; c < C; ++c) {
        a += (double)W0[o * C + c] * Wl[2 * c];
        bb += (double)W0[o * C + c] * Wl[2 * c + 1];
        cc += (double)W0[o * C + c] * bl[c];
      }
      Aw[o] = (float)a;
      Bw[o] = (float)bb;
      Cw[o] = (float)cc;
    }
    op->l0_P = op->upload(P.data(), P.size());
    op->l0_Q = op->upload(Q.data(), Q.size());
    op->l0_A = op->upload(Aw.data(), C);
    op->l0_B = op->upload(Bw.data(), C);
    op->l0_C = op->upload(Cw.data(), C);
  }
  if (!op->F || !op->Ginv || !op->xc || !op->P2b || (layers >= 1 && (!op->l0_P || !op->l0_Q || !op->l0_C))) {
    delete op;
    return cuda_status("FNO upload", cudaErrorMemoryAllocation);
  }
  *out = op;
  return SNOP_OK;
}

snop_status snop_exact_operator_create(snop_ctx* ctx, const snop_grid* grid, int32_t order, double tstar,
                                       double sstar, const snop_solver_config* cfg, snop_op** out) {
  if (!out) return invalid("out is NULL");
  *out = nullptr;
  if (!ctx || !grid || !cfg) return invalid("NULL argument");
  if (grid->n_cells < 1 || grid->n_cells > kMaxCells || !(grid->length_cm > 0)) return invalid("bad grid");
  if (order < 2 || order > 128 || order % 2) return invalid("quadrature order must be even in [2,128]");
  if (!(tstar > 0.0)) return invalid("reference sigma_t must be positive");
  auto* op = new snop_op;
  op->kind = 2;
  op->ctx = ctx;
  op->grid = *grid;
  op->order = order;
  op->tstar = tstar;
  op->sstar = sstar;
  op->cfg = *cfg;
  *out = op;
  return SNOP_OK;
}

snop_status snop_op_save(const snop_op* op, const char* path) {
  if (!op) return invalid("op is NULL");
  ModelFile m;
  m.grid = op->grid;
  m.tstar = op->tstar;
  m.sstar = op->sstar;
  m.act = op->act;
  m.params = op->host_params;
  if (op->kind == 0) {
    m.arch = SNOP_ARCH_DEEPONET;
    m.bs.assign(op->bsizes.begin(), op->bsizes.end());
    m.ts.assign(op->tsizes.begin(), op->tsizes.end());
    m.has_bias0 = op->has_bias0;
    m.bias0 = op->bias0;
  } else if (op->kind == 1) {
    m.arch = SNOP_ARCH_FNO;
    m.width = op->width;
    m.modes = op->modes;
    m.layers = op->layers;
    m.hidden = op->hidden;
  } else {
    return invalid("the exact operator has no weights to save");
  }
  return write_model(path, m);
}

snop_status snop_op_load(snop_ctx* ctx, const char* path, snop_op** out) {
  if (!out) return invalid("out is NULL");
  *out = nullptr;
  if (!ctx) return invalid("ctx is NULL");
  ModelFile m;
  SNOP_TRY(read_model(path, m));
  if (m.arch == SNOP_ARCH_DEEPONET) {
    const size_t nbp = dense_param_count(m.bs);
    return snop_deeponet_create(ctx, &m.grid, m.tstar, m.sstar, m.act, (int32_t)m.bs.size(), m.bs.data(),
                                m.params.data(), (int32_t)m.ts.size(), m.ts.data(), m.params.data() + nbp,
                                m.has_bias0 ? 1 : 0, m.bias0, out);
  }
  return snop_fno_create(ctx, &m.grid, m.tstar, m.sstar, m.act, m.width, m.modes, m.layers, m.hidden,
                         m.params.data(), out);
}

snop_status snop_op_destroy(snop_op* op) {
  if (op) {
    if (op->ctx) {
      cudaSetDevice(op->ctx->device);
      cudaStreamSynchronize(op->ctx->stream);
    }
    delete op;
  }
  return SNOP_OK;
}

snop_status snop_op_predict(snop_ctx* ctx, snop_op* op, int32_t memspace, int32_t batch, const double* source,
                            double* out) {
  SNOP_TRY(check_op(ctx, op));
  if (batch < 0) return invalid("batch must be >= 0");
  if (batch == 0) return SNOP_OK;
  if (!source || !out) return invalid("NULL array");
  cudaSetDevice(ctx->device);
  const size_t N = (size_t)batch * op->grid.n_cells;
  if (memspace == SNOP_MEM_DEVICE) return op_predict_dev(*ctx, *op, batch, source, out);
  if (memspace != SNOP_MEM_HOST) return invalid("memspace must be HOST(0) or DEVICE(1)");
  double *s, *o;
  SNOP_TRY(stage(*ctx, 60, source, N, &s));
  o = static_cast<double*>(ctx->slot(61, N * sizeof(double)));
  if (!o) return cuda_status("cudaMalloc", cudaErrorMemoryAllocation);
  SNOP_TRY(op_predict_dev(*ctx, *op, batch, s, o));
  SNOP_TRY(unstage(*ctx, out, o, N));
  return drain(*ctx);
}

snop_status snop_recast_fixed_point(snop_ctx* ctx, snop_op* op, int32_t memspace, int32_t batch, const double* source,
                                    const double* sigma_t, const double* sigma_s0, double tol, int32_t max_it,
                                    int32_t norm, const double* initial_phi, double* phi_out, int32_t* iterations,
                                    int32_t* status) {
  SNOP_TRY(check_op(ctx, op));
  if (batch < 0 || max_it < 0) return invalid("batch and max iterations must be >= 0");
  if (!(tol > 0.0)) return invalid("recast tolerance must be positive");
  if (norm != 0 && norm != 1) return invalid("norm must be rel-Linf(0) or rel-L2(1)");
  if (batch == 0) return SNOP_OK;
  if (!source || !sigma_t || !sigma_s0 || !phi_out || !iterations || !status) return invalid("NULL array");
  cudaSetDevice(ctx->device);
  const size_t N = (size_t)batch * op->grid.n_cells;
  if (memspace == SNOP_MEM_DEVICE)
    return recast_fp_dev(*ctx, *op, batch, source, sigma_t, sigma_s0, tol, max_it, norm, initial_phi, phi_out,
                         iterations, status);
  if (memspace != SNOP_MEM_HOST) return invalid("memspace must be HOST(0) or DEVICE(1)");
  double *S, *st, *ss, *p0, *phi;
  int32_t *it, *stt;
  SNOP_TRY(stage(*ctx, 62, source, N, &S));
  SNOP_TRY(stage(*ctx, 63, sigma_t, N, &st));
  SNOP_TRY(stage(*ctx, 64, sigma_s0, N, &ss));
  SNOP_TRY(stage(*ctx, 65, initial_phi, N, &p0));
  phi = static_cast<double*>(ctx->slot(66, N * sizeof(double)));
  it = static_cast<int32_t*>(ctx->slot(67, (size_t)batch * sizeof(int32_t)));
  stt = static_cast<int32_t*>(ctx->slot(68, (size_t)batch * sizeof(int32_t)));
  if (!phi || !it || !stt) return cuda_status("cudaMalloc", cudaErrorMemoryAllocation);
  SNOP_TRY(recast_fp_dev(*ctx, *op, batch, S, st, ss, tol, max_it, norm, p0, phi, it, stt));
  SNOP_TRY(unstage(*ctx, phi_out, phi, N));
  SNOP_TRY(unstage(*ctx, iterations, it, (size_t)batch));
  SNOP_TRY(unstage(*ctx, status, stt, (size_t)batch));
  return drain(*ctx);
}

snop_status snop_precondition_fixed_source(snop_ctx* ctx, snop_op* op, int32_t memspace, int32_t order,
                                           int32_t batch, const double* sigma_t, const double* sigma_s0,
                                           const double* sigma_s1, const double* source, double rtol, int32_t rmax,
                                           const snop_solver_config* cfg, double* phi_out, int32_t* piters,
                                           int32_t* rstatus, int32_t* riters, uint8_t* conv) {
  SNOP_TRY(check_op(ctx, op));
  if (!cfg) return invalid("config is NULL");
  if (order < 2 || order > 128 || order % 2) return invalid("quadrature order must be even in [2,128]");
  if (batch < 0 || rmax < 0 || !(rtol > 0.0)) return invalid("bad batch / recast settings");
  if (op->grid.n_cells > kMaxCells) return invalid("n_cells exceeds the per-CTA sweep limit");
  if (batch == 0) return SNOP_OK;
  if (!sigma_t || !sigma_s0 || !source || !phi_out || !piters || !rstatus || !riters || !conv)
    return invalid("NULL array");
  cudaSetDevice(ctx->device);
  const size_t N = (size_t)batch * op->grid.n_cells;
  const double *st = sigma_t, *ss = sigma_s0, *s1 = sigma_s1, *S = source;
  double* phi = phi_out;
  int32_t *pi = piters, *rs = rstatus, *ri = riters;
  uint8_t* cv = conv;
  const bool host = memspace == SNOP_MEM_HOST;
  if (!host && memspace != SNOP_MEM_DEVICE) return invalid("memspace must be HOST(0) or DEVICE(1)");
  if (host) {
    double *a, *b, *c, *d;
    SNOP_TRY(stage(*ctx, 62, sigma_t, N, &a));
    SNOP_TRY(stage(*ctx, 63, sigma_s0, N, &b));
    SNOP_TRY(stage(*ctx, 64, sigma_s1, N, &c));
    SNOP_TRY(stage(*ctx, 65, source, N, &d));
    st = a; ss = b; s1 = c; S = d;
    phi = static_cast<double*>(ctx->slot(66, N * sizeof(double)));
    pi = static_cast<int32_t*>(ctx->slot(67, (size_t)batch * sizeof(int32_t)));
    rs = static_cast<int32_t*>(ctx->slot(68, (size_t)batch * sizeof(int32_t)));
    ri = static_cast<int32_t*>(ctx->slot(69, (size_t)batch * sizeof(int32_t)));
    cv = static_cast<uint8_t*>(ctx->slot(70, (size_t)batch));
    if (!phi || !pi || !rs || !ri || !cv) return cuda_status("cudaMalloc", cudaErrorMemoryAllocation);
  }
  double* phi_no = static_cast<double*>(ctx->slot(71, N * sizeof(double)));
  if (!phi_no) return cuda_status("cudaMalloc", cudaErrorMemoryAllocation);
  SNOP_TRY(recast_fp_dev(*ctx, *op, batch, S, st, ss, rtol, rmax, cfg->norm, nullptr, phi_no, pi, rs));
  SNOP_TRY(launch_source_iteration(*ctx, op->grid, order, batch, st, ss, s1, S, *cfg, phi_no, phi, nullptr, ri, cv));
  if (host) {
    SNOP_TRY(unstage(*ctx, phi_out, phi, N));
    SNOP_TRY(unstage(*ctx, piters, pi, (size_t)batch));
    SNOP_TRY(unstage(*ctx, rstatus, rs, (size_t)batch));
    SNOP_TRY(unstage(*ctx, riters, ri, (size_t)batch));
    SNOP_TRY(unstage(*ctx, conv, cv, (size_t)batch));
    return drain(*ctx);
  }
  return SNOP_OK;
}

static snop_status hybrid_eigen(snop_ctx* ctx, snop_op* op, int algorithm, int32_t memspace, int32_t order,
                                int32_t batch, int32_t G, const double* sigma_t, const double* sigma_s0,
                                const double* sigma_s1, const double* nu_sigma_f, const double* chi,
                                const snop_solver_config* cfg, double rtol, int32_t rmax, double* k_out,
                                double* phi_out, double* stage1_k, int32_t* stage1_outer, int64_t* stage1_inner,
                                int32_t* stage2_outer, int64_t* stage2_inner, uint8_t* converged, uint8_t* fallback,
                                bool stage1_only = false) {
  SNOP_TRY(check_op(ctx, op));
  if (!cfg) return invalid("config is NULL");
  if (order < 2 || order > 128 || order % 2) return invalid("quadrature order must be even in [2,128]");
  if (!(cfg->tolerance > 0.0) || !(cfg->tolerance_k > 0.0) || !(cfg->tolerance_phi > 0.0) || cfg->max_inner < 1 ||
      cfg->max_outer < 1)
    return invalid("config: tolerances must be positive and iteration limits >= 1");
  if (batch < 0 || rmax < 0 || !(rtol > 0.0)) return invalid("bad batch / recast settings");
  if (G < 1 || G > 64) return invalid("n_groups must be in [1,64]");
  if (op->grid.n_cells > kMaxCells) return invalid("n_cells exceeds the per-CTA sweep limit");
  if (batch == 0) return SNOP_OK;
  if (!sigma_t || !sigma_s0 || !nu_sigma_f || !chi || !k_out || !phi_out || !stage1_k || !stage1_outer ||
      !stage1_inner || (!stage1_only && (!stage2_outer || !stage2_inner)) || !converged || !fallback)
    return invalid("NULL array");
  const bool host = memspace == SNOP_MEM_HOST;
  if (!host && memspace != SNOP_MEM_DEVICE) return invalid("memspace must be HOST(0) or DEVICE(1)");
  cudaSetDevice(ctx->device);
  const size_t B = batch, n = B * G * op->grid.n_cells;
  const double *st = sigma_t, *ss = sigma_s0, *s1 = sigma_s1, *nsf = nu_sigma_f, *ch = chi;
  HybridOut o{k_out, phi_out, stage1_k, stage1_outer, stage2_outer, stage1_inner, stage2_inner, converged, fallback};
  if (host) {
    double *a, *b, *c, *d, *e;
    SNOP_TRY(stage(*ctx, 100, sigma_t, n, &a));
    SNOP_TRY(stage(*ctx, 101, sigma_s0, n * G, &b));
    SNOP_TRY(stage(*ctx, 102, sigma_s1, n, &c));
    SNOP_TRY(stage(*ctx, 103, nu_sigma_f, n, &d));
    SNOP_TRY(stage(*ctx, 104, chi, B * G, &e));
    st = a; ss = b; s1 = c; nsf = d; ch = e;
    o.k = static_cast<double*>(ctx->slot(105, B * sizeof(double)));
    o.phi = static_cast<double*>(ctx->slot(106, n * sizeof(double)));
    o.k1 = static_cast<double*>(ctx->slot(107, B * sizeof(double)));
    o.outer1 = static_cast<int32_t*>(ctx->slot(108, B * sizeof(int32_t)));
    o.outer2 = static_cast<int32_t*>(ctx->slot(109, B * sizeof(int32_t)));
    o.inner1 = static_cast<int64_t*>(ctx->slot(110, B * sizeof(int64_t)));
    o.inner2 = static_cast<int64_t*>(ctx->slot(111, B * sizeof(int64_t)));
    o.conv = static_cast<uint8_t*>(ctx->slot(112, B));
    o.fb = static_cast<uint8_t*>(ctx->slot(113, B));
    if (!o.k || !o.phi || !o.k1 || !o.outer1 || !o.outer2 || !o.inner1 || !o.inner2 || !o.conv || !o.fb)
      return cuda_status("cudaMalloc", cudaErrorMemoryAllocation);
  }
  SNOP_TRY(hybrid_eigen_dev(*ctx, *op, algorithm, order, batch, G, st, ss, s1, nsf, ch, *cfg, rtol, rmax, o,
                            stage1_only));
  if (!host) return SNOP_OK;
  SNOP_TRY(unstage(*ctx, k_out, o.k, B));
  SNOP_TRY(unstage(*ctx, phi_out, o.phi, n));
  if (stage1_k != k_out) SNOP_TRY(unstage(*ctx, stage1_k, o.k1, B));
  SNOP_TRY(unstage(*ctx, stage1_outer, o.outer1, B));
  SNOP_TRY(unstage(*ctx, stage1_inner, o.inner1, B));
  if (!stage1_only) {
    SNOP_TRY(unstage(*ctx, stage2_outer, o.outer2, B));
    SNOP_TRY(unstage(*ctx, stage2_inner, o.inner2, B));
  }
  SNOP_TRY(unstage(*ctx, converged, o.conv, B));
  SNOP_TRY(unstage(*ctx, fallback, o.fb, B));
  return drain(*ctx);
}

#define SNOP_HYBRID_ARGS                                                                                          \
  snop_ctx *ctx, snop_op *op, int32_t memspace, int32_t order, int32_t batch, int32_t n_groups,                   \
      const double *sigma_t, const double *sigma_s0, const double *sigma_s1, const double *nu_sigma_f,           \
      const double *chi, const snop_solver_config *cfg, double recast_tolerance, int32_t recast_max_iterations,   \
      double *k_out, double *phi_out, double *stage1_k, int32_t *stage1_outer, int64_t *stage1_inner,            \
      int32_t *stage2_outer, int64_t *stage2_inner, uint8_t *converged, uint8_t *fallback
#define SNOP_HYBRID_FWD                                                                                          \
  memspace, order, batch, n_groups, sigma_t, sigma_s0, sigma_s1, nu_sigma_f, chi, cfg, recast_tolerance,         \
      recast_max_iterations, k_out, phi_out, stage1_k, stage1_outer, stage1_inner, stage2_outer, stage2_inner,    \
      converged, fallback

// power_iteration with the operator as inner_solver: stage 1 of SP / CP on its own.
snop_status snop_power_iteration_operator_batched(
    snop_ctx* ctx, snop_op* op, int32_t inner_solver, int32_t memspace, int32_t order, int32_t batch,
    int32_t n_groups, const double* sigma_t, const double* sigma_s0, const double* sigma_s1,
    const double* nu_sigma_f, const double* chi, const snop_solver_config* cfg, double recast_tolerance,
    int32_t recast_max_iterations, double* k_out, double* phi_out, int32_t* outer_iterations,
    int64_t* inner_iterations, uint8_t* converged, uint8_t* diverged) {
  if (inner_solver != SNOP_INNER_RECAST_FIXED_POINT && inner_solver != SNOP_INNER_PREDICT_REFINE)
    return invalid("inner_solver must be RECAST_FIXED_POINT(0) or PREDICT_REFINE(1)");
  return hybrid_eigen(ctx, op, inner_solver, memspace, order, batch, n_groups, sigma_t, sigma_s0, sigma_s1, nu_sigma_f,
                      chi, cfg, recast_tolerance, recast_max_iterations, k_out, phi_out, k_out, outer_iterations,
                      inner_iterations, nullptr, nullptr, converged, diverged, true);
}

snop_status snop_sp_eigen_batched(SNOP_HYBRID_ARGS) { return hybrid_eigen(ctx, op, 0, SNOP_HYBRID_FWD); }
snop_status snop_cp_eigen_batched(SNOP_HYBRID_ARGS) { return hybrid_eigen(ctx, op, 1, SNOP_HYBRID_FWD); }

}  // extern "C"
