// snop ORACLE — TEST INFRASTRUCTURE ONLY. extern "C" layer so pytest (ctypes) can drive the
// CPU restatement with exactly the argument layout of the product C-ABI (include/snop_cuda.h),
// host pointers only. Batched entry points parallelise over instances with the restated
// parallel_chunks (proj/core/include/snop/parallel.hpp:17-48): one chunk per instance, so
// results are bit-identical at any thread count.
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <memory>
#include <mutex>
#include <thread>
#include <string>

#include "../include/snop_cuda.h"
#include "snop_oracle.hpp"

using namespace snop::oracle;

namespace {
thread_local std::string g_err;

int map_exc() {
  try {
    throw;
  } catch (const DegenerateProblem& e) {
    g_err = e.what();
    return SNOP_DEGENERATE_PROBLEM;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return SNOP_NUMERICAL_ERROR;
  } catch (const InvalidArgument& e) {
    g_err = e.what();
    return SNOP_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SNOP_NUMERICAL_ERROR;
  }
}

SolverConfig to_cfg(const snop_solver_config* c) {
  SolverConfig s;
  s.tolerance = c->tolerance;
  s.tolerance_k = c->tolerance_k;
  s.tolerance_phi = c->tolerance_phi;
  s.max_inner = c->max_inner;
  s.max_outer = c->max_outer;
  s.left = static_cast<Boundary>(c->bc_left);
  s.right = static_cast<Boundary>(c->bc_right);
  s.norm = static_cast<Norm>(c->norm);
  return s;
}

DenseNetwork unpack_dense(int n_sizes, const int32_t* sizes, const float* params, Activation act) {
  DenseNetwork d;
  d.act = act;
  d.sizes.assign(sizes, sizes + n_sizes);
  std::size_t off = 0;
  for (int l = 0; l + 1 < n_sizes; ++l) {
    const std::size_t nw = (std::size_t)sizes[l] * sizes[l + 1];
    d.W.emplace_back(params + off, params + off + nw);
    off += nw;
    d.b.emplace_back(params + off, params + off + sizes[l + 1]);
    off += sizes[l + 1];
  }
  return d;
}

struct OracleOp {
  int kind = 0;  // 0 deeponet, 1 fno, 2 exact
  Grid1D grid;
  double tstar = 1.0, sstar = 0.5;
  DeepONet don;
  FNO fno;
  Quadrature quad;
  SolverConfig cfg;
  void predict(const double* s, double* out) const {
    if (kind == 0) {
      deeponet_predict(don, grid, s, out);
    } else if (kind == 1) {
      fno_predict(fno, grid, s, out);
    } else {
      const int n = grid.n_cells;
      std::vector<double> st(n, tstar), ss(n, sstar);
      std::fill(out, out + n, 0.0);
      source_iteration(grid, quad, st.data(), ss.data(), nullptr, s, cfg, out, nullptr);
    }
  }
};
}  // namespace

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }
unsigned oracle_hardware_threads(void) { return std::thread::hardware_concurrency(); }

int oracle_gauss_legendre(int32_t order, double* mu, double* w) {
  try {
    const Quadrature q = gauss_legendre(order);
    std::memcpy(mu, q.mu.data(), sizeof(double) * order);
    std::memcpy(w, q.w.data(), sizeof(double) * order);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

// The reference's own parallel_chunks partition, restated (golden-checked in tests).
void oracle_chunk_bounds(uint64_t n_items, uint64_t n_chunks, uint64_t* begins /* n_chunks+1 */) {
  if (n_chunks == 0 || n_chunks > n_items) n_chunks = n_items;
  const uint64_t base = n_items / n_chunks, extra = n_items % n_chunks;
  for (uint64_t c = 0; c <= n_chunks; ++c) begins[c] = c * base + std::min(c, extra);
}

void oracle_rng_stream(uint64_t seed, int32_t n_u64, uint64_t* u64, int32_t n_uniform, double* uni,
                       int32_t n_normal, double* nrm) {
  Rng a(seed);
  for (int i = 0; i < n_u64; ++i) u64[i] = a.next_u64();
  Rng b(seed);
  for (int i = 0; i < n_uniform; ++i) uni[i] = b.uniform();
  Rng c(seed);
  for (int i = 0; i < n_normal; ++i) nrm[i] = c.normal();
}

// sweep, batched: emission [B][Nc][N], psi_avg [B][N][Nc], net outflows [B].
int oracle_sweep_batched(const snop_grid* grid, int32_t order, int32_t batch, const double* st,
                         const double* emission, int32_t bc_left, int32_t bc_right, double* psi_avg,
                         double* out_left, double* out_right, int32_t n_threads) {
  try {
    const Grid1D g{grid->length_cm, grid->n_cells};
    const Quadrature q = gauss_legendre(order);
    const std::size_t Nc = g.n_cells, N = order;
    const Boundary bl = bc_left ? Boundary::Reflective : Boundary::Vacuum;
    const Boundary br = bc_right ? Boundary::Reflective : Boundary::Vacuum;
    std::string err;
    int code = 0;
    std::mutex mu;
    parallel_chunks(batch, batch, [&](std::size_t, std::size_t b0, std::size_t b1) {
      for (std::size_t b = b0; b < b1; ++b) {
        try {
          sweep(g, q, st + b * Nc, emission + b * Nc * N, bl, br, psi_avg + b * N * Nc,
                out_left ? out_left + b : nullptr, out_right ? out_right + b : nullptr);
        } catch (...) {
          std::lock_guard<std::mutex> lk(mu);
          code = map_exc();
          err = g_err;
        }
      }
    }, n_threads);
    if (code) { g_err = err; return code; }
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int oracle_source_iteration_batched(const snop_grid* grid, int32_t order, int32_t batch,
                                    const double* st, const double* ss0, const double* ss1,
                                    const double* src, const snop_solver_config* ccfg,
                                    const double* init_phi, double* phi_out, double* cur_out,
                                    int32_t* iters, uint8_t* conv, double* leak /* [B][2] or null */,
                                    int32_t n_threads) {
  try {
    const Grid1D g{grid->length_cm, grid->n_cells};
    const Quadrature q = gauss_legendre(order);
    const SolverConfig cfg = to_cfg(ccfg);
    const std::size_t Nc = g.n_cells;
    std::string err;
    int code = 0;
    std::mutex mu;
    parallel_chunks(batch, batch, [&](std::size_t, std::size_t b0, std::size_t b1) {
      for (std::size_t b = b0; b < b1; ++b) {
        try {
          double* phi = phi_out + b * Nc;
          if (init_phi) std::memcpy(phi, init_phi + b * Nc, sizeof(double) * Nc);
          else std::fill(phi, phi + Nc, 0.0);
          const SIResult r = source_iteration(g, q, st + b * Nc, ss0 + b * Nc, ss1 ? ss1 + b * Nc : nullptr,
                                              src + b * Nc, cfg, phi, cur_out ? cur_out + b * Nc : nullptr);
          iters[b] = r.iterations;
          conv[b] = r.converged ? 1 : 0;
          if (leak) { leak[2 * b] = r.out_left; leak[2 * b + 1] = r.out_right; }
        } catch (...) {
          std::lock_guard<std::mutex> lk(mu);
          code = map_exc();
          err = g_err;
        }
      }
    }, n_threads);
    if (code) { g_err = err; return code; }
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int oracle_power_iteration_batched(const snop_grid* grid, int32_t order, int32_t batch, int32_t G,
                                   const double* st, const double* ss0, const double* ss1, const double* nsf,
                                   const double* chi, const snop_solver_config* ccfg, const double* init_k,
                                   const double* init_phi, double* k_out, double* phi_out, int32_t* outer,
                                   int64_t* inner, uint8_t* conv, int32_t n_threads) {
  try {
    const Grid1D g{grid->length_cm, grid->n_cells};
    const Quadrature q = gauss_legendre(order);
    const SolverConfig cfg = to_cfg(ccfg);
    const std::size_t Nc = g.n_cells, GN = (std::size_t)G * Nc;
    std::string err;
    int code = 0;
    std::mutex mu;
    parallel_chunks(batch, batch, [&](std::size_t, std::size_t b0, std::size_t b1) {
      for (std::size_t b = b0; b < b1; ++b) {
        try {
          MGView m;
          m.G = G;
          m.sigma_t = st + b * GN;
          m.sigma_s0 = ss0 + b * GN * G;
          m.sigma_s1 = ss1 ? ss1 + b * GN : nullptr;
          m.nu_sigma_f = nsf + b * GN;
          m.chi = chi + b * G;
          double* phi = phi_out + b * GN;
          if (init_phi) std::memcpy(phi, init_phi + b * GN, sizeof(double) * GN);
          else std::fill(phi, phi + GN, 1.0);  // SPEC.md:209 flat flux
          const EigenResult r = power_iteration(g, q, m, cfg, phi, true, init_k ? init_k[b] : 1.0, nullptr);
          k_out[b] = r.k;
          outer[b] = r.outer;
          inner[b] = r.inner;
          conv[b] = r.converged ? 1 : 0;
        } catch (...) {
          std::lock_guard<std::mutex> lk(mu);
          code = map_exc();
          err = g_err;
        }
      }
    }, n_threads);
    if (code) { g_err = err; return code; }
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int oracle_infinite_medium_k(int32_t G, const double* st, const double* ss0, const double* nsf,
                             const double* chi, double* k) {
  try {
    *k = infinite_medium_k(G, st, ss0, nsf, chi);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int oracle_recast_source(int32_t batch, int32_t n, const double* S, const double* phi, const double* st,
                         const double* ss0, double tstar, double sstar, double* out) {
  for (int b = 0; b < batch; ++b)
    recast_source(n, S + (std::size_t)b * n, phi + (std::size_t)b * n, st + (std::size_t)b * n,
                  ss0 + (std::size_t)b * n, tstar, sstar, out + (std::size_t)b * n);
  return 0;
}

void* oracle_deeponet_create(const snop_grid* grid, double tstar, double sstar, int32_t act,
                             int32_t nb, const int32_t* bs, const float* bp, int32_t nt, const int32_t* ts,
                             const float* tp, int32_t has_bias0, float bias0) {
  auto* op = new OracleOp;
  op->kind = 0;
  op->grid = Grid1D{grid->length_cm, grid->n_cells};
  op->tstar = tstar;
  op->sstar = sstar;
  op->don.branch = unpack_dense(nb, bs, bp, static_cast<Activation>(act));
  op->don.trunk = unpack_dense(nt, ts, tp, static_cast<Activation>(act));
  op->don.has_bias0 = has_bias0 != 0;
  op->don.bias0 = bias0;
  return op;
}

void* oracle_fno_create(const snop_grid* grid, double tstar, double sstar, int32_t act, int32_t width,
                        int32_t modes, int32_t layers, int32_t hidden, const float* p) {
  auto* op = new OracleOp;
  op->kind = 1;
  op->grid = Grid1D{grid->length_cm, grid->n_cells};
  op->tstar = tstar;
  op->sstar = sstar;
  FNO& f = op->fno;
  f.width = width;
  f.modes = modes;
  f.layers = layers;
  f.proj_hidden = hidden;
  f.act = static_cast<Activation>(act);
  const std::size_t C = width, M = modes;
  auto take = [&](std::size_t n) { std::vector<float> v(p, p + n); p += n; return v; };
  f.lift_W = take(C * 2);
  f.lift_b = take(C);
  for (int l = 0; l < layers; ++l) {
    f.R_re.push_back(take(M * C * C));
    f.R_im.push_back(take(M * C * C));
    f.W.push_back(take(C * C));
    f.b.push_back(take(C));
  }
  f.P1_W = take((std::size_t)hidden * C);
  f.P1_b = take(hidden);
  f.P2_W = take(hidden);
  f.P2_b = take(1);
  return op;
}

// load_model: streaming restatement of the reader side of the reference's
// binary container (binary_io.cpp:12-17 FNV-1a-64 running hash; :88-141 little-endian reads,
// truncation error, trailing-digest verify) over the record of csrc/model_io.h.
namespace {
struct IoFail : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StreamReader {
  std::FILE* f = nullptr;
  std::uint64_t h = 0xcbf29ce484222325ull;
  ~StreamReader() { if (f) std::fclose(f); }
  void bytes(unsigned char* p, std::size_t n) {
    if (std::fread(p, 1, n, f) != n) throw IoFail("unexpected end of file (truncated?)");
    for (std::size_t i = 0; i < n; ++i) h = (h ^ p[i]) * 0x100000001b3ull;
  }
  std::uint64_t uint(int n) {
    unsigned char b[8];
    bytes(b, n);
    std::uint64_t v = 0;
    for (int i = n - 1; i >= 0; --i) v = (v << 8) | b[i];
    return v;
  }
  double f64() {
    const std::uint64_t u = uint(8);
    double d;
    std::memcpy(&d, &u, 8);
    return d;
  }
  std::string str() {
    const std::uint64_t n = uint(4);
    if (n > 4096) throw IoFail("string length implausible");
    std::string s(n, '\0');
    bytes(reinterpret_cast<unsigned char*>(s.data()), n);
    return s;
  }
  void verify() {
    const std::uint64_t expect = h;
    unsigned char b[8];
    if (std::fread(b, 1, 8, f) != 8) throw IoFail("checksum missing (truncated file)");
    std::uint64_t v = 0;
    for (int i = 7; i >= 0; --i) v = (v << 8) | b[i];
    if (v != expect) throw IoFail("checksum mismatch");
    if (std::fgetc(f) != EOF) throw IoFail("trailing bytes after checksum");
  }
};
}  // namespace

int oracle_model_load(const char* path, void** out) {
  *out = nullptr;
  try {
    StreamReader r;
    r.f = std::fopen(path, "rb");
    if (!r.f) throw IoFail("cannot open");
    if (r.str() != "SNOP-MODEL") throw IoFail("bad magic");
    if (r.uint(4) != 1) throw IoFail("version mismatch");
    const std::string arch = r.str();
    snop_grid g{};
    g.length_cm = r.f64();
    g.n_cells = (int32_t)r.uint(8);
    const double tstar = r.f64(), sstar = r.f64();
    const int act = (int)r.uint(4);
    std::vector<int32_t> bs, ts;
    bool hb = false;
    double b0 = 0.0;
    std::uint64_t arch_dims[4] = {0, 0, 0, 0};
    if (arch == "deeponet") {
      for (auto* v : {&bs, &ts}) {
        const std::uint64_t n = r.uint(4);
        if (n > 64) throw IoFail("implausible layer count");
        for (std::uint64_t i = 0; i < n; ++i) v->push_back((int32_t)r.uint(8));
      }
      hb = r.uint(1) != 0;
      b0 = r.f64();
    } else if (arch == "fno") {
      for (auto& d : arch_dims) d = r.uint(8);
    } else {
      throw IoFail("unknown architecture");
    }
    const std::uint64_t np = r.uint(8);
    if (np > (1ull << 32)) throw IoFail("implausible parameter count");
    std::vector<float> prm(np);
    for (auto& x : prm) x = (float)r.f64();
    r.verify();
    if (arch == "deeponet") {
      std::size_t nbp = 0;
      for (std::size_t l = 0; l + 1 < bs.size(); ++l) nbp += (std::size_t)bs[l] * bs[l + 1] + bs[l + 1];
      *out = oracle_deeponet_create(&g, tstar, sstar, act, (int32_t)bs.size(), bs.data(), prm.data(),
                                    (int32_t)ts.size(), ts.data(), prm.data() + nbp, hb ? 1 : 0, (float)b0);
    } else {
      *out = oracle_fno_create(&g, tstar, sstar, act, (int32_t)arch_dims[0], (int32_t)arch_dims[1],
                               (int32_t)arch_dims[2], (int32_t)arch_dims[3], prm.data());
    }
    return 0;
  } catch (const IoFail& e) {
    g_err = std::string("model load: ") + e.what();
    return SNOP_IO_ERROR;
  } catch (...) {
    return map_exc();
  }
}

void* oracle_exact_operator_create(const snop_grid* grid, int32_t order, double tstar, double sstar,
                                   const snop_solver_config* cfg) {
  auto* op = new OracleOp;
  op->kind = 2;
  op->grid = Grid1D{grid->length_cm, grid->n_cells};
  op->tstar = tstar;
  op->sstar = sstar;
  op->quad = gauss_legendre(order);
  op->cfg = to_cfg(cfg);
  return op;
}

void oracle_op_destroy(void* op) { delete static_cast<OracleOp*>(op); }

int oracle_op_predict(void* vop, int32_t batch, const double* src, double* out, int32_t n_threads) {
  try {
    const auto* op = static_cast<const OracleOp*>(vop);
    const std::size_t Nc = op->grid.n_cells;
    parallel_chunks(batch, batch, [&](std::size_t, std::size_t b0, std::size_t b1) {
      for (std::size_t b = b0; b < b1; ++b) op->predict(src + b * Nc, out + b * Nc);
    }, n_threads);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int oracle_recast_fixed_point(void* vop, int32_t batch, const double* src, const double* st, const double* ss0,
                              double tol, int32_t max_it, int32_t norm, const double* init_phi, double* phi_out,
                              int32_t* iters, int32_t* status, int32_t n_threads) {
  try {
    const auto* op = static_cast<const OracleOp*>(vop);
    const std::size_t Nc = op->grid.n_cells;
    parallel_chunks(batch, batch, [&](std::size_t, std::size_t b0, std::size_t b1) {
      for (std::size_t b = b0; b < b1; ++b) {
        const RecastResult r = recast_fixed_point(
            (int)Nc, src + b * Nc, st + b * Nc, ss0 + b * Nc, op->tstar, op->sstar,
            [&](const double* s, double* o) { op->predict(s, o); }, tol, max_it, static_cast<Norm>(norm),
            init_phi ? init_phi + b * Nc : nullptr, phi_out + b * Nc);
        iters[b] = r.iterations;
        status[b] = static_cast<int32_t>(r.status);
      }
    }, n_threads);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

// recast fixed point, then source iteration on the full target warm-started.
int oracle_precondition_fixed_source(void* vop, int32_t order, int32_t batch, const double* st,
                                     const double* ss0, const double* ss1, const double* src, double rtol,
                                     int32_t rmax, const snop_solver_config* ccfg, double* phi_out,
                                     int32_t* piters, int32_t* rstatus, int32_t* riters, uint8_t* conv,
                                     int32_t n_threads) {
  try {
    const auto* op = static_cast<const OracleOp*>(vop);
    const Grid1D& g = op->grid;
    const Quadrature q = gauss_legendre(order);
    const SolverConfig cfg = to_cfg(ccfg);
    const std::size_t Nc = g.n_cells;
    parallel_chunks(batch, batch, [&](std::size_t, std::size_t b0, std::size_t b1) {
      for (std::size_t b = b0; b < b1; ++b) {
        double* phi = phi_out + b * Nc;
        const RecastResult r = recast_fixed_point(
            (int)Nc, src + b * Nc, st + b * Nc, ss0 + b * Nc, op->tstar, op->sstar,
            [&](const double* s, double* o) { op->predict(s, o); }, rtol, rmax, cfg.norm, nullptr, phi);
        piters[b] = r.iterations;
        rstatus[b] = static_cast<int32_t>(r.status);
        const SIResult s = source_iteration(g, q, st + b * Nc, ss0 + b * Nc, ss1 ? ss1 + b * Nc : nullptr,
                                            src + b * Nc, cfg, phi, nullptr);
        riters[b] = s.iterations;
        conv[b] = s.converged ? 1 : 0;
      }
    }, n_threads);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

// SPEC.md:423-441 (paper Eqs. A5-A8). Stage 1: power iteration whose inner solver is the
// operator through the recast fixed point, warm-started from the current group flux (SP), or
// that prediction refined by a model-based source iteration (CP). Stage 2: model-based power
// iteration from (k_NO, phi_NO); stage-1 divergence falls back to the cold start.
int oracle_sp_cp_eigen_batched(void* vop, int32_t algorithm, int32_t order, int32_t batch, int32_t G,
                               const double* st, const double* ss0, const double* ss1, const double* nsf,
                               const double* chi, const snop_solver_config* ccfg, double rtol, int32_t rmax,
                               double* k_out, double* phi_out, double* s1_k, int32_t* s1_outer, int64_t* s1_inner,
                               int32_t* s2_outer, int64_t* s2_inner, uint8_t* conv, uint8_t* fallback,
                               int32_t n_threads) {
  try {
    const auto* op = static_cast<const OracleOp*>(vop);
    const Grid1D g = op->grid;
    const Quadrature q = gauss_legendre(order);
    const SolverConfig cfg = to_cfg(ccfg);
    const std::size_t Nc = g.n_cells, GN = (std::size_t)G * Nc;
    std::string err;
    int code = 0;
    std::mutex mu;
    parallel_chunks(batch, batch, [&](std::size_t, std::size_t b0, std::size_t b1) {
      for (std::size_t b = b0; b < b1; ++b) {
        try {
          MGView m;
          m.G = G;
          m.sigma_t = st + b * GN;
          m.sigma_s0 = ss0 + b * GN * G;
          m.sigma_s1 = ss1 ? ss1 + b * GN : nullptr;
          m.nu_sigma_f = nsf + b * GN;
          m.chi = chi + b * G;
          double* phi = phi_out + b * GN;
          std::fill(phi, phi + GN, 1.0);
          bool diverged = false;
          InnerSolver stage1 = [&](int gg, const double* qe, double* phig) -> int {
            const double* stg = m.sigma_t + (std::size_t)gg * Nc;
            const double* ssg = m.sigma_s0 + ((std::size_t)gg * G + gg) * Nc;
            std::vector<double> pred(Nc);
            const RecastResult r = recast_fixed_point(
                (int)Nc, qe, stg, ssg, op->tstar, op->sstar, [&](const double* s, double* o) { op->predict(s, o); },
                rtol, rmax, cfg.norm, phig, pred.data());
            if (r.status == RecastStatus::Diverged) diverged = true;
            int count = r.iterations;
            if (algorithm == 1) {  // CP: model-based refinement of the prediction (Eq. A8)
              SolverConfig icfg = cfg;
              std::copy(pred.begin(), pred.end(), phig);
              const double* s1g = m.sigma_s1 ? m.sigma_s1 + (std::size_t)gg * Nc : nullptr;
              count += source_iteration(g, q, stg, ssg, s1g, qe, icfg, phig, nullptr).iterations;
            } else {
              std::copy(pred.begin(), pred.end(), phig);
            }
            return count;
          };
          EigenResult r1;
          bool fb = false;
          try {
            r1 = power_iteration(g, q, m, cfg, phi, true, 1.0, &stage1);
            if (diverged || !std::isfinite(r1.k) || !(r1.k > 0.0)) fb = true;
          } catch (const DegenerateProblem&) {
            fb = true;
          }
          if (fb) std::fill(phi, phi + GN, 1.0);
          const EigenResult r2 = power_iteration(g, q, m, cfg, phi, true, fb ? 1.0 : r1.k, nullptr);
          k_out[b] = r2.k;
          s1_k[b] = r1.k;
          s1_outer[b] = r1.outer;
          s1_inner[b] = r1.inner;
          s2_outer[b] = r2.outer;
          s2_inner[b] = r2.inner;
          conv[b] = r2.converged ? 1 : 0;
          fallback[b] = fb ? 1 : 0;
        } catch (...) {
          std::lock_guard<std::mutex> lk(mu);
          code = map_exc();
          err = g_err;
        }
      }
    }, n_threads);
    if (code) { g_err = err; return code; }
    return 0;
  } catch (...) {
    return map_exc();
  }
}

// GRF sampling / dataset generation. spec = {mean, variance, length_scale,
// jitter, seed} as snop_grf_spec.
int oracle_grf_sample(const snop_grid* grid, const snop_grf_spec* sp, int64_t first, int32_t n_samples,
                      double* out, int64_t* negatives, double* jitter_used) {
  try {
    const Grid1D g{grid->length_cm, grid->n_cells};
    const GrfSpec spec{sp->mean, sp->variance, sp->length_scale_cm, sp->jitter, sp->seed};
    double jit = 0.0;
    const std::vector<double> L = grf_cholesky(g, spec, &jit);
    if (jitter_used) *jitter_used = jit;
    for (int32_t s = 0; s < n_samples; ++s) {
      const long long neg = sample_grf(g, spec, L, (std::uint64_t)(first + s), out + (std::size_t)s * g.n_cells);
      if (negatives) negatives[s] = neg;
    }
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int oracle_normalize_source(const snop_grid* grid, int32_t n, const double* raw, double* out) {
  try {
    const Grid1D g{grid->length_cm, grid->n_cells};
    for (int32_t s = 0; s < n; ++s)
      normalize_source(g, raw + (std::size_t)s * g.n_cells, out + (std::size_t)s * g.n_cells);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

// generate_dataset: per sample sample_grf -> normalize -> source_iteration at p*
// (zero initial guess, vacuum both sides); non-convergence aborts with the sample index.
int oracle_generate_dataset(const snop_grid* grid, int32_t order, const snop_grf_spec* sp, int32_t n_samples,
                            double tstar, double sstar, double tol, double* sources, double* fluxes,
                            int32_t* iterations, int32_t n_threads) {
  try {
    const Grid1D g{grid->length_cm, grid->n_cells};
    const GrfSpec spec{sp->mean, sp->variance, sp->length_scale_cm, sp->jitter, sp->seed};
    const std::vector<double> L = grf_cholesky(g, spec);
    const Quadrature q = gauss_legendre(order);
    SolverConfig cfg;
    cfg.tolerance = tol;
    const std::size_t Nc = g.n_cells;
    const std::vector<double> st(Nc, tstar), ss(Nc, sstar);
    std::string err;
    int code = 0;
    std::mutex mu;
    parallel_chunks(n_samples, n_samples, [&](std::size_t, std::size_t b0, std::size_t b1) {
      for (std::size_t b = b0; b < b1; ++b) {
        try {
          std::vector<double> raw(Nc);
          sample_grf(g, spec, L, b, raw.data());
          normalize_source(g, raw.data(), sources + b * Nc);
          double* phi = fluxes + b * Nc;
          std::fill(phi, phi + Nc, 0.0);
          const SIResult r = source_iteration(g, q, st.data(), ss.data(), nullptr, sources + b * Nc, cfg, phi, nullptr);
          iterations[b] = r.iterations;
          if (!r.converged) throw NumericalError("generate_dataset: sample " + std::to_string(b) + " did not converge");
        } catch (...) {
          std::lock_guard<std::mutex> lk(mu);
          code = map_exc();
          err = g_err;
        }
      }
    }, n_threads);
    if (code) { g_err = err; return code; }
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int oracle_balance_residual(const snop_grid* grid, const double* st, const double* ss0, const double* src,
                            const double* phi, double leak_left, double leak_right, double* out) {
  try {
    const Grid1D g{grid->length_cm, grid->n_cells};
    *out = balance_residual(g, st, ss0, src, phi, leak_left, leak_right);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

}  // extern "C"
