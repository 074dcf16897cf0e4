// snop/cuda.hpp — header-only C++ host layer over the C-ABI (include/snop_cuda.h), mirroring the
// reference's planned snop:: solver API (SPEC.md [OP] signatures; the reference ships no solver
// headers) and rethrowing its exception classes (proj/core/include/snop/errors.hpp:8-41).
//
//   snop::cuda::Context ctx;                     // one GPU + stream + workspace
//   auto r = snop::cuda::source_iteration(ctx, grid, 32, materials, source, cfg);
//   auto e = snop::cuda::power_iteration(ctx, grid, 16, mg_materials, cfg);
//
// Arrays are host std::vector<double> (the call stages H2D/D2H); batched [B][Nc] layouts.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../snop_cuda.h"

namespace snop {

// errors.hpp:8-41 (same hierarchy; defined here so this header is self-contained)
#ifndef SNOP_ERRORS_DEFINED
#define SNOP_ERRORS_DEFINED
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class InvalidArgument : public Error {
 public:
  using Error::Error;
};
class NumericalError : public Error {
 public:
  using Error::Error;
};
class DegenerateProblem : public NumericalError {
 public:
  using NumericalError::NumericalError;
};
class IoError : public Error {
 public:
  using Error::Error;
};
class ConfigError : public Error {
 public:
  using Error::Error;
};
#endif

namespace cuda {

inline void check(snop_status s) {
  if (s == SNOP_OK) return;
  const std::string m = snop_last_error();
  switch (s) {
    case SNOP_INVALID_ARGUMENT: throw InvalidArgument(m);
    case SNOP_DEGENERATE_PROBLEM: throw DegenerateProblem(m);
    case SNOP_NUMERICAL_ERROR: throw NumericalError(m);
    case SNOP_IO_ERROR: throw IoError(m);
    case SNOP_CONFIG_ERROR: throw ConfigError(m);
    default: throw Error(m);
  }
}

struct Grid1D {
  double length_cm = 10.0;
  int n_cells = 100;
  snop_grid c() const { return snop_grid{length_cm, n_cells, 0}; }
};

enum class Boundary : int32_t { Vacuum = SNOP_BC_VACUUM, Reflective = SNOP_BC_REFLECTIVE };
enum class Norm : int32_t { RelativeLinf = SNOP_NORM_REL_LINF, RelativeL2 = SNOP_NORM_REL_L2 };

struct SolverConfig {
  double tolerance = 1e-4, tolerance_k = 1e-4, tolerance_phi = 1e-4;
  int max_inner_iterations = 10000, max_outer_iterations = 5000;
  Boundary boundary_left = Boundary::Vacuum, boundary_right = Boundary::Vacuum;
  Norm convergence_norm = Norm::RelativeLinf;
  snop_solver_config c() const {
    return snop_solver_config{tolerance, tolerance_k, tolerance_phi, max_inner_iterations, max_outer_iterations,
                              (int32_t)boundary_left, (int32_t)boundary_right, (int32_t)convergence_norm, 0};
  }
};

struct AngularQuadrature {
  int order = 0;
  std::vector<double> mu, w;
};

inline AngularQuadrature gauss_legendre(int order) {
  AngularQuadrature q;
  q.order = order;
  q.mu.resize(order > 0 ? order : 0);
  q.w.resize(q.mu.size());
  check(snop_gauss_legendre(order, q.mu.data(), q.w.data()));
  return q;
}

class Context {
 public:
  explicit Context(int device = 0) { check(snop_ctx_create(device, &ctx_)); }
  ~Context() { snop_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  snop_ctx* get() const { return ctx_; }
  // execution options (include/snop_cuda.h snop_ctx_options; zero fields = automatic)
  snop_ctx_options options() const {
    snop_ctx_options o{};
    check(snop_ctx_get_options(ctx_, &o));
    return o;
  }
  void set_options(const snop_ctx_options& o) { check(snop_ctx_set_options(ctx_, &o)); }

 private:
  snop_ctx* ctx_ = nullptr;
};

// single-group batched materials for source_iteration ([B][Nc] each; sigma_s1 optional)
struct SingleGroupMaterials {
  int batch = 0;
  std::vector<double> sigma_t, sigma_s0, sigma_s1;
};

struct FixedSourceSolution {  // (FluxField, iterations, converged), batched
  std::vector<double> phi, current;
  std::vector<int32_t> iterations;
  std::vector<uint8_t> converged;
};

// SPEC.md:125-134
inline FixedSourceSolution source_iteration(Context& ctx, const Grid1D& grid, int order,
                                            const SingleGroupMaterials& m, const std::vector<double>& source,
                                            const SolverConfig& cfg,
                                            const std::vector<double>* initial_phi = nullptr,
                                            bool want_current = false) {
  const size_t n = (size_t)m.batch * grid.n_cells;
  if (m.sigma_t.size() != n || m.sigma_s0.size() != n || source.size() != n ||
      (!m.sigma_s1.empty() && m.sigma_s1.size() != n) || (initial_phi && initial_phi->size() != n))
    throw InvalidArgument("source_iteration: array sizes must be batch * n_cells");
  FixedSourceSolution r;
  r.phi.resize(n);
  if (want_current) r.current.resize(n);
  r.iterations.resize(m.batch);
  r.converged.resize(m.batch);
  const snop_grid g = grid.c();
  const snop_solver_config c = cfg.c();
  check(snop_source_iteration_batched(ctx.get(), SNOP_MEM_HOST, &g, order, m.batch, m.sigma_t.data(),
                                      m.sigma_s0.data(), m.sigma_s1.empty() ? nullptr : m.sigma_s1.data(),
                                      source.data(), &c, initial_phi ? initial_phi->data() : nullptr, r.phi.data(),
                                      want_current ? r.current.data() : nullptr, r.iterations.data(),
                                      r.converged.data()));
  return r;
}

// multigroup batched materials for power_iteration (SPEC.md:37-43 layout)
struct MultiGroupMaterials {
  int batch = 0, groups = 1;
  std::vector<double> sigma_t;     // [B][G][Nc]
  std::vector<double> sigma_s0;    // [B][G'][G][Nc], g' -> g
  std::vector<double> sigma_s1;    // [B][G][Nc] or empty
  std::vector<double> nu_sigma_f;  // [B][G][Nc]
  std::vector<double> chi;         // [B][G]
};

struct EigenSolution {  // SPEC.md:172-176, batched
  std::vector<double> k, phi;
  std::vector<int32_t> outer_iterations;
  std::vector<int64_t> total_inner_iterations;
  std::vector<uint8_t> converged;
};

// SPEC.md:179-189 with the model-based inner solver; initial = optional (k, flux)
inline EigenSolution power_iteration(Context& ctx, const Grid1D& grid, int order, const MultiGroupMaterials& m,
                                     const SolverConfig& cfg, const std::vector<double>* initial_k = nullptr,
                                     const std::vector<double>* initial_phi = nullptr) {
  const size_t n = (size_t)m.batch * m.groups * grid.n_cells;
  if (m.sigma_t.size() != n || m.nu_sigma_f.size() != n || m.sigma_s0.size() != n * m.groups ||
      m.chi.size() != (size_t)m.batch * m.groups)
    throw InvalidArgument("power_iteration: array sizes do not match batch/groups/n_cells");
  EigenSolution e;
  e.k.resize(m.batch);
  e.phi.resize(n);
  e.outer_iterations.resize(m.batch);
  e.total_inner_iterations.resize(m.batch);
  e.converged.resize(m.batch);
  const snop_grid g = grid.c();
  const snop_solver_config c = cfg.c();
  check(snop_power_iteration_batched(ctx.get(), SNOP_MEM_HOST, &g, order, m.batch, m.groups, m.sigma_t.data(),
                                     m.sigma_s0.data(), m.sigma_s1.empty() ? nullptr : m.sigma_s1.data(),
                                     m.nu_sigma_f.data(), m.chi.data(), &c, initial_k ? initial_k->data() : nullptr,
                                     initial_phi ? initial_phi->data() : nullptr, e.k.data(), e.phi.data(),
                                     e.outer_iterations.data(), e.total_inner_iterations.data(), e.converged.data()));
  return e;
}

// sweep, batched over instances: emission [B][Nc][order] -> psi_avg [B][order][Nc]
// and the net outgoing partial currents at the two faces.
struct SweepResult {
  std::vector<double> psi_avg, outflow_left, outflow_right;
};
inline SweepResult sweep(Context& ctx, const Grid1D& grid, int order, int batch, const std::vector<double>& sigma_t,
                         const std::vector<double>& emission, int boundary_left = SNOP_BC_VACUUM,
                         int boundary_right = SNOP_BC_VACUUM) {
  SweepResult r;
  r.psi_avg.resize(emission.size());
  r.outflow_left.resize(batch);
  r.outflow_right.resize(batch);
  const snop_grid g = grid.c();
  check(snop_sweep_batched(ctx.get(), SNOP_MEM_HOST, &g, order, batch, sigma_t.data(), emission.data(),
                           boundary_left, boundary_right, r.psi_avg.data(), r.outflow_left.data(),
                           r.outflow_right.data()));
  return r;
}

// SPEC.md:393-401
inline std::vector<double> recast_source(Context& ctx, int batch, int n_cells, const std::vector<double>& S,
                                         const std::vector<double>& phi, const std::vector<double>& sigma_t,
                                         const std::vector<double>& sigma_s0, double sigma_t_star,
                                         double sigma_s0_star) {
  std::vector<double> out(S.size());
  check(snop_recast_source(ctx.get(), SNOP_MEM_HOST, batch, n_cells, S.data(), phi.data(), sigma_t.data(),
                           sigma_s0.data(), sigma_t_star, sigma_s0_star, out.data()));
  return out;
}

// SolutionOperator: owns an snop_op handle.
class SolutionOperator {
 public:
  SolutionOperator(Context& ctx, snop_op* op, int n_cells) : ctx_(&ctx), op_(op), n_(n_cells) {}
  ~SolutionOperator() { snop_op_destroy(op_); }
  SolutionOperator(const SolutionOperator&) = delete;
  SolutionOperator& operator=(const SolutionOperator&) = delete;
  snop_op* get() const { return op_; }
  Context& context() const { return *ctx_; }
  int n_cells() const { return n_; }

  // predict(model, source), batched [B][Nc]
  std::vector<double> predict(const std::vector<double>& source) const {
    std::vector<double> out(source.size());
    check(snop_op_predict(ctx_->get(), op_, SNOP_MEM_HOST, (int32_t)(source.size() / n_), source.data(),
                          out.data()));
    return out;
  }

  static SolutionOperator exact(Context& ctx, const Grid1D& grid, int order, double st_star, double ss_star,
                                const SolverConfig& cfg) {
    snop_op* op = nullptr;
    const snop_grid g = grid.c();
    const snop_solver_config c = cfg.c();
    check(snop_exact_operator_create(ctx.get(), &g, order, st_star, ss_star, &c, &op));
    return SolutionOperator(ctx, op, grid.n_cells);
  }

  // load_model / save_model: DeepONet or FNO model files.
  static SolutionOperator load(Context& ctx, const std::string& path) {
    snop_model_info info{};
    check(snop_model_inspect(path.c_str(), &info));
    snop_op* op = nullptr;
    check(snop_op_load(ctx.get(), path.c_str(), &op));
    return SolutionOperator(ctx, op, info.grid.n_cells);
  }
  void save(const std::string& path) const { check(snop_op_save(op_, path.c_str())); }

  SolutionOperator(SolutionOperator&& o) noexcept : ctx_(o.ctx_), op_(o.op_), n_(o.n_) { o.op_ = nullptr; }

 private:
  Context* ctx_;
  snop_op* op_;
  int n_;
};

struct RecastResult {
  std::vector<double> phi;
  std::vector<int32_t> iterations, status;  // status: snop_recast_status
};

// SPEC.md:403-411
inline RecastResult recast_fixed_point(const SolutionOperator& op, const std::vector<double>& S,
                                       const std::vector<double>& sigma_t, const std::vector<double>& sigma_s0,
                                       double tolerance = 1e-4, int max_iterations = 50,
                                       Norm norm = Norm::RelativeLinf) {
  const int B = (int)(S.size() / op.n_cells());
  RecastResult r;
  r.phi.resize(S.size());
  r.iterations.resize(B);
  r.status.resize(B);
  check(snop_recast_fixed_point(op.context().get(), op.get(), SNOP_MEM_HOST, B, S.data(), sigma_t.data(),
                                sigma_s0.data(), tolerance, max_iterations, (int32_t)norm, nullptr, r.phi.data(),
                                r.iterations.data(), r.status.data()));
  return r;
}

struct HybridEigenSolution : EigenSolution {  // EigenSolution + stage diagnostics
  std::vector<double> stage1_k;
  std::vector<int32_t> stage1_outer;
  std::vector<int64_t> stage1_inner;
  std::vector<uint8_t> fallback;
};

enum class HybridAlgorithm { SP, CP };

// power_iteration(grid, quadrature, materials, config, inner_solver, initial) with a
// neural-operator-backed inner_solver: the within-group solve is the operator's
// recast fixed point (SP) or that prediction refined by a model-based source iteration (CP) --
// stage 1 of the hybrids on its own. The model-based inner solver is snop::power_iteration.
struct OperatorEigenSolution : EigenSolution {
  std::vector<uint8_t> diverged;
};
inline OperatorEigenSolution power_iteration(HybridAlgorithm inner_solver, const SolutionOperator& op, int order,
                                             const MultiGroupMaterials& m, const SolverConfig& cfg,
                                             double recast_tolerance = 1e-4, int recast_max_iterations = 50) {
  const size_t n = (size_t)m.batch * m.groups * op.n_cells();
  if (m.sigma_t.size() != n || m.nu_sigma_f.size() != n || m.sigma_s0.size() != n * m.groups ||
      m.chi.size() != (size_t)m.batch * m.groups || (!m.sigma_s1.empty() && m.sigma_s1.size() != n))
    throw InvalidArgument("power_iteration: array sizes do not match batch/groups/n_cells");
  OperatorEigenSolution e;
  e.k.resize(m.batch);
  e.phi.resize(n);
  e.outer_iterations.resize(m.batch);
  e.total_inner_iterations.resize(m.batch);
  e.converged.resize(m.batch);
  e.diverged.resize(m.batch);
  const snop_solver_config c = cfg.c();
  check(snop_power_iteration_operator_batched(
      op.context().get(), op.get(),
      inner_solver == HybridAlgorithm::SP ? SNOP_INNER_RECAST_FIXED_POINT : SNOP_INNER_PREDICT_REFINE, SNOP_MEM_HOST,
      order, m.batch, m.groups, m.sigma_t.data(), m.sigma_s0.data(), m.sigma_s1.empty() ? nullptr : m.sigma_s1.data(),
      m.nu_sigma_f.data(), m.chi.data(), &c, recast_tolerance, recast_max_iterations, e.k.data(), e.phi.data(),
      e.outer_iterations.data(), e.total_inner_iterations.data(), e.converged.data(), e.diverged.data()));
  return e;
}

// sp_eigen / cp_eigen: stage 1 with the operator as the within-group solver,
// stage 2 model-based from (k_NO, phi_NO); divergence falls back to the cold start.
inline HybridEigenSolution hybrid_eigen(HybridAlgorithm alg, const SolutionOperator& op, int order,
                                        const MultiGroupMaterials& m, const SolverConfig& cfg,
                                        double recast_tolerance = 1e-4, int recast_max_iterations = 50) {
  const size_t n = (size_t)m.batch * m.groups * op.n_cells();
  if (m.sigma_t.size() != n || m.nu_sigma_f.size() != n || m.sigma_s0.size() != n * m.groups ||
      m.chi.size() != (size_t)m.batch * m.groups || (!m.sigma_s1.empty() && m.sigma_s1.size() != n))
    throw InvalidArgument("hybrid_eigen: array sizes do not match batch/groups/n_cells");
  HybridEigenSolution e;
  e.k.resize(m.batch);
  e.phi.resize(n);
  e.stage1_k.resize(m.batch);
  e.stage1_outer.resize(m.batch);
  e.stage1_inner.resize(m.batch);
  e.outer_iterations.resize(m.batch);
  e.total_inner_iterations.resize(m.batch);
  e.converged.resize(m.batch);
  e.fallback.resize(m.batch);
  const snop_solver_config c = cfg.c();
  auto fn = alg == HybridAlgorithm::SP ? snop_sp_eigen_batched : snop_cp_eigen_batched;
  check(fn(op.context().get(), op.get(), SNOP_MEM_HOST, order, m.batch, m.groups, m.sigma_t.data(),
           m.sigma_s0.data(), m.sigma_s1.empty() ? nullptr : m.sigma_s1.data(), m.nu_sigma_f.data(), m.chi.data(), &c,
           recast_tolerance, recast_max_iterations, e.k.data(), e.phi.data(), e.stage1_k.data(),
           e.stage1_outer.data(), e.stage1_inner.data(), e.outer_iterations.data(), e.total_inner_iterations.data(),
           e.converged.data(), e.fallback.data()));
  return e;
}

}  // namespace cuda
}  // namespace snop
