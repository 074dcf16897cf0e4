// ============================================================================
// snop ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain-C++ CPU restatement of the reference's S_N transport hot path, written
// from the reference's behavioural contract because the
// reference ships none of the hot-path translation units (transport.cpp,
// eigenvalue.cpp, precond.cpp, deeponet.cpp, fno.cpp, quadrature.cpp listed at
// proj/core/CMakeLists.txt:5-17 are absent).
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load this library. The product path
// (paper_2509_01416_b200/, libsnop_cuda.so) never links or calls it.
//
// Parity pins: SPEC [OP] examples (gauss_legendre
// SPEC.md:70-72, sweep :121-123, source_iteration :131-134, power_iteration
// :185-188, recast :399-401, predict :325-326); paper Table 9 k = 1.30621
// (PAPER.md:379); the reference's own shipped rng.hpp / parallel.hpp compiled
// under oracle/_ref (stream + partition golden vectors).
// ============================================================================
#pragma once

#include <cstdint>
#include <cstddef>
#include <functional>
#include <random>
#include <vector>
#include <cmath>
#include <numbers>
#include <stdexcept>
#include <string>

namespace snop::oracle {

// --- errors (restates proj/core/include/snop/errors.hpp:8-41) ---------------
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct InvalidArgument : Error { using Error::Error; };
struct NumericalError : Error { using Error::Error; };
struct DegenerateProblem : NumericalError { using NumericalError::NumericalError; };

// --- Rng (restates proj/core/include/snop/rng.hpp:17-49) --------------------
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : engine_(seed) {}
  std::uint64_t next_u64() { return engine_(); }
  double uniform() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double normal() {
    if (has_spare_) { has_spare_ = false; return spare_; }
    const double u1 = (static_cast<double>(engine_() >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 2.0 * std::numbers::pi * u2;
    spare_ = r * std::sin(a);
    has_spare_ = true;
    return r * std::cos(a);
  }
 private:
  std::mt19937_64 engine_;
  bool has_spare_ = false;
  double spare_ = 0.0;
};

// --- parallel_chunks (restates proj/core/include/snop/parallel.hpp:17-48) ----
void parallel_chunks(std::size_t n_items, std::size_t n_chunks,
                     const std::function<void(std::size_t, std::size_t, std::size_t)>& fn,
                     unsigned n_threads = 0);

// --- core types ---------------------------------------------
enum class Boundary : int { Vacuum = 0, Reflective = 1 };
enum class Norm : int { RelLinf = 0, RelL2 = 1 };

struct Grid1D {
  double length = 10.0;
  int n_cells = 100;
  double dx() const { return length / n_cells; }
  double center(int i) const { return (i + 0.5) * dx(); }
};

struct Quadrature {  // SPEC.md:29-35; nodes ascending (mu[n] = -mu[N-1-n])
  int order = 0;
  std::vector<double> mu, w;
};

struct SolverConfig {  // SPEC.md:57-61 (+ split eigen tolerances)
  double tolerance = 1e-4;      // inner / fixed-source tolerance
  double tolerance_k = 1e-4;    // eigen: |dk|/k
  double tolerance_phi = 1e-4;  // eigen: outer flux change
  int max_inner = 10000;
  int max_outer = 5000;
  Boundary left = Boundary::Vacuum, right = Boundary::Vacuum;
  Norm norm = Norm::RelLinf;
};

Quadrature gauss_legendre(int order);
double integrate_cellwise(const double* f, const Grid1D& g);
double relative_change(const double* a_new, const double* a_old, std::size_t n, Norm norm);

// --- transport --------------------------------------------
// emission[i*N + n]; psi_avg[n*Nc + i]. Returns outgoing partial currents.
void sweep(const Grid1D& g, const Quadrature& q, const double* sigma_t, const double* emission,
           Boundary left, Boundary right, double* psi_avg, double* out_left, double* out_right,
           std::vector<double>* lag_right = nullptr);

struct SIResult { int iterations = 0; bool converged = false; double out_left = 0, out_right = 0; };

// One single-group fixed-source solve. sigma_s1 may be null (isotropic).
// phi holds the initial guess on entry (zeros = SPEC default) and the result on exit.
SIResult source_iteration(const Grid1D& g, const Quadrature& q, const double* sigma_t,
                          const double* sigma_s0, const double* sigma_s1, const double* source,
                          const SolverConfig& cfg, double* phi, double* current);

double balance_residual(const Grid1D& g, const double* sigma_t, const double* sigma_s0_total_out,
                        const double* source, const double* phi, double out_left, double out_right);

// --- eigen ------------------------------------------------
struct EigenResult { double k = 1.0; int outer = 0; long long inner = 0; bool converged = false; };

// Multigroup materials for one instance: sigma_t[g*Nc+i], sigma_s0[(gp*G+g)*Nc+i] (gp->g),
// sigma_s1[g*Nc+i] (nullable), nu_sigma_f[g*Nc+i], chi[g].
struct MGView {
  int G = 1;
  const double* sigma_t = nullptr;
  const double* sigma_s0 = nullptr;
  const double* sigma_s1 = nullptr;
  const double* nu_sigma_f = nullptr;
  const double* chi = nullptr;
};

// inner_solver(g, q_ext, phi_g in/out) -> sweeps used. Default = source_iteration.
using InnerSolver = std::function<int(int g, const double* q_ext, double* phi_g)>;

EigenResult power_iteration(const Grid1D& grid, const Quadrature& q, const MGView& m,
                            const SolverConfig& cfg, double* phi /* [G*Nc], initial on entry if has_initial */,
                            bool has_initial, double initial_k, const InnerSolver* inner = nullptr);

double infinite_medium_k(int G, const double* sigma_t, const double* sigma_s0 /* [gp][g] */,
                         const double* nu_sigma_f, const double* chi);

// --- neural operators, forward only ------------------------
enum class Activation : int { ReLU = 0, Tanh = 1, GELU = 2, Identity = 3 };

template <class T> T activate(T x, Activation a) {
  switch (a) {
    case Activation::ReLU: return x > T(0) ? x : T(0);
    case Activation::Tanh: return std::tanh(x);
    case Activation::GELU: return T(0.5) * x * (T(1) + std::erf(x * T(0.70710678118654752440)));
    default: return x;
  }
}

struct DenseNetwork {  // layer l: W[l] is [n_out][n_in] row-major, b[l] is [n_out]
  std::vector<int> sizes;
  std::vector<std::vector<float>> W, b;
  Activation act = Activation::ReLU;
};

struct DeepONet { DenseNetwork branch, trunk; bool has_bias0 = false; float bias0 = 0.f; };

struct FNO {
  int width = 64, modes = 16, layers = 4, proj_hidden = 128;
  Activation act = Activation::GELU;
  std::vector<float> lift_W, lift_b;            // [width][2], [width]
  std::vector<std::vector<float>> R_re, R_im;   // per layer [modes][in][out]
  std::vector<std::vector<float>> W, b;         // per layer [out][in], [out]
  std::vector<float> P1_W, P1_b, P2_W, P2_b;    // [hidden][width],[hidden],[1][hidden],[1]
};

// Forward passes in double arithmetic on float parameters ("fp64 reference mode").
void dense_forward(const DenseNetwork& net, const double* in, double* out);
void deeponet_predict(const DeepONet& m, const Grid1D& g, const double* source, double* out);
void fno_predict(const FNO& m, const Grid1D& g, const double* source, double* out);

// --- precond -----------------------------------------------
using SolutionOperator = std::function<void(const double* s, double* phi)>;

void recast_source(int n, const double* S, const double* phi, const double* sigma_t,
                   const double* sigma_s0, double sigma_t_star, double sigma_s0_star, double* out);

enum class RecastStatus : int { Converged = 0, MaxIterations = 1, Diverged = 2 };
struct RecastResult { int iterations = 0; RecastStatus status = RecastStatus::Converged; };

RecastResult recast_fixed_point(int n, const double* S, const double* sigma_t, const double* sigma_s0,
                                double sigma_t_star, double sigma_s0_star, const SolutionOperator& op,
                                double tol, int max_it, Norm norm, const double* initial_phi,
                                double* phi_out);

// --- grf ------------------------------------------------------
struct GrfSpec {
  double mean = 0.07, variance = 3e-4, length_scale = 1.2, jitter = 1e-10;
  std::uint64_t seed = 0;
};

// Row-major lower-triangular L with L L^T = C + jitter var I, C_ij = var exp(-(x_i-x_j)^2 / (2 l^2))
// at the cell centres (Cholesky-Banachiewicz, row by row); on a non-positive pivot the jitter is
// escalated x10 while <= 1e-6, else NumericalError. The jitter is relative to the
// variance: SPEC.md:245's example (variance 1e-18 -> field constant within 1e-8) is unreachable
// with an absolute 1e-10 jitter (noise sqrt(1e-10) = 1e-5), so the SPEC's own example pins it.
std::vector<double> grf_cholesky(const Grid1D& g, const GrfSpec& spec, double* jitter_used = nullptr);

// sample_grf: out_i = mean + sum_{j<=i} L_ij z_j, z_j = Rng(seed + sample).normal()
// drawn j = 0..n-1. Returns the number of negative entries (reported, not clipped).
long long sample_grf(const Grid1D& g, const GrfSpec& spec, const std::vector<double>& L, std::uint64_t sample,
                     double* out);

// normalize_source: raw / (dx sum raw); InvalidArgument if the integral <= 0.
void normalize_source(const Grid1D& g, const double* raw, double* out);

}  // namespace snop::oracle
