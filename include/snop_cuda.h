/*
 * snop_cuda.h — C-ABI of the B200-native S_N transport hot path (libsnop_cuda.so).
 *
 * Drop-in boundary for the reference's planned `snop::` solver API. The reference ships no
 * solver headers (only proj/core/include/snop/{binary_io,errors,parallel,rng}.hpp); its API
 * exists as the SPEC [OP] signatures cited on each entry point below. Every entry point:
 *   - takes plain pointers + sizes (no C++ / torch types),
 *   - never throws; returns snop_status (1:1 with proj/core/include/snop/errors.hpp:8-41),
 *     with a thread-local message from snop_last_error(),
 *   - reports per-instance non-convergence as data (converged[b] = 0), never as an error
 *     (SPEC.md:129,183),
 *   - accepts HOST pointers (SNOP_MEM_HOST: the call copies in/out, synchronous) or DEVICE
 *     pointers (SNOP_MEM_DEVICE: enqueued on the context's stream, asynchronous; caller syncs
 *     with snop_ctx_synchronize()).
 *
 * Array layouts (row-major, fp64 unless noted), B = batch, G = groups, Nc = cells:
 *   per-cell single group  [B][Nc]
 *   multigroup             [B][G][Nc]
 *   scattering matrix      [B][G][G][Nc], entry [b][g'][g][i] = Sigma_s0^{g'->g}(x_i)
 *   fission spectrum chi   [B][G]
 */
#ifndef SNOP_CUDA_H
#define SNOP_CUDA_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SNOP_ABI_VERSION 1

typedef enum {
  SNOP_OK = 0,
  SNOP_INVALID_ARGUMENT = 1,   /* snop::InvalidArgument  (errors.hpp:13-17)  */
  SNOP_NUMERICAL_ERROR = 2,    /* snop::NumericalError   (errors.hpp:19-23)  */
  SNOP_DEGENERATE_PROBLEM = 3, /* snop::DegenerateProblem(errors.hpp:25-29)  */
  SNOP_IO_ERROR = 4,           /* snop::IoError          (errors.hpp:31-35)  */
  SNOP_CONFIG_ERROR = 5,       /* snop::ConfigError      (errors.hpp:37-41)  */
  SNOP_CUDA_ERROR = 6          /* device/runtime failure (no reference analogue) */
} snop_status;

typedef enum { SNOP_MEM_HOST = 0, SNOP_MEM_DEVICE = 1 } snop_memspace;
typedef enum { SNOP_BC_VACUUM = 0, SNOP_BC_REFLECTIVE = 1 } snop_boundary;
typedef enum { SNOP_NORM_REL_LINF = 0, SNOP_NORM_REL_L2 = 1 } snop_norm;
typedef enum { SNOP_ACT_RELU = 0, SNOP_ACT_TANH = 1, SNOP_ACT_GELU = 2 } snop_activation;
typedef enum { SNOP_RECAST_CONVERGED = 0, SNOP_RECAST_MAXED = 1, SNOP_RECAST_DIVERGED = 2 } snop_recast_status;

/* Grid1D: uniform slab, dx = length / n_cells, x_i = (i + 1/2) dx. */
typedef struct {
  double length_cm;
  int32_t n_cells;
  int32_t reserved;
} snop_grid;

/* SolverConfig with the eigen tolerances split. */
typedef struct {
  double tolerance;       /* fixed-source / inner tolerance (default 1e-4) */
  double tolerance_k;     /* eigen |dk|/k (default = tolerance) */
  double tolerance_phi;   /* eigen outer flux change (default = tolerance) */
  int32_t max_inner;      /* default 10000 */
  int32_t max_outer;      /* default 5000 */
  int32_t bc_left;        /* snop_boundary */
  int32_t bc_right;       /* snop_boundary */
  int32_t norm;           /* snop_norm */
  int32_t reserved;
} snop_solver_config;

/* Model-file architecture tags and header summary (snop_model_inspect). */
typedef enum { SNOP_ARCH_DEEPONET = 0, SNOP_ARCH_FNO = 1 } snop_arch;
typedef struct {
  int32_t arch;              /* snop_arch */
  snop_grid grid;            /* grid provenance */
  double sigma_t_star;       /* p* */
  double sigma_s0_star;
  int32_t activation;        /* snop_activation */
  int64_t n_params;
  int32_t n_branch, n_trunk, latent, has_bias0;  /* DeepONet */
  float bias0;
  int32_t width, modes, layers, hidden;          /* FNO */
} snop_model_info;

/* GrfSpec: paper Appendix A1 defaults mean 0.07, variance 3e-4, length
 * scale 1.2 cm, jitter 1e-10; sample s of a stream draws from Rng(seed + s). */
typedef struct {
  double mean;
  double variance;
  double length_scale_cm;
  double jitter;
  uint64_t seed;
} snop_grf_spec;

/* Training-dataset provenance. */
typedef struct {
  int64_t n_samples;
  snop_grid grid;
  int32_t order;
  int32_t reserved;
  snop_grf_spec spec;
  double sigma_t_star, sigma_s0_star, tolerance;
} snop_dataset_info;

typedef struct snop_ctx snop_ctx;  /* owns one CUDA stream + device workspace */
typedef struct snop_op snop_op;    /* SolutionOperator handle */

int32_t snop_abi_version(void);
const char* snop_last_error(void);

snop_status snop_ctx_create(int32_t device, snop_ctx** out);
snop_status snop_ctx_destroy(snop_ctx* ctx);

/* Per-context execution options (no process-global state, no environment variables). Every
 * field's zero value means "automatic" (the measured default); results of a solve never depend on
 * the execution options except where noted (the kernels are deterministic for a given shape).
 *   cell_cluster   K1/K2 cell split over a thread-block cluster: 0 auto (one CTA per instance up to
 *                  4096 cells, the smallest cluster that holds the slab up to 16384 cells, the
 *                  streaming kernel beyond), 1 never, 2/4/8 force that cluster size, -1 force the
 *                  streaming kernel (tile-by-tile sweep, per-cell state in a device workspace).
 *   pair_split     single-group eigen pair-split cluster size: 0 auto (8 with the tail split), -1
 *                  off, 2..8 force.
 *   pi_tail_cap    outer iterations of the tail split's first phase: 0 auto (12), -1 off (one launch).
 *   host_chunks    pageable-host pipeline chunk count: 0 auto (4), 1..8.
 *   gemm_engine    operator contractions: 0 auto (tcgen05 engines), 1 tcgen05 engine v1 only,
 *                  2 FFMA engine (fp32 cross-check; slow).
 *   fno_dft        FNO forward truncated DFT of layers >= 1: 0 auto (tcgen05), 1 FFMA kernel.
 *   fno_mix        FNO spectral channel mixing: 0 auto (tcgen05), 1 FFMA kernel. */
typedef struct {
  int32_t cell_cluster;
  int32_t pair_split;
  int32_t pi_tail_cap;
  int32_t host_chunks;
  int32_t gemm_engine;
  int32_t fno_dft;
  int32_t fno_mix;
  int32_t reserved[9];
} snop_ctx_options;

snop_status snop_ctx_set_options(snop_ctx* ctx, const snop_ctx_options* options);
snop_status snop_ctx_get_options(const snop_ctx* ctx, snop_ctx_options* options);
snop_status snop_ctx_synchronize(snop_ctx* ctx);
/* Number of snop kernels this context has launched (for the bench's gpu_launches claim). */
int64_t snop_ctx_launch_count(const snop_ctx* ctx);
/* The CUDA stream (cudaStream_t) the context enqueues on, as an opaque pointer. */
void* snop_ctx_stream(snop_ctx* ctx);

/* gauss_legendre: nodes ascending, mu[n] = -mu[order-1-n]. Host pointers. */
snop_status snop_gauss_legendre(int32_t order, double* mu, double* w);

/*
 * Batched single-group fixed-source solve — replaces
 *   source_iteration(grid, quadrature, materials, external_source, config, initial_phi)
 *   (sweep SPEC.md:115-123), for B independent instances.
 * sigma_s1 (P1 within-group moment, Eq. 25) and initial_phi may be NULL (isotropic / zero guess).
 * current_out may be NULL. iterations = sweeps performed.
 */
snop_status snop_source_iteration_batched(
    snop_ctx* ctx, int32_t memspace, const snop_grid* grid, int32_t order, int32_t batch,
    const double* sigma_t, const double* sigma_s0, const double* sigma_s1, const double* source,
    const snop_solver_config* cfg, const double* initial_phi,
    double* phi_out, double* current_out, int32_t* iterations, uint8_t* converged);

/*
 * Batched transport sweep — replaces
 *   sweep(grid, quadrature, sigma_t, emission, bc) -> (psi_avg, boundary_outflow_left, boundary_outflow_right)
 *   (SPEC.md:115-123), for B independent instances: ONE diamond-difference sweep of all `order`
 *   directions with a per-cell-per-direction emission, the cell-average angular flux materialised.
 * sigma_t [B][Nc]; emission [B][Nc][order] = q(x_i, mu_n) with n ascending in mu (the order of
 * snop_gauss_legendre: n < order/2 are mu < 0); psi_avg_out [B][order][Nc]. outflow_left/right [B]
 * (nullable) = sum over directions of w |mu| (psi_out - psi_in) at x = 0 / x = L (net outgoing
 * partial currents). Boundary order as in source_iteration: reflective left -> the mu < 0
 * directions first; reflective right only -> mu > 0 first; a reflective right face next to a
 * reflective left one is lagged, i.e. zero inflow for a single sweep. Nonpositive sigma_t ->
 * SNOP_INVALID_ARGUMENT. This is the HBM-bound form of the sweep (16 B per cell.angle update);
 * the fused solvers below never materialise psi.
 */
snop_status snop_sweep_batched(
    snop_ctx* ctx, int32_t memspace, const snop_grid* grid, int32_t order, int32_t batch,
    const double* sigma_t, const double* emission, int32_t bc_left, int32_t bc_right,
    double* psi_avg_out, double* outflow_left, double* outflow_right);

/* source_iteration + balance diagnostic: as snop_source_iteration_batched,
 * plus leakage_out[b][2] = the NET outflows (outgoing minus incoming partial currents) at x = 0 and
 * x = L of the last sweep -- the quantities the balance report needs. */
snop_status snop_source_iteration_leakage_batched(
    snop_ctx* ctx, int32_t memspace, const snop_grid* grid, int32_t order, int32_t batch,
    const double* sigma_t, const double* sigma_s0, const double* sigma_s1, const double* source,
    const snop_solver_config* cfg, const double* initial_phi, double* phi_out, double* current_out,
    int32_t* iterations, uint8_t* converged, double* leakage_out);

/* balance_report, batched: residual[b] = |leak_l + leak_r + absorption -
 * production| / production, absorption = dx sum (Sigma_t - Sigma_s0,total-out) phi, production =
 * dx sum S. production == 0 -> SNOP_NUMERICAL_ERROR (division guard). */
snop_status snop_balance_report(snop_ctx* ctx, int32_t memspace, const snop_grid* grid, int32_t batch,
                                const double* sigma_t, const double* sigma_s0_out, const double* source,
                                const double* phi, const double* leakage, double* residual_out);

/*
 * Batched k-eigenvalue power iteration — replaces
 *   power_iteration(grid, quadrature, materials, config, inner_solver, initial)
 *   (decisions :206-209) with the model-based inner solver, G >= 1 groups,
 *   Gauss-Seidel over groups including upscatter.
 * initial_k / initial_phi may be NULL (flat flux, k = 1).
 * Any instance with a zero fission integral fails the call with SNOP_DEGENERATE_PROBLEM.
 */
snop_status snop_power_iteration_batched(
    snop_ctx* ctx, int32_t memspace, const snop_grid* grid, int32_t order, int32_t batch, int32_t n_groups,
    const double* sigma_t, const double* sigma_s0, const double* sigma_s1, const double* nu_sigma_f,
    const double* chi, const snop_solver_config* cfg, const double* initial_k, const double* initial_phi,
    double* k_out, double* phi_out, int32_t* outer_iterations, int64_t* inner_iterations, uint8_t* converged);

/* recast_source (paper Eq. 24): out = S + [(Ss0 - Ss0*) - (St - St*)] phi. */
snop_status snop_recast_source(
    snop_ctx* ctx, int32_t memspace, int32_t batch, int32_t n_cells, const double* source,
    const double* phi, const double* sigma_t, const double* sigma_s0, double sigma_t_star,
    double sigma_s0_star, double* out);

/* ---- SolutionOperators ---------------------------------------------
 * DenseNetwork parameters are packed per layer l as W_l [n_out][n_in] then b_l [n_out] (fp32).
 * (sigma_t_star, sigma_s0_star) is the reference parameter set p* the operator was built at
 * ("reference_params"); recast_* uses it.
 * FNO parameters (fp32) are packed as: lift_W [width][2], lift_b [width]; per layer:
 *   R_re [modes][width][width] (in,out), R_im [modes][width][width], W [width][width] (out,in),
 *   b [width]; then P1_W [hidden][width], P1_b [hidden], P2_W [hidden], P2_b [1].
 */
snop_status snop_deeponet_create(
    snop_ctx* ctx, const snop_grid* grid, double sigma_t_star, double sigma_s0_star, int32_t activation,
    int32_t n_branch_sizes, const int32_t* branch_sizes, const float* branch_params,
    int32_t n_trunk_sizes, const int32_t* trunk_sizes, const float* trunk_params,
    int32_t has_bias0, float bias0, snop_op** out);

snop_status snop_fno_create(
    snop_ctx* ctx, const snop_grid* grid, double sigma_t_star, double sigma_s0_star, int32_t activation, int32_t width, int32_t modes,
    int32_t n_layers, int32_t proj_hidden, const float* params, snop_op** out);

/* The "exact operator": the model-based solve at p* = (St*, Ss0*) wrapped as a
 * SolutionOperator; uses `cfg` for its inner solves. */
snop_status snop_exact_operator_create(
    snop_ctx* ctx, const snop_grid* grid, int32_t order, double sigma_t_star, double sigma_s0_star,
    const snop_solver_config* cfg, snop_op** out);

snop_status snop_op_destroy(snop_op* op);

/* save_model / load_model (file format SPEC.md:373): versioned little-endian
 * record + trailing FNV-1a-64 digest in the reference's binary container
 * (proj/core/include/snop/binary_io.hpp:12-62); record layout in csrc/model_io.h. Load errors
 * (missing file, bad magic, version mismatch, truncation, checksum failure) -> SNOP_IO_ERROR.
 * save -> load -> predict is bit-identical to predict before save. The exact operator has no
 * weights and cannot be saved (SNOP_INVALID_ARGUMENT). */
snop_status snop_op_save(const snop_op* op, const char* path);
snop_status snop_op_load(snop_ctx* ctx, const char* path, snop_op** out);
/* Host-only (no GPU needed): write a model file from parameters laid out as for
 * snop_deeponet_create / snop_fno_create, and read + validate a file's header. */
snop_status snop_model_write_deeponet(const char* path, const snop_grid* grid, double sigma_t_star,
                                      double sigma_s0_star, int32_t activation, int32_t n_branch,
                                      const int32_t* branch_sizes, const float* branch_params,
                                      int32_t n_trunk, const int32_t* trunk_sizes,
                                      const float* trunk_params, int32_t has_bias0, float bias0);
snop_status snop_model_write_fno(const char* path, const snop_grid* grid, double sigma_t_star,
                                 double sigma_s0_star, int32_t activation, int32_t width, int32_t modes,
                                 int32_t layers, int32_t hidden, const float* params);
snop_status snop_model_inspect(const char* path, snop_model_info* info);

/* predict(model, source) for a batch [B][Nc]; fp64 in/out, the neural
 * operators compute in fp32. */
snop_status snop_op_predict(snop_ctx* ctx, snop_op* op, int32_t memspace, int32_t batch,
                            const double* source, double* out);

/* recast_fixed_point: phi^{k+1} = op(recast(S, phi^k)), phi^0 = op(S) or
 * initial_phi. status[b] is snop_recast_status. */
snop_status snop_recast_fixed_point(
    snop_ctx* ctx, snop_op* op, int32_t memspace, int32_t batch, const double* source,
    const double* sigma_t, const double* sigma_s0, double recast_tolerance, int32_t recast_max_iterations,
    int32_t norm, const double* initial_phi, double* phi_out, int32_t* iterations, int32_t* status);

/* precondition_fixed_source (paper Eq. 10): recast fixed point, then the
 * batched source iteration on the full target problem warm-started from phi_NO. */
snop_status snop_precondition_fixed_source(
    snop_ctx* ctx, snop_op* op, int32_t memspace, int32_t order, int32_t batch,
    const double* sigma_t, const double* sigma_s0, const double* sigma_s1, const double* source,
    double recast_tolerance, int32_t recast_max_iterations, const snop_solver_config* cfg,
    double* phi_out, int32_t* precond_iterations, int32_t* recast_status,
    int32_t* refine_iterations, uint8_t* converged);

/* sp_eigen / cp_eigen (paper Appendix A2 Eqs. A5-A8), batched over instances.
 * Stage 1: power iteration whose within-group solve is the operator -- SP: recast fixed point
 * (against the operator's p*, within-group Sigma_t,g / Sigma_s0(g->g) recast, inter-group scatter
 * and fission as external source) warm-started from the current group flux, to recast_tolerance
 * or recast_max_iterations; CP: that prediction refined by a model-based source iteration.
 * Stage 2: model-based power iteration (as snop_power_iteration_batched) from (k_NO, phi_NO).
 * An instance whose stage 1 diverged or degenerated restarts stage 2 cold; fallback[b] = 1.
 * Layouts as snop_power_iteration_batched; the operator's grid is the problem grid. stage1_k =
 * k_NO; stage*_inner count recast iterations (+ refinement sweeps for CP) / sweeps. */
/* power_iteration(grid, quadrature, materials, config, inner_solver, initial) with a
 * neural-operator-backed inner_solver ("inner_solver is any procedure with the
 * source_iteration contract ... this indirection is what SP/CP plug into"): the power iteration whose
 * within-group solve is the operator -- stage 1 of SP (inner_solver = RECAST_FIXED_POINT, Eqs. A5-A6)
 * or of CP (PREDICT_REFINE, Eqs. A7-A8) on its own, from the flat start (k = 1). The model-based
 * inner solver is snop_power_iteration_batched. inner_iterations counts recast iterations (+ refinement
 * sweeps for PREDICT_REFINE); diverged[b] = 1 where the operator iteration diverged or the fission
 * integral degenerated (then converged[b] = 0 and k / phi hold the last iterate). */
typedef enum { SNOP_INNER_RECAST_FIXED_POINT = 0, SNOP_INNER_PREDICT_REFINE = 1 } snop_inner_solver;
snop_status snop_power_iteration_operator_batched(
    snop_ctx* ctx, snop_op* op, int32_t inner_solver, int32_t memspace, int32_t order, int32_t batch,
    int32_t n_groups, const double* sigma_t, const double* sigma_s0, const double* sigma_s1,
    const double* nu_sigma_f, const double* chi, const snop_solver_config* cfg, double recast_tolerance,
    int32_t recast_max_iterations, double* k_out, double* phi_out, int32_t* outer_iterations,
    int64_t* inner_iterations, uint8_t* converged, uint8_t* diverged);

snop_status snop_sp_eigen_batched(
    snop_ctx* ctx, snop_op* op, int32_t memspace, int32_t order, int32_t batch, int32_t n_groups,
    const double* sigma_t, const double* sigma_s0, const double* sigma_s1, const double* nu_sigma_f,
    const double* chi, const snop_solver_config* cfg, double recast_tolerance,
    int32_t recast_max_iterations, double* k_out, double* phi_out, double* stage1_k,
    int32_t* stage1_outer, int64_t* stage1_inner, int32_t* stage2_outer, int64_t* stage2_inner,
    uint8_t* converged, uint8_t* fallback);

snop_status snop_cp_eigen_batched(
    snop_ctx* ctx, snop_op* op, int32_t memspace, int32_t order, int32_t batch, int32_t n_groups,
    const double* sigma_t, const double* sigma_s0, const double* sigma_s1, const double* nu_sigma_f,
    const double* chi, const snop_solver_config* cfg, double recast_tolerance,
    int32_t recast_max_iterations, double* k_out, double* phi_out, double* stage1_k,
    int32_t* stage1_outer, int64_t* stage1_inner, int32_t* stage2_outer, int64_t* stage2_inner,
    uint8_t* converged, uint8_t* fallback);

/* sample_grf: field[s][i] = mean + (L z_s)_i, L L^T = C + jitter variance I
 * (squared-exponential kernel at the cell centres; jitter relative to the variance, escalated x10
 * up to 1e-6), z_s = the first n_cells
 * normals of snop::Rng(seed + first_sample + s) (rng.hpp:17-49). negatives[s] (nullable) counts
 * negative entries (reported, never clipped). n_cells >= 2. */
snop_status snop_grf_sample(snop_ctx* ctx, int32_t memspace, const snop_grid* grid, const snop_grf_spec* spec,
                            int64_t first_sample, int32_t n_samples, double* field_out, int64_t* negatives);

/* normalize_source (paper Eq. 13): out = raw / (dx sum raw) per sample;
 * SNOP_INVALID_ARGUMENT naming the first sample whose integral is <= 0. */
snop_status snop_normalize_source(snop_ctx* ctx, int32_t memspace, const snop_grid* grid, int32_t n_samples,
                                  const double* raw, double* out);

/* generate_dataset: sample s = normalize(sample_grf(seed + s)) and its flux from
 * the source iteration at p* = (sigma_t*, sigma_s0*) (vacuum, zero initial guess, tolerance).
 * Any non-convergent sample -> SNOP_NUMERICAL_ERROR naming the sample index. */
snop_status snop_generate_dataset(snop_ctx* ctx, int32_t memspace, const snop_grid* grid, int32_t order,
                                  const snop_grf_spec* spec, int32_t n_samples, double sigma_t_star,
                                  double sigma_s0_star, double tolerance, double* sources, double* fluxes,
                                  int32_t* iterations);

/* Dataset file, host-only: versioned header (format version, n_samples, n_cells,
 * grid, GRF spec, p*, solver tolerance), sources then fluxes as row-major little-endian f64, and
 * a trailing FNV-1a-64 digest (the reference container, binary_io.hpp:12-62); a text manifest is
 * written alongside at "<path>.txt". snop_dataset_read fills info and, when non-NULL, the
 * [n_samples][n_cells] arrays (call once with NULL arrays to size them). */
snop_status snop_dataset_write(const char* path, const snop_dataset_info* info, const double* sources,
                               const double* fluxes);
snop_status snop_dataset_read(const char* path, snop_dataset_info* info, double* sources, double* fluxes);

#ifdef __cplusplus
}
#endif
#endif /* SNOP_CUDA_H */
