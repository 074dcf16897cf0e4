// snop ORACLE — TEST INFRASTRUCTURE ONLY (see snop_oracle.hpp header).
// Each function cites the SPEC contract it restates.
#include "snop_oracle.hpp"

#include <algorithm>
#include <atomic>
#include <thread>

namespace snop::oracle {

// parallel.hpp:17-48 — fixed partition independent of thread count.
void parallel_chunks(std::size_t n_items, std::size_t n_chunks,
                     const std::function<void(std::size_t, std::size_t, std::size_t)>& fn,
                     unsigned n_threads) {
  if (n_items == 0) return;
  if (n_chunks == 0 || n_chunks > n_items) n_chunks = n_items;
  if (n_threads == 0) n_threads = std::thread::hardware_concurrency();
  if (n_threads == 0) n_threads = 1;
  const std::size_t base = n_items / n_chunks, extra = n_items % n_chunks;
  auto begin_of = [&](std::size_t c) { return c * base + std::min(c, extra); };
  if (n_threads == 1 || n_chunks == 1) {
    for (std::size_t c = 0; c < n_chunks; ++c) fn(c, begin_of(c), begin_of(c + 1));
    return;
  }
  std::atomic<std::size_t> next{0};
  auto worker = [&] {
    for (;;) {
      const std::size_t c = next.fetch_add(1);
      if (c >= n_chunks) return;
      fn(c, begin_of(c), begin_of(c + 1));
    }
  };
  const unsigned n = static_cast<unsigned>(std::min<std::size_t>(n_threads, n_chunks));
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < n; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
}

// SPEC.md:64-72. Newton on P_N from the Chebyshev-like initial guess; nodes mirrored so the
// set is exactly symmetric and sorted ascending.
Quadrature gauss_legendre(int order) {
  if (order < 2 || order > 128 || order % 2 != 0)
    throw InvalidArgument("gauss_legendre: order must be even in [2,128]");
  Quadrature q;
  q.order = order;
  q.mu.assign(order, 0.0);
  q.w.assign(order, 0.0);
  const int N = order;
  for (int i = 0; i < N / 2; ++i) {
    double x = std::cos(std::numbers::pi * (i + 0.75) / (N + 0.5));
    double dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= N; ++k) {
        const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = N * (x * p1 - p0) / (x * x - 1.0);
      const double dx = p1 / dp;
      x -= dx;
      if (std::fabs(dx) < 1e-16) break;
    }
    {  // final derivative at the converged node
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= N; ++k) {
        const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = N * (x * p1 - p0) / (x * x - 1.0);
    }
    const double wt = 2.0 / ((1.0 - x * x) * dp * dp);
    q.mu[N - 1 - i] = x;   // largest positive first from the top
    q.mu[i] = -x;
    q.w[N - 1 - i] = wt;
    q.w[i] = wt;
  }
  return q;
}

// SPEC.md:74-82
double integrate_cellwise(const double* f, const Grid1D& g) {
  double s = 0.0;
  for (int i = 0; i < g.n_cells; ++i) s += f[i];
  return s * g.dx();
}

// SPEC.md:58,92 (relative L-inf default, relative L2 option). Zero-denominator rule (pinned,
// SURVEY §9 #1): 0/0 -> 0 (converged), x/0 -> inf.
double relative_change(const double* a_new, const double* a_old, std::size_t n, Norm norm) {
  double num = 0.0, den = 0.0;
  if (norm == Norm::RelLinf) {
    for (std::size_t i = 0; i < n; ++i) {
      num = std::max(num, std::fabs(a_new[i] - a_old[i]));
      den = std::max(den, std::fabs(a_new[i]));
    }
  } else {
    for (std::size_t i = 0; i < n; ++i) {
      const double d = a_new[i] - a_old[i];
      num += d * d;
      den += a_new[i] * a_new[i];
    }
    num = std::sqrt(num);
    den = std::sqrt(den);
  }
  if (den > 0.0) return num / den;
  return num > 0.0 ? INFINITY : 0.0;
}

// SPEC.md:115-123 diamond difference sweep. Direction order with reflective faces pinned in
// reflective-left -> mu<0 first, then mu>0 fed by the mirrored outflow of the
// same sweep; reflective-right only -> mu>0 first; both reflective -> the right face lags one
// sweep (lag_right holds the previous mu>0 outflow per positive direction).
// out_left/out_right are NET leakages (outgoing minus incoming partial currents).
void sweep(const Grid1D& g, const Quadrature& q, const double* sigma_t, const double* emission,
           Boundary left, Boundary right, double* psi_avg, double* out_left, double* out_right,
           std::vector<double>* lag_right) {
  const int Nc = g.n_cells, N = q.order, H = N / 2;
  const double dx = g.dx();
  for (int i = 0; i < Nc; ++i)
    if (!(sigma_t[i] > 0.0)) throw InvalidArgument("sweep: nonpositive sigma_t");
  std::vector<double> left_out(H, 0.0), right_out(H, 0.0);  // indexed by pair p (n+ = H+p)
  auto sweep_neg = [&](int p, double psi_in) {  // direction n = H-1-p (mu<0), right -> left
    const int n = H - 1 - p;
    const double c = 2.0 * std::fabs(q.mu[n]) / dx;
    double psi = psi_in;
    for (int i = Nc - 1; i >= 0; --i) {
      const double avg = (emission[(std::size_t)i * N + n] + c * psi) / (sigma_t[i] + c);
      psi_avg[(std::size_t)n * Nc + i] = avg;
      psi = 2.0 * avg - psi;
    }
    left_out[p] = psi;
  };
  auto sweep_pos = [&](int p, double psi_in) {  // direction n = H+p (mu>0), left -> right
    const int n = H + p;
    const double c = 2.0 * q.mu[n] / dx;
    double psi = psi_in;
    for (int i = 0; i < Nc; ++i) {
      const double avg = (emission[(std::size_t)i * N + n] + c * psi) / (sigma_t[i] + c);
      psi_avg[(std::size_t)n * Nc + i] = avg;
      psi = 2.0 * avg - psi;
    }
    right_out[p] = psi;
  };
  std::vector<double> in_left(H, 0.0), in_right(H, 0.0);
  const bool rl = left == Boundary::Reflective, rr = right == Boundary::Reflective;
  if (rr && !rl) {
    for (int p = 0; p < H; ++p) sweep_pos(p, 0.0);
    for (int p = 0; p < H; ++p) { in_right[p] = right_out[p]; sweep_neg(p, in_right[p]); }
  } else {
    for (int p = 0; p < H; ++p) {
      in_right[p] = (rr && lag_right) ? (*lag_right)[p] : 0.0;
      sweep_neg(p, in_right[p]);
    }
    for (int p = 0; p < H; ++p) {
      in_left[p] = rl ? left_out[p] : 0.0;
      sweep_pos(p, in_left[p]);
    }
    if (rr && lag_right) *lag_right = right_out;
  }
  double ol = 0.0, orr = 0.0;
  for (int p = 0; p < H; ++p) {
    const double wm = q.w[H + p] * q.mu[H + p];
    ol += wm * (left_out[p] - in_left[p]);
    orr += wm * (right_out[p] - in_right[p]);
  }
  if (out_left) *out_left = ol;
  if (out_right) *out_right = orr;
}

// SPEC.md:125-134. Emission q = 1/2 Ss0 phi + 3/2 Ss1 mu J + 1/2 S; phi = sum_n w psi_avg in
// ascending n (fixed order); count = sweeps.
SIResult source_iteration(const Grid1D& g, const Quadrature& q, const double* sigma_t,
                          const double* sigma_s0, const double* sigma_s1, const double* source,
                          const SolverConfig& cfg, double* phi, double* current) {
  const int Nc = g.n_cells, N = q.order;
  std::vector<double> emission((std::size_t)Nc * N), psi((std::size_t)N * Nc), phin(Nc), J(Nc, 0.0),
      Jn(Nc);
  std::vector<double> lag(N / 2, 0.0);
  SIResult res;
  for (int it = 1; it <= cfg.max_inner; ++it) {
    for (int i = 0; i < Nc; ++i) {
      const double iso = 0.5 * sigma_s0[i] * phi[i] + 0.5 * source[i];
      for (int n = 0; n < N; ++n) {
        double e = iso;
        if (sigma_s1) e += 1.5 * sigma_s1[i] * q.mu[n] * J[i];
        emission[(std::size_t)i * N + n] = e;
      }
    }
    sweep(g, q, sigma_t, emission.data(), cfg.left, cfg.right, psi.data(), &res.out_left,
          &res.out_right, &lag);
    for (int i = 0; i < Nc; ++i) {
      double s = 0.0, j = 0.0;
      for (int n = 0; n < N; ++n) {
        const double a = psi[(std::size_t)n * Nc + i];
        s += q.w[n] * a;
        j += q.w[n] * q.mu[n] * a;
      }
      phin[i] = s;
      Jn[i] = j;
    }
    const double rel = relative_change(phin.data(), phi, Nc, cfg.norm);
    std::copy(phin.begin(), phin.end(), phi);
    J = Jn;
    res.iterations = it;
    if (!std::isfinite(rel) && rel != INFINITY) throw NumericalError("source_iteration: non-finite flux");
    if (rel < cfg.tolerance) { res.converged = true; break; }
  }
  if (current) std::copy(J.begin(), J.end(), current);
  return res;
}

// SPEC.md:136-144
double balance_residual(const Grid1D& g, const double* sigma_t, const double* sigma_s0_out,
                        const double* source, const double* phi, double out_left, double out_right) {
  double absorption = 0.0, production = 0.0;
  for (int i = 0; i < g.n_cells; ++i) {
    absorption += (sigma_t[i] - sigma_s0_out[i]) * phi[i];
    production += source[i];
  }
  absorption *= g.dx();
  production *= g.dx();
  if (production == 0.0) throw NumericalError("balance_residual: zero production");
  return std::fabs(out_left + out_right + absorption - production) / std::fabs(production);
}

// SPEC.md:179-189 with decisions :206-209 and SURVEY §9 #5 (Gauss-Seidel over groups using the
// newest flux of every other group, upscatter included), #10 (inner solves warm-started from the
// current normalised flux). Fission source is frozen at the start of each outer.
EigenResult power_iteration(const Grid1D& grid, const Quadrature& q, const MGView& m,
                            const SolverConfig& cfg, double* phi, bool has_initial, double initial_k,
                            const InnerSolver* inner) {
  const int G = m.G, Nc = grid.n_cells;
  const std::size_t n = (std::size_t)G * Nc;
  if (!has_initial) std::fill(phi, phi + n, 1.0);
  EigenResult res;
  res.k = has_initial ? initial_k : 1.0;
  if (!(res.k > 0.0)) throw InvalidArgument("power_iteration: initial k must be positive");
  auto fission_integral = [&](const double* f) {
    double s = 0.0;
    for (int i = 0; i < Nc; ++i) {
      double fi = 0.0;
      for (int g = 0; g < G; ++g) fi += m.nu_sigma_f[(std::size_t)g * Nc + i] * f[(std::size_t)g * Nc + i];
      s += fi;
    }
    return s * grid.dx();
  };
  double f0 = fission_integral(phi);
  if (!(f0 != 0.0) || !std::isfinite(f0)) throw DegenerateProblem("power_iteration: zero fission integral");
  for (std::size_t i = 0; i < n; ++i) phi[i] /= f0;

  std::vector<double> old(n), fiss(Nc), qext(Nc);
  SolverConfig icfg = cfg;
  InnerSolver default_inner = [&](int g, const double* qe, double* phig) {
    const SIResult r = source_iteration(grid, q, m.sigma_t + (std::size_t)g * Nc,
                                        m.sigma_s0 + ((std::size_t)g * G + g) * Nc,
                                        m.sigma_s1 ? m.sigma_s1 + (std::size_t)g * Nc : nullptr, qe, icfg,
                                        phig, nullptr);
    return r.iterations;
  };
  const InnerSolver& solve = inner ? *inner : default_inner;

  for (int outer = 1; outer <= cfg.max_outer; ++outer) {
    std::copy(phi, phi + n, old.begin());
    for (int i = 0; i < Nc; ++i) {
      double fi = 0.0;
      for (int g = 0; g < G; ++g) fi += m.nu_sigma_f[(std::size_t)g * Nc + i] * phi[(std::size_t)g * Nc + i];
      fiss[i] = fi;
    }
    for (int g = 0; g < G; ++g) {
      for (int i = 0; i < Nc; ++i) {
        double s = m.chi[g] * fiss[i] / res.k;
        for (int gp = 0; gp < G; ++gp) {
          if (gp == g) continue;
          s += m.sigma_s0[((std::size_t)gp * G + g) * Nc + i] * phi[(std::size_t)gp * Nc + i];
        }
        qext[i] = s;
      }
      res.inner += solve(g, qext.data(), phi + (std::size_t)g * Nc);
    }
    const double f1 = fission_integral(phi);
    if (!(f1 != 0.0) || !std::isfinite(f1)) throw DegenerateProblem("power_iteration: zero fission integral");
    const double k_new = res.k * f1;  // old flux normalised to unit fission integral
    for (std::size_t i = 0; i < n; ++i) phi[i] /= f1;
    const double dk = std::fabs(k_new - res.k) / std::fabs(k_new);
    const double dphi = relative_change(phi, old.data(), n, cfg.norm);
    res.k = k_new;
    res.outer = outer;
    if (dk < cfg.tolerance_k && dphi < cfg.tolerance_phi) { res.converged = true; break; }
  }
  return res;
}

// k = nuSf^T (Sigma_t - S^T)^{-1} chi (the fission operator is rank one).
double infinite_medium_k(int G, const double* st, const double* ss0, const double* nsf, const double* chi) {
  std::vector<double> A((std::size_t)G * G), x(chi, chi + G);
  for (int g = 0; g < G; ++g)
    for (int gp = 0; gp < G; ++gp) A[(std::size_t)g * G + gp] = (g == gp ? st[g] : 0.0) - ss0[(std::size_t)gp * G + g];
  for (int c = 0; c < G; ++c) {
    int piv = c;
    for (int r = c + 1; r < G; ++r)
      if (std::fabs(A[(std::size_t)r * G + c]) > std::fabs(A[(std::size_t)piv * G + c])) piv = r;
    if (std::fabs(A[(std::size_t)piv * G + c]) < 1e-300) throw DegenerateProblem("infinite_medium_k: singular");
    if (piv != c) {
      for (int k = 0; k < G; ++k) std::swap(A[(std::size_t)c * G + k], A[(std::size_t)piv * G + k]);
      std::swap(x[c], x[piv]);
    }
    for (int r = c + 1; r < G; ++r) {
      const double f = A[(std::size_t)r * G + c] / A[(std::size_t)c * G + c];
      for (int k = c; k < G; ++k) A[(std::size_t)r * G + k] -= f * A[(std::size_t)c * G + k];
      x[r] -= f * x[c];
    }
  }
  for (int r = G - 1; r >= 0; --r) {
    double s = x[r];
    for (int k = r + 1; k < G; ++k) s -= A[(std::size_t)r * G + k] * x[k];
    x[r] = s / A[(std::size_t)r * G + r];
  }
  double k = 0.0;
  for (int g = 0; g < G; ++g) k += nsf[g] * x[g];
  if (!(k > 0.0)) throw DegenerateProblem("infinite_medium_k: no fission");
  return k;
}

// affine layers, activation on hidden layers, linear output.
void dense_forward(const DenseNetwork& net, const double* in, double* out) {
  const int L = (int)net.sizes.size() - 1;
  std::vector<double> h(in, in + net.sizes[0]), nx;
  for (int l = 0; l < L; ++l) {
    const int ni = net.sizes[l], no = net.sizes[l + 1];
    nx.assign(no, 0.0);
    for (int o = 0; o < no; ++o) {
      double s = net.b[l][o];
      const float* w = net.W[l].data() + (std::size_t)o * ni;
      for (int i = 0; i < ni; ++i) s += (double)w[i] * h[i];
      nx[o] = (l + 1 < L) ? activate(s, net.act) : s;
    }
    h.swap(nx);
  }
  std::copy(h.begin(), h.end(), out);
}

// SPEC.md:300-304,319-322; paper Eq. 11.
void deeponet_predict(const DeepONet& m, const Grid1D& g, const double* source, double* out) {
  const int p = m.branch.sizes.back();
  std::vector<double> in(m.branch.sizes[0]);
  for (int i = 0; i < m.branch.sizes[0]; ++i) in[i] = (double)(float)source[i];  // fp32 operator input
  std::vector<double> b(p), t(p);
  dense_forward(m.branch, in.data(), b.data());
  for (int i = 0; i < g.n_cells; ++i) {
    const double x = (double)(float)g.center(i);
    dense_forward(m.trunk, &x, t.data());
    double s = m.has_bias0 ? (double)m.bias0 : 0.0;
    for (int k = 0; k < p; ++k) s += b[k] * t[k];
    out[i] = s;
  }
}

// SPEC.md:306-311,322,368 (+ SURVEY §9 #9): unnormalised truncated rDFT over modes 0..M-1,
// complex mixing R[m][in][out], inverse with 1/n and conjugate symmetry (imaginary part of DC
// and of a Nyquist mode dropped), pointwise W path + bias, activation after every layer.
void fno_predict(const FNO& m, const Grid1D& g, const double* source, double* out) {
  const int n = g.n_cells, C = m.width, M = m.modes;
  std::vector<double> v((std::size_t)C * n), vn((std::size_t)C * n);
  for (int c = 0; c < C; ++c)
    for (int i = 0; i < n; ++i)
      v[(std::size_t)c * n + i] = (double)m.lift_W[c * 2 + 0] * (double)(float)source[i] +
                                  (double)m.lift_W[c * 2 + 1] * (double)(float)g.center(i) +
                                  (double)m.lift_b[c];
  std::vector<double> cs((std::size_t)M * n), sn((std::size_t)M * n);
  for (int k = 0; k < M; ++k)
    for (int i = 0; i < n; ++i) {
      const double ang = 2.0 * std::numbers::pi * (double)(((long long)k * i) % n) / n;
      cs[(std::size_t)k * n + i] = std::cos(ang);
      sn[(std::size_t)k * n + i] = std::sin(ang);
    }
  std::vector<double> Vr((std::size_t)M * C), Vi((std::size_t)M * C), Ur((std::size_t)M * C), Ui((std::size_t)M * C);
  for (int l = 0; l < m.layers; ++l) {
    for (int k = 0; k < M; ++k)
      for (int c = 0; c < C; ++c) {
        double re = 0.0, im = 0.0;
        for (int i = 0; i < n; ++i) {
          re += v[(std::size_t)c * n + i] * cs[(std::size_t)k * n + i];
          im -= v[(std::size_t)c * n + i] * sn[(std::size_t)k * n + i];
        }
        Vr[(std::size_t)k * C + c] = re;
        Vi[(std::size_t)k * C + c] = im;
      }
    const float* Rr = m.R_re[l].data();
    const float* Ri = m.R_im[l].data();
    for (int k = 0; k < M; ++k)
      for (int o = 0; o < C; ++o) {
        double re = 0.0, im = 0.0;
        for (int c = 0; c < C; ++c) {
          const double a = Rr[((std::size_t)k * C + c) * C + o], b = Ri[((std::size_t)k * C + c) * C + o];
          re += a * Vr[(std::size_t)k * C + c] - b * Vi[(std::size_t)k * C + c];
          im += a * Vi[(std::size_t)k * C + c] + b * Vr[(std::size_t)k * C + c];
        }
        Ur[(std::size_t)k * C + o] = re;
        Ui[(std::size_t)k * C + o] = im;
      }
    for (int o = 0; o < C; ++o)
      for (int i = 0; i < n; ++i) {
        double s = Ur[o];  // DC: real part only
        for (int k = 1; k < M; ++k) {
          const double wgt = (2 * k == n) ? 1.0 : 2.0;
          const double re = Ur[(std::size_t)k * C + o] * cs[(std::size_t)k * n + i];
          const double im = (2 * k == n) ? 0.0 : Ui[(std::size_t)k * C + o] * sn[(std::size_t)k * n + i];
          s += wgt * (re - im);
        }
        double wv = m.b[l][o];
        const float* Wrow = m.W[l].data() + (std::size_t)o * C;
        for (int c = 0; c < C; ++c) wv += (double)Wrow[c] * v[(std::size_t)c * n + i];
        vn[(std::size_t)o * n + i] = activate(s / n + wv, m.act);
      }
    v.swap(vn);
  }
  const int Hd = m.proj_hidden;
  std::vector<double> h(Hd);
  for (int i = 0; i < n; ++i) {
    for (int k = 0; k < Hd; ++k) {
      double s = m.P1_b[k];
      for (int c = 0; c < C; ++c) s += (double)m.P1_W[(std::size_t)k * C + c] * v[(std::size_t)c * n + i];
      h[k] = activate(s, m.act);
    }
    double s = m.P2_b[0];
    for (int k = 0; k < Hd; ++k) s += (double)m.P2_W[k] * h[k];
    out[i] = s;
  }
}

// SPEC.md:393-401; paper Eq. 24 (isotropic approximation Eq. 23).
void recast_source(int n, const double* S, const double* phi, const double* st, const double* ss0,
                   double tstar, double sstar, double* out) {
  for (int i = 0; i < n; ++i) out[i] = S[i] + ((ss0[i] - sstar) - (st[i] - tstar)) * phi[i];
}

// SPEC.md:403-411. phi0 = op(S) unless an initial flux is given (Eq. 9); divergence guard at
// 1e6 x the initial max-norm (or any non-finite value) returns phi0 — the "best available
// iterate" handed to refinement (pinned in DESIGN.md).
RecastResult recast_fixed_point(int n, const double* S, const double* st, const double* ss0, double tstar,
                                double sstar, const SolutionOperator& op, double tol, int max_it, Norm norm,
                                const double* initial_phi, double* phi_out) {
  std::vector<double> phi0(n), phi(n), s(n), nx(n);
  if (initial_phi) std::copy(initial_phi, initial_phi + n, phi0.begin());
  else op(S, phi0.data());
  double norm0 = 0.0;
  for (double v : phi0) norm0 = std::max(norm0, std::fabs(v));
  phi = phi0;
  RecastResult r;
  r.status = RecastStatus::MaxIterations;
  for (int it = 1; it <= max_it; ++it) {
    recast_source(n, S, phi.data(), st, ss0, tstar, sstar, s.data());
    op(s.data(), nx.data());
    double mx = 0.0;
    bool finite = true;
    for (double v : nx) { finite = finite && std::isfinite(v); mx = std::max(mx, std::fabs(v)); }
    r.iterations = it;
    if (!finite || (norm0 > 0.0 && mx > 1e6 * norm0)) {
      r.status = RecastStatus::Diverged;
      phi = phi0;
      break;
    }
    const double rel = relative_change(nx.data(), phi.data(), n, norm);
    phi = nx;
    if (rel < tol) { r.status = RecastStatus::Converged; break; }
  }
  std::copy(phi.begin(), phi.end(), phi_out);
  return r;
}

// --- grf -----------------------------------------------------------------------
std::vector<double> grf_cholesky(const Grid1D& g, const GrfSpec& spec, double* jitter_used) {
  if (!(spec.variance > 0.0) || !(spec.length_scale > 0.0) || !(spec.jitter > 0.0))
    throw InvalidArgument("grf: variance, length scale and jitter must be positive");
  if (g.n_cells < 2) throw InvalidArgument("grf: n_cells must be >= 2");
  const int n = g.n_cells;
  const double inv2l2 = 1.0 / (2.0 * spec.length_scale * spec.length_scale);
  std::vector<double> L((std::size_t)n * n);
  for (double jitter = spec.jitter; jitter <= 1e-6 * (1.0 + 1e-12); jitter *= 10.0) {
    std::fill(L.begin(), L.end(), 0.0);
    bool ok = true;
    for (int i = 0; i < n && ok; ++i) {
      for (int j = 0; j <= i; ++j) {
        const double d = g.center(i) - g.center(j);
        double s = spec.variance * (std::exp(-d * d * inv2l2) + (i == j ? jitter : 0.0));
        for (int k = 0; k < j; ++k) s -= L[(std::size_t)i * n + k] * L[(std::size_t)j * n + k];
        if (i == j) {
          if (!(s > 0.0)) { ok = false; break; }
          L[(std::size_t)i * n + i] = std::sqrt(s);
        } else {
          L[(std::size_t)i * n + j] = s / L[(std::size_t)j * n + j];
        }
      }
    }
    if (ok) {
      if (jitter_used) *jitter_used = jitter;
      return L;
    }
  }
  throw NumericalError("grf: covariance factorization failed after jitter escalation to 1e-6");
}

long long sample_grf(const Grid1D& g, const GrfSpec& spec, const std::vector<double>& L, std::uint64_t sample,
                     double* out) {
  const int n = g.n_cells;
  Rng r(spec.seed + sample);
  std::vector<double> z(n);
  for (int j = 0; j < n; ++j) z[j] = r.normal();
  long long neg = 0;
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int j = 0; j <= i; ++j) s += L[(std::size_t)i * n + j] * z[j];
    out[i] = spec.mean + s;
    neg += out[i] < 0.0;
  }
  return neg;
}

void normalize_source(const Grid1D& g, const double* raw, double* out) {
  double s = 0.0;
  for (int i = 0; i < g.n_cells; ++i) s += raw[i];
  s *= g.dx();
  if (!(s > 0.0) || !std::isfinite(s)) throw InvalidArgument("normalize_source: non-positive integral (resample)");
  for (int i = 0; i < g.n_cells; ++i) out[i] = raw[i] / s;
}

}  // namespace snop::oracle
