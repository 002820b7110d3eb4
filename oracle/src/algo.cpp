// Oracle HALLaR algorithm: AL core, ADAP-FISTA, ADAP-AIPP, thick-restart
// Lanczos, HLR inner method, outer AL driver + certificate.  Restates the
// reference sdp_instance.cpp, adap_fista.cpp, adap_aipp.cpp, lanczos.cpp,
// hlr.cpp and solver.cpp statement by statement (cited per function).
// TEST INFRASTRUCTURE ONLY (see orc.hpp).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <limits>

#include "orc.hpp"

namespace orc {

namespace {
void check_mult(const Instance& I, const Vec& p, const char* where) {
  if (i64(p.size()) != I.m)
    throw InputError(std::string(where) + ": multiplier has length " +
                     std::to_string(p.size()) + ", instance needs " + std::to_string(I.m));
}
void check_fin(double v, const char* where) {
  if (!std::isfinite(v)) throw NumericalError(std::string(where) + ": non-finite result");
}
Vec residual_of(const Instance& I, const Mat& U) {
  Vec r = I.apply_map(U);
  for (i64 k = 0; k < I.m; ++k) r[k] = r[k] - I.b[k];
  return r;
}
Vec q_of(const Vec& p, double beta, const Vec& r) {
  Vec q(r.size());
  for (size_t k = 0; k < r.size(); ++k) q[k] = p[k] + beta * r[k];
  return q;
}
Mat sub(const Mat& a, const Mat& b) {
  Mat o(a.rows, a.cols);
  for (i64 t = 0; t < a.size(); ++t) o.a[t] = a.a[t] - b.a[t];
  return o;
}
double sqdist(const Mat& a, const Mat& b) {
  return esum_fn(a.size(), [&](i64 t) {
    const double d = a.a[t] - b.a[t];
    return d * d;
  });
}
}  // namespace

// Debug record of every fista() call (ORC_DEBUG_FISTA=<file>): used to locate
// the first divergence between the parity-mode device solve and this checker.
static void dbg_fista(double L0, int status, int iters, double L, double psi_y, int cap) {
  static FILE* f = [] {
    const char* p = std::getenv("ORC_DEBUG_FISTA");
    return p ? std::fopen(p, "w") : nullptr;
  }();
  if (f) {
    std::fprintf(f, "%.17g %d %d %.17g %.17g %d\n", L0, status, iters, L, psi_y, cap);
    std::fflush(f);
  }
}

// ------------------------------------------------------------- AL core ---
// sdp_instance.cpp:50-60
double al_value(const Instance& I, const Mat& U, const Vec& p, double beta) {
  I.check_dims(U, "al_value");
  check_mult(I, p, "al_value");
  need(beta > 0, "al_value: beta must be positive");
  const Vec r = residual_of(I, U);
  const double cdot = frob_dot(I.apply_C(U), U);
  const double val = cdot + dot(p, r) + 0.5 * beta * sqnorm(r);
  check_fin(val, "al_value");
  return val;
}

// sdp_instance.cpp:62-71
Mat al_gradient(const Instance& I, const Mat& U, const Vec& p, double beta) {
  I.check_dims(U, "al_gradient");
  check_mult(I, p, "al_gradient");
  need(beta > 0, "al_gradient: beta must be positive");
  const Vec q = q_of(p, beta, residual_of(I, U));
  Mat g = I.C_plus_adjoint(q, U);
  for (auto& x : g.a) x = 2.0 * x;
  if (!all_finite(g)) throw NumericalError("al_gradient: non-finite result");
  return g;
}

// sdp_instance.cpp:73-92
GradOp::GradOp(const Instance& inst, const Mat& U, const Vec& p, double beta) : I(&inst) {
  inst.check_dims(U, "gradient_operator");
  check_mult(inst, p, "gradient_operator");
  need(beta > 0, "gradient_operator: beta must be positive");
  residual = residual_of(inst, U);
  q = q_of(p, beta, residual);
  if (!all_finite(q)) throw NumericalError("gradient_operator: non-finite multiplier");
}
Mat GradOp::apply(const Mat& V) const {
  I->check_dims(V, "gradient_operator::apply");
  return I->C_plus_adjoint(q, V);
}
Vec GradOp::apply_vec(const Vec& v) const {
  Mat V(i64(v.size()), 1);
  V.a = v;
  return apply(V).a;
}

// sdp_instance.cpp:94-99
Mat project_ball(const Mat& U) {
  if (!all_finite(U)) throw InputError("project_ball: non-finite input");
  const double nrm = norm(U);
  if (nrm <= 1.0) return U;
  Mat o = U;
  for (auto& x : o.a) x = x / nrm;
  return o;
}

double AlFn::value(const Mat& U) const { return al_value(*I, U, p, beta); }
Mat AlFn::gradient(const Mat& U) const { return al_gradient(*I, U, p, beta); }
// sdp_instance.cpp:115-127 (adjoint identity for C.UU^T)
std::pair<double, Mat> AlFn::value_and_gradient(const Mat& U) const {
  I->check_dims(U, "AlFunction::value_and_gradient");
  const Vec r = residual_of(*I, U);
  const Vec q = q_of(p, beta, r);
  Mat h = I->C_plus_adjoint(q, U);
  const double qrb = esum_fn(I->m, [&](i64 k) { return q[k] * (r[k] + I->b[k]); });
  const double cdot = frob_dot(h, U) - qrb;
  const double val = cdot + dot(p, r) + 0.5 * beta * sqnorm(r);
  check_fin(val, "AlFunction::value_and_gradient");
  for (auto& x : h.a) x = 2.0 * x;
  return {val, std::move(h)};
}

// ---------------------------------------------------------- ADAP-FISTA ---
void FistaParams::validate() const {
  need(sigma > 0 && sigma < 0.5, "fista: sigma must lie in (0, 1/2)");
  need(chi > 0 && chi < 1, "fista: chi must lie in (0, 1)");
  need(mu > 0, "fista: mu must be positive");
  need(L0 > mu, "fista: L0 must exceed mu");
}

// adap_fista.cpp:14-103
FistaResult fista(const Smooth& psi, const Mat& x0, const FistaParams& prm) {
  prm.validate();
  need(norm(x0) <= 1.0 + 1e-12, "fista: x0 outside the unit ball");
  const double mu = prm.mu, chi = prm.chi, sigma = prm.sigma;
  double A = 0.0, tau = 1.0, L = prm.L0;
  Mat x = x0, y = x0;
  FistaResult out;
  for (int it = 0;; ++it) {
    const int cap = prm.max_iters > 0
                        ? prm.max_iters
                        : 50 + int(10.0 * std::sqrt(L / mu) * std::log2(4.0 + L / prm.L0));
    if (it >= cap) {
      out.status = FistaStatus::kIterLimit;
      out.y = y;
      out.v = Mat(x0.rows, x0.cols);
      out.L = L;
      out.iters = it;
      dbg_fista(prm.L0, 2, it, L, 0.0, cap);
      return out;
    }
    double a = 0, psi_t = 0, psi_n = 0, dsq = 0;
    Mat xt, gt, yn;
    for (;;) {
      a = (tau + std::sqrt(tau * tau + 4.0 * tau * A * (L - mu))) / (2.0 * (L - mu));
      xt = Mat(x.rows, x.cols);
      for (i64 t = 0; t < x.size(); ++t) xt.a[t] = (A * y.a[t] + a * x.a[t]) / (A + a);
      auto ev = psi.eval(xt);
      psi_t = ev.first;
      gt = std::move(ev.second);
      Mat z(x.rows, x.cols);
      for (i64 t = 0; t < x.size(); ++t) z.a[t] = xt.a[t] - gt.a[t] / L;
      yn = project_ball(z);
      psi_n = psi.value(yn);
      dsq = sqdist(yn, xt);
      const double lin = psi_t + esum_fn(x.size(), [&](i64 t) {
                           return gt.a[t] * (yn.a[t] - xt.a[t]);
                         });
      const double noise = 1e-14 * (std::fabs(psi_n) + std::fabs(psi_t) + 1.0);
      if (lin + (1.0 - chi) * L / 4.0 * dsq >= psi_n - noise) break;
      L *= 2.0;
      if (L > 1e18) throw NumericalError("fista: curvature estimate diverged");
    }
    const double A_next = A + a;
    tau += a * mu;
    for (i64 t = 0; t < x.size(); ++t) {
      const double s = (L - mu) * (xt.a[t] - yn.a[t]);
      x.a[t] = (mu * a * yn.a[t] + (tau - a * mu) * x.a[t] - a * s) / tau;
    }
    const double dist0 = sqdist(yn, x0);
    if (dist0 < chi * A_next * L * sqdist(yn, xt)) {
      out.status = FistaStatus::kFailure;
      out.y = yn;
      out.v = Mat(x0.rows, x0.cols);
      out.L = L;
      out.psi_y = psi_n;
      out.iters = it + 1;
      out.x_tilde = xt;
      out.A = A_next;
      dbg_fista(prm.L0, 1, it + 1, L, psi_n, -1);
      return out;
    }
    const Mat gy = psi.gradient(yn);
    Mat v(x.rows, x.cols);
    for (i64 t = 0; t < x.size(); ++t)
      v.a[t] = gy.a[t] - gt.a[t] + L * (xt.a[t] - yn.a[t]);
    if (norm(v) <= sigma * std::sqrt(dist0)) {
      out.status = FistaStatus::kSuccess;
      out.y = yn;
      out.v = std::move(v);
      out.L = L;
      out.psi_y = psi_n;
      out.iters = it + 1;
      out.x_tilde = xt;
      out.A = A_next;
      dbg_fista(prm.L0, 0, it + 1, L, psi_n, -1);
      return out;
    }
    A = A_next;
    y = std::move(yn);
  }
}

// ----------------------------------------------------------- ADAP-AIPP ---
void AippParams::validate() const {
  need(lambda0 > 0, "aipp: lambda0 must be positive");
  need(rho > 0, "aipp: rho must be positive");
  fista.validate();
  need(max_outer >= 1, "aipp: max_outer must be >= 1");
}

// adap_aipp.cpp:20-36 — psi(u) = lambda g(u) + 0.5 ||u - W||^2
static Smooth prox_objective(const Smooth* g, double lambda, const Mat* W) {
  Smooth psi;
  psi.value = [g, lambda, W](const Mat& u) {
    return lambda * g->value(u) + 0.5 * sqdist(u, *W);
  };
  psi.gradient = [g, lambda, W](const Mat& u) {
    Mat gg = g->gradient(u);
    for (i64 t = 0; t < u.size(); ++t) gg.a[t] = lambda * gg.a[t] + (u.a[t] - W->a[t]);
    return gg;
  };
  psi.value_and_gradient = [g, lambda, W](const Mat& u) {
    auto [gv, gg] = g->eval(u);
    const Mat d = sub(u, *W);
    const double val = lambda * gv + 0.5 * sqnorm(d);
    for (i64 t = 0; t < u.size(); ++t) gg.a[t] = lambda * gg.a[t] + d.a[t];
    return std::pair<double, Mat>(val, std::move(gg));
  };
  return psi;
}

// adap_aipp.cpp:40-116
AippResult aipp(const Smooth& g, const Mat& W_init, const AippParams& prm) {
  prm.validate();
  need(norm(W_init) <= 1.0 + 1e-12, "aipp: W_init outside the unit ball");
  double lambda = prm.lambda0, M_bar = 1.0;
  Mat Wp = W_init;
  double g_prev = g.value(Wp);
  AippResult out;
  out.W = Wp;
  out.R = Mat(W_init.rows, W_init.cols);
  out.R_norm = std::numeric_limits<double>::infinity();
  out.g_value = g_prev;
  out.lambda = lambda;
  for (int j = 1; j <= prm.max_outer; ++j) {
    Mat W, V;
    double L_out = 0.0, g_W = 0.0;
    for (;;) {
      if (lambda < prm.lambda_underflow * prm.lambda0) {
        out.status = AippStatus::kLambdaUnderflow;
        return out;
      }
      const Smooth psi = prox_objective(&g, lambda, &Wp);
      FistaParams fp = prm.fista;
      fp.L0 = std::max(1.0, M_bar / 2.0);
      FistaResult res = fista(psi, Wp, fp);
      out.fista_iters += res.iters;
      if (res.status == FistaStatus::kSuccess) {
        const double step_sq = sqdist(res.y, Wp);
        g_W = (res.psi_y - 0.5 * step_sq) / lambda;
        const double descent = lambda * g_prev - (lambda * g_W + 0.5 * step_sq);
        const double vw = esum_fn(Wp.size(), [&](i64 t) {
          return res.v.a[t] * (Wp.a[t] - res.y.a[t]);
        });
        if (descent >= vw) {
          W = std::move(res.y);
          V = std::move(res.v);
          L_out = res.L;
          break;
        }
      }
      lambda /= 2.0;
    }
    M_bar = L_out;
    Mat R(W.rows, W.cols);
    for (i64 t = 0; t < W.size(); ++t) R.a[t] = (V.a[t] + Wp.a[t] - W.a[t]) / lambda;
    const double R_norm = norm(R);
    ++out.prox_iters;
    if (R_norm <= prm.rho) {
      out.status = AippStatus::kConverged;
      out.W = std::move(W);
      out.R = std::move(R);
      out.R_norm = R_norm;
      out.g_value = g_W;
      out.lambda = lambda;
      return out;
    }
    if (R_norm < out.R_norm) {
      out.W = W;
      out.R = R;
      out.R_norm = R_norm;
      out.g_value = g_W;
      out.lambda = lambda;
    }
    Wp = std::move(W);
    g_prev = g_W;
  }
  out.status = AippStatus::kIterLimit;
  return out;
}

// ------------------------------------------------------------- Lanczos ---
void EigSettings::validate() const {
  need(tol > 0, "eig: tol must be positive");
  need(block_restart >= 2, "eig: block_restart must be >= 2");
  need(max_iters >= block_restart, "eig: max_iters < block_restart");
}

namespace {
// lanczos.cpp:22-28 — CGS2 against the first k columns of V (ordered GEMV).
void cgs2(const Mat& V, i64 k, Vec& w, Vec& h) {
  const i64 n = V.rows;
  auto tdot = [&](Vec& out) {
    out.assign(static_cast<size_t>(k), 0.0);
    for (i64 c = 0; c < k; ++c) {
      const double* v = V.col(c);
      double s = 0.0;
      for (i64 i = 0; i < n; ++i) s = s + v[i] * w[i];
      out[c] = s;
    }
  };
  auto minus_Vh = [&](const Vec& hh) {
    for (i64 i = 0; i < n; ++i) {
      double s = 0.0;
      for (i64 c = 0; c < k; ++c) s = s + V(i, c) * hh[c];
      w[i] = w[i] - s;
    }
  };
  tdot(h);
  minus_Vh(h);
  Vec h2;
  tdot(h2);
  minus_Vh(h2);
  for (i64 c = 0; c < k; ++c) h[c] = h[c] + h2[c];
}
}  // namespace

// lanczos.cpp:32-141 (Jacobi replaces SelfAdjointEigenSolver, see orc.hpp)
EigResult min_eigenpair(const LinOp& op, i64 n, const EigSettings& cfg) {
  cfg.validate();
  need(n >= 1, "min_eigenpair: dimension must be >= 1");
  auto applyB = [&op](const Vec& v) {
    Vec o = op(v);
    for (auto& x : o) x = -x;
    return o;
  };
  const i64 kmax = std::min<i64>(cfg.block_restart, n);
  const i64 keep = std::max<i64>(1, kmax / 3);
  Mat V(n, kmax + 1);
  Mat H(kmax + 1, kmax + 1);
  Rng rng(cfg.seed ^ 0x9b97f4a7c15ULL);
  {
    Vec v0 = gaussian_vector(n, rng);
    const double nv = norm(v0);
    for (i64 i = 0; i < n; ++i) V(i, 0) = v0[i] / nv;
  }
  int matvecs = 0;
  i64 basis = 1, filled = 0;
  double beta = 0.0;
  Vec w, h;
  EigResult best;
  best.residual = std::numeric_limits<double>::infinity();

  auto measure = [&](Vec x) {
    EigResult o;
    const double nx = norm(x);
    for (auto& t : x) t = t / nx;
    const Vec Bx = applyB(x);
    ++matvecs;
    const double mu = dot(x, Bx);
    o.lambda = -mu;
    o.residual = std::sqrt(esum_fn(n, [&](i64 i) {
      const double d = Bx[i] - mu * x[i];
      return d * d;
    }));
    o.v = std::move(x);
    o.matvecs = matvecs;
    o.converged = o.residual <= cfg.tol * std::max(1.0, std::fabs(o.lambda));
    return o;
  };

  std::vector<double> Hs, ev, evec;
  for (;;) {
    bool breakdown = false;
    while (filled < basis && matvecs < cfg.max_iters) {
      const i64 j = filled;
      w = applyB(Vec(V.col(j), V.col(j) + n));
      ++matvecs;
      cgs2(V, basis, w, h);
      for (i64 t = 0; t < basis; ++t) {
        H(t, j) = h[t];
        H(j, t) = h[t];
      }
      ++filled;
      beta = norm(w);
      double hmax = 0.0;
      for (double x : h) hmax = std::max(hmax, std::fabs(x));
      if (beta <= 1e-13 * std::max(1.0, hmax)) {
        breakdown = true;
        break;
      }
      if (basis < kmax) {
        for (i64 i = 0; i < n; ++i) V(i, basis) = w[i] / beta;
        H(basis, j) = beta;
        H(j, basis) = beta;
        ++basis;
      }
    }
    const int f = int(filled);
    Hs.assign(static_cast<size_t>(f) * f, 0.0);
    for (int c = 0; c < f; ++c)
      for (int r = 0; r < f; ++r) Hs[r + size_t(c) * f] = H(r, c);
    ev.assign(static_cast<size_t>(f), 0.0);
    evec.assign(static_cast<size_t>(f) * f, 0.0);
    jacobi_eigh(f, Hs.data(), ev.data(), evec.data());
    const int top = f - 1;
    const double mu = ev[top];
    const double res_est = breakdown ? 0.0 : beta * std::fabs(evec[(f - 1) + size_t(top) * f]);
    const bool budget_left = matvecs + 1 < cfg.max_iters;
    auto ritz = [&](int col) {
      Vec x(static_cast<size_t>(n));
      for (i64 i = 0; i < n; ++i) {
        double s = 0.0;
        for (int c = 0; c < f; ++c) s = s + V(i, c) * evec[c + size_t(col) * f];
        x[i] = s;
      }
      return x;
    };
    if (res_est <= cfg.tol * std::max(1.0, std::fabs(mu)) || !budget_left ||
        (breakdown && filled >= n)) {
      EigResult o = measure(ritz(top));
      if (o.residual < best.residual) best = o;
      if (best.converged || matvecs >= cfg.max_iters || (breakdown && filled >= n))
        return best;
    }
    const i64 l = std::min<i64>(keep, filled - 1 > 0 ? filled - 1 : 1);
    std::vector<Vec> kept;
    for (i64 t = 0; t < l; ++t) kept.push_back(ritz(int(filled - 1 - t)));
    std::fill(H.a.begin(), H.a.end(), 0.0);
    for (i64 t = 0; t < l; ++t) H(t, t) = ev[size_t(filled - 1 - t)];
    for (i64 t = 0; t < l; ++t)
      for (i64 i = 0; i < n; ++i) V(i, t) = kept[t][i];
    if (breakdown) {
      Vec fr = gaussian_vector(n, rng), dummy;
      cgs2(V, l, fr, dummy);
      const double fn = norm(fr);
      if (fn <= 1e-13) return best;
      for (i64 i = 0; i < n; ++i) V(i, l) = fr[i] / fn;
    } else {
      for (i64 i = 0; i < n; ++i) V(i, l) = w[i] / beta;
    }
    basis = l + 1;
    filled = l;
  }
}

// ------------------------------------------------------------------ HLR ---
// hlr.cpp:8-10
double fw_gap(const GradOp& G, const Mat& Y, double theta) {
  return frob_dot(G.apply(Y), Y) + theta;
}
// hlr.cpp:12-29
Escape escape_direction(const GradOp& G, i64 n, const EigSettings& cfg) {
  EigResult e = min_eigenpair([&G](const Vec& v) { return G.apply_vec(v); }, n, cfg);
  Escape o;
  o.lambda_min = e.lambda;
  o.eig_residual = e.residual;
  o.eig_products = e.matvecs;
  o.eig_trusted = e.converged;
  if (e.lambda < 0) {
    o.theta = -e.lambda;
    o.y = std::move(e.v);
  } else {
    o.theta = 0.0;
    o.y.assign(static_cast<size_t>(n), 0.0);
  }
  return o;
}
// hlr.cpp:31-44
double fw_stepsize(const Instance& I, const Mat& Y, const Vec& y, double theta,
                   const Vec& p, double beta) {
  need(i64(y.size()) == I.n, "fw_stepsize: y has the wrong length");
  const GradOp G(I, Y, p, beta);
  const double numer = fw_gap(G, Y, theta);
  Mat ym(I.n, 1);
  ym.a = y;
  const Vec map_y = I.apply_map(ym);
  const double denom = beta * esum_fn(I.m, [&](i64 k) {
                         const double d = (G.residual[k] + I.b[k]) - map_y[k];
                         return d * d;
                       });
  if (denom <= 1e-14) return numer > 0 ? 1.0 : 0.0;
  return std::clamp(numer / denom, 0.0, 1.0);
}
// hlr.cpp:46-53
Mat rank_update(const Mat& Y, const Vec& y, double alpha) {
  need(alpha >= 0.0 && alpha <= 1.0, "rank_update: alpha outside [0,1]");
  if (alpha == 1.0) {
    Mat o(Y.rows, 1);
    o.a = y;
    return o;
  }
  Mat o(Y.rows, Y.cols + 1);
  const double sa = std::sqrt(1.0 - alpha), sb = std::sqrt(alpha);
  for (i64 t = 0; t < Y.size(); ++t) o.a[t] = sa * Y.a[t];
  for (i64 i = 0; i < Y.rows; ++i) o(i, Y.cols) = sb * y[i];
  return o;
}

// hlr.cpp:55-151
HlrOutcome hlr_solve(const Instance& I, Mat U_init, const Vec& p, double beta,
                     double eps_t, const HlrSettings& hs, const Sink& sink) {
  need(eps_t > 0, "hlr_solve: eps_t must be positive");
  I.check_dims(U_init, "hlr_solve");
  need(norm(U_init) <= 1.0 + 1e-12, "hlr_solve: start factor outside unit ball");
  AlFn al{&I, p, beta};
  Smooth g;
  g.value = [&al](const Mat& u) { return al.value(u); };
  g.gradient = [&al](const Mat& u) { return al.gradient(u); };
  g.value_and_gradient = [&al](const Mat& u) { return al.value_and_gradient(u); };
  AippParams ap = hs.aipp;
  ap.rho = eps_t;
  EigSettings eig = hs.eig;
  eig.tol = 0.1 * eps_t;
  HlrOutcome out;
  Mat Yt = std::move(U_init);
  for (int step = 0;; ++step) {
    AippResult st = aipp(g, Yt, ap);
    ++out.stats.aipp_calls;
    out.stats.aipp_iters += st.prox_iters;
    out.stats.fista_iters += st.fista_iters;
    Mat Y = std::move(st.W);
    const GradOp G(I, Y, p, beta);
    const Escape esc = escape_direction(G, I.n, eig);
    out.stats.eig_products += esc.eig_products;
    const double gap = fw_gap(G, Y, esc.theta);
    if (sink) {
      TraceEvent ev;
      ev.kind = 0;
      ev.outer_iter = hs.outer_iter;
      ev.beta = beta;
      ev.eps_inner = eps_t;
      ev.gap = gap;
      ev.theta = esc.theta;
      ev.rank = Y.cols;
      ev.al_value = st.g_value;
      sink(ev);
    }
    const bool done = gap <= eps_t;
    const bool no_steps = step >= hs.max_fw_steps;
    const bool no_time = hs.deadline && std::chrono::steady_clock::now() >= *hs.deadline;
    if (done || no_steps || no_time || !esc.eig_trusted) {
      out.U = std::move(Y);
      out.theta = esc.theta;
      out.gap = gap;
      out.lambda_min = esc.lambda_min;
      out.al_val = st.g_value;
      out.residual = G.residual;
      out.cdot = st.g_value - dot(p, out.residual) - 0.5 * beta * sqnorm(out.residual);
      out.eig_trusted = esc.eig_trusted;
      out.status = done ? HlrStatus::kConverged
                        : no_time ? HlrStatus::kTimeLimit : HlrStatus::kStepLimit;
      if (!esc.eig_trusted && !done) out.status = HlrStatus::kStepLimit;
      return out;
    }
    const double alpha = fw_stepsize(I, Y, esc.y, esc.theta, p, beta);
    if (esc.theta > 0) {
      Yt = rank_update(Y, esc.y, alpha);
    } else if (alpha == 1.0) {
      Yt = Mat(I.n, 1);
    } else {
      Yt = Y;
      const double sa = std::sqrt(1.0 - alpha);
      for (auto& x : Yt.a) x = sa * x;
    }
    ++out.stats.fw_steps;
    if (sink) {
      TraceEvent ev;
      ev.kind = 1;
      ev.outer_iter = hs.outer_iter;
      ev.beta = beta;
      ev.eps_inner = eps_t;
      ev.gap = gap;
      ev.theta = esc.theta;
      ev.rank = Yt.cols;
      ev.fw_alpha = alpha;
      ev.al_value = al.value(Yt);
      sink(ev);
    }
  }
}

// --------------------------------------------------------------- solver ---
void SolverConfig::validate() const {
  need(eps > 0, "config: eps must be positive");
  need(beta_growth >= 1.0, "config: beta_growth must be >= 1");
  need(eps_decay > 0 && eps_decay <= 1.0, "config: eps_decay in (0,1]");
  need(max_outer >= 1, "config: max_outer must be >= 1");
  need(time_limit > 0, "config: time_limit must be positive");
  need(max_fw_steps >= 1, "config: max_fw_steps must be >= 1");
}

// solver.cpp:31-42
Instance scale_instance(const Instance& I, double* tau_orig) {
  I.validate();
  Instance o = I;
  *tau_orig = I.tau;
  if (I.tau != 1.0) {
    for (auto& x : o.b) x = x / I.tau;
    o.norm_b1 = I.norm_b1 / I.tau;
    o.tau = 1.0;
  }
  return o;
}

// solver.cpp:51-76
Termination check_termination(const Instance& I, const Mat& U, const Vec& p,
                              double theta, const EigSettings& eig, double eps) {
  I.check_dims(U, "check_termination");
  Termination t;
  const Vec r = residual_of(I, U);
  t.rel_pfeas = norm(r) / (1.0 + I.norm_b1);
  t.pval = frob_dot(I.apply_C(U), U);
  t.dval = -dot(I.b, p) - theta;
  t.rel_gap = std::fabs(t.pval - t.dval) / (1.0 + std::fabs(t.pval) + std::fabs(t.dval));
  EigResult de = min_eigenpair(
      [&I, &p](const Vec& v) {
        Mat V(i64(v.size()), 1);
        V.a = v;
        return I.C_plus_adjoint(p, V).a;
      },
      I.n, eig);
  t.dual_lambda_min = de.lambda;
  t.eig_products = de.matvecs;
  t.eig_trusted = de.converged;
  t.rel_dfeas = std::max(0.0, -t.dual_lambda_min) / (1.0 + I.norm_C1);
  t.done = t.eig_trusted && t.rel_pfeas <= eps && t.rel_gap <= eps && t.rel_dfeas <= eps;
  return t;
}

namespace {
struct Certified {
  Termination terms;
  Vec p;
  double theta = 0.0;
};
// solver.cpp:92-122
Certified certify(const Instance& I, const Mat& U, const Vec& p, double theta,
                  const EigSettings& eig, double eps) {
  Certified ct;
  ct.p = p;
  ct.theta = theta;
  if (I.identity_constraint && theta > 0) {
    ct.p[*I.identity_constraint] += theta;
    ct.theta = 0.0;
  }
  ct.terms = check_termination(I, U, ct.p, ct.theta, eig, eps);
  if (!ct.terms.eig_trusted) return ct;
  Termination& t = ct.terms;
  if (I.identity_constraint) {
    if (t.dual_lambda_min < 0) {
      ct.p[*I.identity_constraint] -= t.dual_lambda_min;
      t.dval += t.dual_lambda_min * I.b[*I.identity_constraint];
      t.dual_lambda_min = 0.0;
      t.rel_dfeas = 0.0;
    }
  } else {
    const double tight = std::max(0.0, -t.dual_lambda_min);
    t.dval += ct.theta - tight;
    ct.theta = tight;
  }
  t.rel_gap = std::fabs(t.pval - t.dval) / (1.0 + std::fabs(t.pval) + std::fabs(t.dval));
  t.done = t.rel_pfeas <= eps && t.rel_gap <= eps && t.rel_dfeas <= eps;
  return ct;
}
}  // namespace

// solver.cpp:126-134
SolveReport solve(const Instance& I, const SolverConfig& cfg, const Sink& sink) {
  cfg.validate();
  I.validate();
  Rng rng(cfg.seed);
  Vec u0 = gaussian_vector(I.n, rng);
  const double nu = norm(u0);
  Mat U0(I.n, 1);
  for (i64 i = 0; i < I.n; ++i) U0(i, 0) = u0[i] / nu;
  return solve_warm(I, cfg, U0, Vec(static_cast<size_t>(I.m), 0.0), sink);
}

// solver.cpp:136-279
SolveReport solve_warm(const Instance& I, const SolverConfig& cfg, const Mat& U0,
                       const Vec& p0, const Sink& sink) {
  using clock = std::chrono::steady_clock;
  const auto t0 = clock::now();
  const auto deadline =
      t0 + std::chrono::duration_cast<clock::duration>(std::chrono::duration<double>(cfg.time_limit));
  cfg.validate();
  I.validate();
  double tau = 1.0;
  const Instance si = scale_instance(I, &tau);
  const double nb1 = si.norm_b1, nb2 = norm(si.b);
  const double eps_floor = cfg.eps_floor > 0 ? cfg.eps_floor : cfg.eps * (1.0 + nb1) / 10.0;
  double eps_t = cfg.eps0 > 0 ? cfg.eps0 : 1e-2 * (1.0 + nb1);
  eps_t = std::max(eps_t, eps_floor);
  double beta = cfg.beta0 > 0 ? cfg.beta0 : 10.0 * std::max(1.0, nb2 > 0 ? 1.0 / nb2 : 1.0);

  SolveReport rep;
  rep.tau = tau;
  rep.U = U0;
  need(norm(rep.U) <= 1.0 + 1e-12, "solve: warm-start factor outside unit ball");
  rep.p = p0;
  need(i64(rep.p.size()) == si.m, "solve: warm-start multiplier length");
  EigSettings eig_term = cfg.eig;
  eig_term.tol = std::min(cfg.eig.tol, 1e-7);
  eig_term.seed = cfg.seed;
  std::optional<Certified> final_ct;
  double prev_pfeas = std::numeric_limits<double>::infinity();

  auto finish = [&](SolveStatus status) {
    rep.status = status;
    if (!final_ct) {
      if (!all_finite(rep.U) || !all_finite(rep.p)) {
        const double nan = std::numeric_limits<double>::quiet_NaN();
        rep.rel_pfeas = rep.rel_gap = rep.rel_dfeas = nan;
        rep.pval = rep.dval = rep.dval_no_theta = nan;
        rep.rank = rep.U.cols;
        rep.wall_seconds = std::chrono::duration<double>(clock::now() - t0).count();
        return rep;
      }
      final_ct = certify(si, rep.U, rep.p, rep.theta, eig_term, cfg.eps);
      rep.eig_products += final_ct->terms.eig_products;
    }
    rep.p = final_ct->p;
    rep.theta = final_ct->theta;
    rep.rel_pfeas = final_ct->terms.rel_pfeas;
    rep.rel_gap = final_ct->terms.rel_gap;
    rep.rel_dfeas = final_ct->terms.rel_dfeas;
    rep.pval = tau * final_ct->terms.pval;
    rep.dval = tau * final_ct->terms.dval;
    rep.dval_no_theta = tau * -dot(si.b, rep.p);
    rep.rank = rep.U.cols;
    rep.wall_seconds = std::chrono::duration<double>(clock::now() - t0).count();
    return rep;
  };

  try {
    for (int t = 1; t <= cfg.max_outer; ++t) {
      if (clock::now() >= deadline) return finish(SolveStatus::kTimeLimit);
      HlrSettings hs;
      hs.eig = cfg.eig;
      hs.eig.seed = cfg.seed;
      hs.aipp = cfg.aipp;
      hs.max_fw_steps = cfg.max_fw_steps;
      hs.outer_iter = t;
      hs.deadline = deadline;
      HlrOutcome out = hlr_solve(si, rep.U, rep.p, beta, eps_t, hs, sink);
      rep.outer_iters = t;
      rep.fw_steps += out.stats.fw_steps;
      rep.aipp_iters += out.stats.aipp_iters;
      rep.fista_iters += out.stats.fista_iters;
      rep.eig_products += out.stats.eig_products;
      rep.U = std::move(out.U);
      for (i64 k = 0; k < si.m; ++k) rep.p[k] = rep.p[k] + beta * out.residual[k];
      rep.theta = out.theta;
      if (!all_finite(rep.U) || !all_finite(rep.p)) {
        rep.message = "non-finite iterate";
        return finish(SolveStatus::kNumericalFailure);
      }
      const double rel_pfeas = norm(out.residual) / (1.0 + nb1);
      const double pval = out.cdot;
      const double dval = -dot(si.b, rep.p) - out.theta;
      const double rel_gap = std::fabs(pval - dval) / (1.0 + std::fabs(pval) + std::fabs(dval));
      const double lam = si.identity_constraint ? out.lambda_min + out.theta : out.lambda_min;
      const double rel_dfeas_est = std::max(0.0, -lam) / (1.0 + si.norm_C1);
      if (sink) {
        TraceEvent ev;
        ev.kind = 2;
        ev.outer_iter = t;
        ev.beta = beta;
        ev.eps_inner = eps_t;
        ev.gap = out.gap;
        ev.theta = out.theta;
        ev.rank = rep.U.cols;
        ev.al_value = out.al_val;
        ev.rel_pfeas = rel_pfeas;
        ev.rel_gap = rel_gap;
        ev.rel_dfeas = rel_dfeas_est;
        sink(ev);
      }
      if (out.eig_trusted && rel_pfeas <= cfg.eps && rel_gap <= cfg.eps &&
          rel_dfeas_est <= cfg.eps) {
        Certified ct = certify(si, rep.U, rep.p, rep.theta, eig_term, cfg.eps);
        rep.eig_products += ct.terms.eig_products;
        if (ct.terms.done) {
          final_ct = std::move(ct);
          return finish(SolveStatus::kOptimal);
        }
      }
      if (rel_pfeas > 0.9 * prev_pfeas) beta *= cfg.beta_growth;
      prev_pfeas = rel_pfeas;
      eps_t = std::max(eps_floor, eps_t * cfg.eps_decay);
    }
  } catch (const NumericalError& e) {
    rep.message = e.what();
    return finish(SolveStatus::kNumericalFailure);
  }
  return finish(SolveStatus::kIterationLimit);
}

}  // namespace orc
