// extern "C" surface of the oracle for the Python test harness (ctypes).
// TEST INFRASTRUCTURE ONLY (see orc.hpp).  Column-major factors, host memory.
#include <cstring>
#include <memory>

#include "orc.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;

struct Handle {
  Instance inst;
  int family = 0;  // 0 theta/graph, 1 matcomp, 2 phaseret, 3 dense
  std::vector<i64> oi, oj, gi, gj;
  double nuclear = 0.0;
  std::vector<cplx> hidden_x, masks;
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const InputError& e) {
    g_err = e.what();
    return 64;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 66;
  }
}

Mat to_mat(const double* U, i64 n, i64 s) {
  Mat M(n, s);
  std::memcpy(M.a.data(), U, sizeof(double) * size_t(n * s));
  return M;
}
Handle* theta_handle(const Graph& g) {
  auto* h = new Handle;
  h->inst = theta_instance(g);
  h->family = 0;
  for (auto [u, v] : g.edges) {
    h->gi.push_back(u);
    h->gj.push_back(v);
  }
  return h;
}
}  // namespace

extern "C" {

typedef struct {
  double eps, beta0, beta_growth, eps0, eps_decay, eps_floor;
  int max_outer;
  double time_limit;
  unsigned long long seed;
  double eig_tol;
  int eig_max_iters, eig_block_restart;
  double aipp_lambda0, aipp_rho;
  int aipp_max_outer;
  double aipp_lambda_underflow;
  double fista_sigma, fista_chi, fista_mu, fista_L0;
  int fista_max_iters, max_fw_steps, threads;
} orc_config;

typedef struct {
  int status;
  double pval, dval, dval_no_theta, rel_pfeas, rel_gap, rel_dfeas;
  long long rank;
  int outer_iters, fw_steps;
  long long aipp_iters, fista_iters, eig_products;
  double wall_seconds, tau, theta;
  char message[256];
} orc_report;

typedef struct {
  int kind, outer_iter;
  double beta, eps_inner, gap, theta;
  long long rank;
  double al_value, fw_alpha, rel_pfeas, rel_gap, rel_dfeas;
} orc_trace;

typedef void (*orc_trace_fn)(const orc_trace*, void*);

const char* orc_last_error() { return g_err.c_str(); }
void orc_set_threads(int n) { set_max_threads(n); }

int orc_theta_hypercube(int d, void** out) {
  return guard([&] { *out = theta_handle(make_hypercube(d)); });
}
int orc_theta_cycle(int n, void** out) {
  return guard([&] { *out = theta_handle(make_cycle(n)); });
}
int orc_theta_petersen(void** out) {
  return guard([&] { *out = theta_handle(make_petersen()); });
}
int orc_theta_edges(long long n, long long ne, const long long* ei, const long long* ej,
                    void** out) {
  return guard([&] {
    std::vector<std::pair<i64, i64>> raw;
    for (i64 k = 0; k < ne; ++k) raw.emplace_back(ei[k], ej[k]);
    *out = theta_handle(graph_from_pairs(n, raw));
  });
}
int orc_theta_file(const char* path, int format, void** out) {
  return guard([&] { *out = theta_handle(load_graph(path, format)); });
}
int orc_matcomp(long long n1, long long n2, int r, unsigned long long seed, int offset,
                double tau_safety, void** out) {
  return guard([&] {
    McData d = matrix_completion(n1, n2, r, seed, offset != 0, tau_safety);
    auto* h = new Handle;
    h->inst = std::move(d.inst);
    h->family = 1;
    h->oi = std::move(d.omega_i);
    h->oj = std::move(d.omega_j);
    h->nuclear = d.nuclear_norm;
    *out = h;
  });
}
int orc_matcomp_paper(long long n1, long long n2, int r, unsigned long long seed,
                      long long draws, double tau_safety, void** out) {
  return guard([&] {
    McData d = matrix_completion(n1, n2, r, seed, false, tau_safety, draws);
    auto* h = new Handle;
    h->inst = std::move(d.inst);
    h->family = 1;
    h->oi = std::move(d.omega_i);
    h->oj = std::move(d.omega_j);
    h->nuclear = d.nuclear_norm;
    *out = h;
  });
}
long long orc_matcomp_count(long long n1, long long n2, int r, int offset) {
  return mc_count(n1, n2, r, offset != 0);
}
int orc_phaseret(long long n, int L, unsigned long long seed, double tau_slack, void** out) {
  return guard([&] {
    PrData d = phase_retrieval(n, L, seed, tau_slack);
    auto* h = new Handle;
    h->inst = std::move(d.inst);
    h->family = 2;
    h->hidden_x = std::move(d.hidden_x);
    h->masks = std::move(d.masks);
    *out = h;
  });
}
// Gaussian phase retrieval from given measurement vectors (m x n row-major
// re / im) and signal (n re / im)
int orc_gauss_pr(long long n, long long m, const double* A_re, const double* A_im, const double* x_re,
                 const double* x_im, double tau_slack, void** out) {
  return guard([&] {
    std::vector<cplx> x(static_cast<size_t>(n));
    for (long long j = 0; j < n; ++j) x[j] = cplx(x_re[j], x_im[j]);
    auto* h = new Handle;
    h->inst = gauss_pr_instance(n, m, A_re, A_im, x, tau_slack);
    h->family = 4;
    *out = h;
  });
}
// C: n x n col-major; A: m blocks of n x n col-major; b: m
int orc_dense(long long n, long long m, const double* C, const double* A, const double* b,
              double tau, void** out) {
  return guard([&] {
    DenseSdp d;
    d.C = to_mat(C, n, n);
    for (i64 k = 0; k < m; ++k) d.A.push_back(to_mat(A + k * n * n, n, n));
    d.b.assign(b, b + m);
    d.tau = tau;
    auto* h = new Handle;
    h->inst = dense_instance(d);
    h->family = 3;
    *out = h;
  });
}
void orc_free(void* h) { delete static_cast<Handle*>(h); }

// info: n, m, identity(-1 none), field ; doubles: tau, norm_b1, norm_C1, nuclear
void orc_info(void* hp, long long* ints, double* dbls) {
  auto* h = static_cast<Handle*>(hp);
  ints[0] = h->inst.n;
  ints[1] = h->inst.m;
  ints[2] = h->inst.identity_constraint ? *h->inst.identity_constraint : -1;
  ints[3] = int(h->inst.field);
  ints[4] = h->family;
  dbls[0] = h->inst.tau;
  dbls[1] = h->inst.norm_b1;
  dbls[2] = h->inst.norm_C1;
  dbls[3] = h->nuclear;
}
void orc_get_b(void* hp, double* b) {
  auto* h = static_cast<Handle*>(hp);
  std::memcpy(b, h->inst.b.data(), sizeof(double) * h->inst.b.size());
}
// pair index sets (theta: edges; matcomp: omega with j in [0,n2))
long long orc_get_pairs(void* hp, long long* i, long long* j) {
  auto* h = static_cast<Handle*>(hp);
  const auto& I = h->family == 1 ? h->oi : h->gi;
  const auto& J = h->family == 1 ? h->oj : h->gj;
  if (i)
    for (size_t k = 0; k < I.size(); ++k) {
      i[k] = I[k];
      j[k] = J[k];
    }
  return (long long)I.size();
}
// phase retrieval: hidden_x (2*nc: re,im interleaved), masks (2*nc*L)
void orc_get_pr(void* hp, double* x, double* masks) {
  auto* h = static_cast<Handle*>(hp);
  if (x) std::memcpy(x, h->hidden_x.data(), sizeof(cplx) * h->hidden_x.size());
  if (masks) std::memcpy(masks, h->masks.data(), sizeof(cplx) * h->masks.size());
}

int orc_apply_map(void* hp, const double* U, long long s, double* out) {
  auto* h = static_cast<Handle*>(hp);
  return guard([&] {
    const Vec r = h->inst.apply_map(to_mat(U, h->inst.n, s));
    std::memcpy(out, r.data(), sizeof(double) * r.size());
  });
}
int orc_apply_C(void* hp, const double* U, long long s, double* out) {
  auto* h = static_cast<Handle*>(hp);
  return guard([&] {
    const Mat r = h->inst.apply_C(to_mat(U, h->inst.n, s));
    std::memcpy(out, r.a.data(), sizeof(double) * r.a.size());
  });
}
int orc_apply_adjoint(void* hp, const double* p, const double* U, long long s, double* out) {
  auto* h = static_cast<Handle*>(hp);
  return guard([&] {
    const Vec pv(p, p + h->inst.m);
    const Mat r = h->inst.apply_adjoint(pv, to_mat(U, h->inst.n, s));
    std::memcpy(out, r.a.data(), sizeof(double) * r.a.size());
  });
}
int orc_apply_C_plus_adjoint(void* hp, const double* q, const double* U, long long s,
                             double* out) {
  auto* h = static_cast<Handle*>(hp);
  return guard([&] {
    const Vec qv(q, q + h->inst.m);
    const Mat r = h->inst.C_plus_adjoint(qv, to_mat(U, h->inst.n, s));
    std::memcpy(out, r.a.data(), sizeof(double) * r.a.size());
  });
}
int orc_al_value(void* hp, const double* U, long long s, const double* p, double beta,
                 double* val) {
  auto* h = static_cast<Handle*>(hp);
  return guard([&] {
    *val = al_value(h->inst, to_mat(U, h->inst.n, s), Vec(p, p + h->inst.m), beta);
  });
}
int orc_al_gradient(void* hp, const double* U, long long s, const double* p, double beta,
                    double* grad) {
  auto* h = static_cast<Handle*>(hp);
  return guard([&] {
    const Mat g = al_gradient(h->inst, to_mat(U, h->inst.n, s), Vec(p, p + h->inst.m), beta);
    std::memcpy(grad, g.a.data(), sizeof(double) * g.a.size());
  });
}
int orc_al_value_and_gradient(void* hp, const double* U, long long s, const double* p,
                              double beta, double* val, double* grad) {
  auto* h = static_cast<Handle*>(hp);
  return guard([&] {
    AlFn f{&h->inst, Vec(p, p + h->inst.m), beta};
    auto [v, g] = f.value_and_gradient(to_mat(U, h->inst.n, s));
    *val = v;
    std::memcpy(grad, g.a.data(), sizeof(double) * g.a.size());
  });
}
// Lanczos min eigenpair of G = C + A*(p + beta (A(UU')-b)) (hlr escape step)
int orc_min_eig_G(void* hp, const double* U, long long s, const double* p, double beta,
                  double tol, int max_iters, int block_restart, unsigned long long seed,
                  double* lambda, double* v, double* residual, int* matvecs, int* converged) {
  auto* h = static_cast<Handle*>(hp);
  return guard([&] {
    const GradOp G(h->inst, to_mat(U, h->inst.n, s), Vec(p, p + h->inst.m), beta);
    EigSettings e;
    e.tol = tol;
    e.max_iters = max_iters;
    e.block_restart = block_restart;
    e.seed = seed;
    const EigResult r = min_eigenpair([&G](const Vec& x) { return G.apply_vec(x); },
                                      h->inst.n, e);
    *lambda = r.lambda;
    if (v) std::memcpy(v, r.v.data(), sizeof(double) * r.v.size());
    *residual = r.residual;
    *matvecs = r.matvecs;
    *converged = r.converged;
  });
}
// Dense Lanczos on an explicit symmetric matrix (test_lanczos.cpp analogue).
int orc_min_eig_dense(long long n, const double* A, double tol, int max_iters,
                      int block_restart, unsigned long long seed, double* lambda, double* v,
                      double* residual, int* matvecs, int* converged) {
  return guard([&] {
    const Mat M = to_mat(A, n, n);
    EigSettings e;
    e.tol = tol;
    e.max_iters = max_iters;
    e.block_restart = block_restart;
    e.seed = seed;
    const EigResult r = min_eigenpair(
        [&M, n](const Vec& x) {
          Vec o(static_cast<size_t>(n), 0.0);
          for (i64 c = 0; c < n; ++c)
            for (i64 i = 0; i < n; ++i) o[i] += M(i, c) * x[c];
          return o;
        },
        n, e);
    *lambda = r.lambda;
    if (v) std::memcpy(v, r.v.data(), sizeof(double) * r.v.size());
    *residual = r.residual;
    *matvecs = r.matvecs;
    *converged = r.converged;
  });
}
void orc_jacobi_eigh(int k, const double* H, double* ev, double* evec) {
  jacobi_eigh(k, H, ev, evec);
}

static SolverConfig to_cfg(const orc_config* c) {
  SolverConfig s;
  s.eps = c->eps;
  s.beta0 = c->beta0;
  s.beta_growth = c->beta_growth;
  s.eps0 = c->eps0;
  s.eps_decay = c->eps_decay;
  s.eps_floor = c->eps_floor;
  s.max_outer = c->max_outer;
  s.time_limit = c->time_limit;
  s.seed = c->seed;
  s.eig.tol = c->eig_tol;
  s.eig.max_iters = c->eig_max_iters;
  s.eig.block_restart = c->eig_block_restart;
  s.aipp.lambda0 = c->aipp_lambda0;
  s.aipp.rho = c->aipp_rho;
  s.aipp.max_outer = c->aipp_max_outer;
  s.aipp.lambda_underflow = c->aipp_lambda_underflow;
  s.aipp.fista.sigma = c->fista_sigma;
  s.aipp.fista.chi = c->fista_chi;
  s.aipp.fista.mu = c->fista_mu;
  s.aipp.fista.L0 = c->fista_L0;
  s.aipp.fista.max_iters = c->fista_max_iters;
  s.max_fw_steps = c->max_fw_steps;
  return s;
}

// AIPP on g = L_beta(.; p) from W (rank s) — the HLR stationary-point step.
int orc_aipp_al(void* hp, const double* p, double beta, const double* W, long long s,
                double rho, const orc_config* cfg, double* W_out, int* status,
                int* prox_iters, int* fista_iters, double* R_norm, double* g_value,
                double* lambda) {
  auto* h = static_cast<Handle*>(hp);
  return guard([&] {
    AlFn al{&h->inst, Vec(p, p + h->inst.m), beta};
    Smooth g;
    g.value = [&al](const Mat& u) { return al.value(u); };
    g.gradient = [&al](const Mat& u) { return al.gradient(u); };
    g.value_and_gradient = [&al](const Mat& u) { return al.value_and_gradient(u); };
    AippParams ap = to_cfg(cfg).aipp;
    ap.rho = rho;
    const AippResult r = aipp(g, to_mat(W, h->inst.n, s), ap);
    std::memcpy(W_out, r.W.a.data(), sizeof(double) * r.W.a.size());
    *status = int(r.status);
    *prox_iters = r.prox_iters;
    *fista_iters = r.fista_iters;
    *R_norm = r.R_norm;
    *g_value = r.g_value;
    *lambda = r.lambda;
  });
}

int orc_solve(void* hp, const orc_config* cfg, const double* U0, long long s0,
              const double* p0, orc_report* rep, double* U_out, long long U_cap,
              double* p_out, orc_trace_fn fn, void* user) {
  auto* h = static_cast<Handle*>(hp);
  return guard([&] {
    const SolverConfig c = to_cfg(cfg);
    if (cfg->threads >= 0) set_max_threads(cfg->threads);
    Sink sink;
    if (fn)
      sink = [fn, user](const TraceEvent& e) {
        orc_trace t{e.kind, e.outer_iter, e.beta, e.eps_inner, e.gap, e.theta,
                    (long long)e.rank, e.al_value, e.fw_alpha, e.rel_pfeas, e.rel_gap,
                    e.rel_dfeas};
        fn(&t, user);
      };
    SolveReport r = U0 ? solve_warm(h->inst, c, to_mat(U0, h->inst.n, s0),
                                    p0 ? Vec(p0, p0 + h->inst.m) : Vec(static_cast<size_t>(h->inst.m), 0.0),
                                    sink)
                       : solve(h->inst, c, sink);
    rep->status = int(r.status);
    rep->pval = r.pval;
    rep->dval = r.dval;
    rep->dval_no_theta = r.dval_no_theta;
    rep->rel_pfeas = r.rel_pfeas;
    rep->rel_gap = r.rel_gap;
    rep->rel_dfeas = r.rel_dfeas;
    rep->rank = r.rank;
    rep->outer_iters = r.outer_iters;
    rep->fw_steps = r.fw_steps;
    rep->aipp_iters = r.aipp_iters;
    rep->fista_iters = r.fista_iters;
    rep->eig_products = r.eig_products;
    rep->wall_seconds = r.wall_seconds;
    rep->tau = r.tau;
    rep->theta = r.theta;
    std::snprintf(rep->message, sizeof(rep->message), "%s", r.message.c_str());
    if (U_out && r.U.size() <= U_cap)
      std::memcpy(U_out, r.U.a.data(), sizeof(double) * r.U.a.size());
    if (p_out) std::memcpy(p_out, r.p.data(), sizeof(double) * r.p.size());
  });
}

}  // extern "C"
