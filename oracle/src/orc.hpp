// HALLaR CPU oracle — TEST INFRASTRUCTURE ONLY.
//
// A plain-C++ (no Eigen) restatement of the reference lrsdp library
// (/root/reference/proj/src/*.cpp) used as the parity checker for the B200
// product path.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load it.  It is never linked into
// the product library (paper_2505_13719_b200/libcuhallar.so).
//
// Arithmetic model: the reference binary is built with
// -O3 and no -march, i.e. SSE2 with no FMA contraction.  We compile with
// -ffp-contract=off and restate Eigen's LinearVectorized redux order (two
// 2-wide packet accumulators) in esum(), so contiguous reductions follow the
// reference's order.  Deviations, all tolerance-level:
//   * GEMV inside Lanczos CGS2 is a plain ordered dot/axpy (Eigen's GEMV
//     blocking is version-dependent and unpinned);
//   * the <=31x31 symmetric eigen-solve is a cyclic (tournament-ordered)
//     Jacobi method instead of Eigen's SelfAdjointEigenSolver, eigenvector
//     signs normalised (largest-|.| component positive); the device solver
//     runs the identical Jacobi so Lanczos decisions track it;
//   * the MC nuclear norm uses Householder QR + one-sided Jacobi SVD on the
//     r x r core (Eigen: HouseholderQR + JacobiSVD).
#pragma once

#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>
#include <complex>
#include <optional>
#include <chrono>
#include <cmath>

namespace orc {

using i64 = std::int64_t;
using u64 = std::uint64_t;
using cplx = std::complex<double>;

struct InputError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
inline void need(bool ok, const std::string& why) {
  if (!ok) throw InputError(why);
}

// ---------------------------------------------------------------- dense ---
// Column-major dense matrix (Eigen::MatrixXd layout, types.hpp:9).
struct Mat {
  i64 rows = 0, cols = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(i64 r, i64 c, double fill = 0.0) : rows(r), cols(c), a(static_cast<size_t>(r * c), fill) {}
  double& operator()(i64 i, i64 j) { return a[size_t(i + j * rows)]; }
  double operator()(i64 i, i64 j) const { return a[size_t(i + j * rows)]; }
  double* col(i64 j) { return a.data() + j * rows; }
  const double* col(i64 j) const { return a.data() + j * rows; }
  i64 size() const { return rows * cols; }
};
using Vec = std::vector<double>;

// Eigen LinearVectorized redux order (SSE2 packets of 2, two accumulators,
// aligned start 0) for sum_i term(i), i in [0,n).
template <class F>
double esum_fn(i64 n, F term) {
  if (n <= 0) return 0.0;
  const i64 aligned = (n / 2) * 2;
  if (aligned == 0) {
    double r = term(0);
    for (i64 i = 1; i < n; ++i) r = r + term(i);
    return r;
  }
  double p0a = term(0), p0b = term(1);
  if (aligned > 2) {
    const i64 aligned2 = (n / 4) * 4;
    double p1a = term(2), p1b = term(3);
    for (i64 i = 4; i < aligned2; i += 4) {
      p0a = p0a + term(i);
      p0b = p0b + term(i + 1);
      p1a = p1a + term(i + 2);
      p1b = p1b + term(i + 3);
    }
    p0a = p0a + p1a;
    p0b = p0b + p1b;
    if (aligned > aligned2) {
      p0a = p0a + term(aligned2);
      p0b = p0b + term(aligned2 + 1);
    }
  }
  double r = p0a + p0b;
  for (i64 i = aligned; i < n; ++i) r = r + term(i);
  return r;
}
// Same order for a contiguous block whose first element sits `start_off`
// (0 or 1) doubles past a 16-byte boundary (Eigen first_default_aligned).
double esum_block(const double* x, i64 n, int start_off);

inline double esum(const double* x, i64 n) {
  return esum_fn(n, [x](i64 i) { return x[i]; });
}
inline double sqnorm(const double* x, i64 n) {
  return esum_fn(n, [x](i64 i) { return x[i] * x[i]; });
}
inline double dot(const double* x, const double* y, i64 n) {
  return esum_fn(n, [x, y](i64 i) { return x[i] * y[i]; });
}
inline double sqnorm(const Mat& m) { return sqnorm(m.a.data(), m.size()); }
inline double norm(const Mat& m) { return std::sqrt(sqnorm(m)); }
inline double sqnorm(const Vec& v) { return sqnorm(v.data(), i64(v.size())); }
inline double norm(const Vec& v) { return std::sqrt(sqnorm(v)); }
inline double dot(const Vec& a, const Vec& b) { return dot(a.data(), b.data(), i64(a.size())); }
inline double frob_dot(const Mat& a, const Mat& b) { return dot(a.a.data(), b.a.data(), a.size()); }
bool all_finite(const Mat& m);
bool all_finite(const Vec& v);

// Symmetric eigen-decomposition by tournament-ordered cyclic Jacobi.
// H is k x k column-major; outputs ascending eigenvalues and the matching
// unit eigenvectors (column-major k x k), signs normalised.
void jacobi_eigh(int k, const double* H, double* evals, double* evecs);

// -------------------------------------------------------------- parallel ---
void set_max_threads(int n);
int max_threads();
void parallel_for(i64 n, i64 grain, const std::function<void(i64, i64)>& body);

// ------------------------------------------------------------------- rng ---
class Rng {
 public:
  explicit Rng(u64 seed);
  u64 next_u64();
  double uniform();
  u64 uniform_below(u64 bound);
  double normal();

 private:
  u64 s_[4];
  double cached_ = 0.0;
  bool has_cached_ = false;
};
Mat gaussian_matrix(i64 rows, i64 cols, Rng& rng);
Vec gaussian_vector(i64 n, Rng& rng);

// ----------------------------------------------------------------- graph ---
struct Graph {
  i64 n_vertices = 0;
  std::vector<std::pair<i64, i64>> edges;  // i < j, sorted, unique
  int dropped_self_loops = 0;
};
Graph make_cycle(int n);
Graph make_petersen();
Graph make_hypercube(int d);
Graph graph_from_pairs(i64 n_hint, const std::vector<std::pair<i64, i64>>& raw);
Graph load_graph(const std::string& path, int format);  // 0 edge-list, 1 mm, 2 gset

// -------------------------------------------------------------- instance ---
enum class Field { kReal = 0, kComplexEmbedded = 1 };

struct Instance {
  i64 n = 0, m = 0;
  Vec b;
  double tau = 1.0, norm_b1 = 0.0, norm_C1 = 0.0;
  Field field = Field::kReal;
  std::optional<i64> identity_constraint;
  std::function<Mat(const Mat&)> apply_C;
  std::function<Mat(const Vec&, const Mat&)> apply_adjoint;
  std::function<Vec(const Mat&)> apply_map;
  std::function<Mat(const Vec&, const Mat&)> apply_C_plus_adjoint;

  Mat C_plus_adjoint(const Vec& q, const Mat& U) const;
  void validate() const;
  void check_dims(const Mat& U, const char* where) const;
};

Instance theta_instance(const Graph& g);

struct McData {
  Instance inst;
  Mat hidden_U, hidden_V;
  double nuclear_norm = 0.0;
  std::vector<i64> omega_i, omega_j;
};
i64 mc_count(i64 n1, i64 n2, int r, bool offset);
McData matrix_completion(i64 n1, i64 n2, int r, u64 seed, bool offset,
                         double tau_safety, i64 paper_draws = 0);

struct PrData {
  Instance inst;
  std::vector<cplx> hidden_x;  // nc
  std::vector<cplx> masks;     // nc x L column-major
  i64 nc = 0;
  int L = 0;
};
PrData phase_retrieval(i64 n, int L, u64 seed, double tau_slack);

// Gaussian-measurement phase retrieval (NOT in the
// reference, parity unpinned against it): b_i = |a_i^* x|^2 for given
// measurement vectors a_i in C^n (A_re, A_im: m x n row-major) and signal x;
// C = I, tau = tau_slack ||x||^2, real embedding [Re u; Im u] as the
// coded-diffraction family (instances.cpp:266-269, 341-387).
Instance gauss_pr_instance(i64 n, i64 m, const double* A_re, const double* A_im,
                           const std::vector<cplx>& x, double tau_slack);

// Explicit dense SDP (tests/support/oracles.hpp DenseInstance).
struct DenseSdp {
  Mat C;
  std::vector<Mat> A;
  Vec b;
  double tau = 1.0;
};
Instance dense_instance(const DenseSdp& d);

void fft_plan_twiddles(i64 n, std::vector<cplx>& tw, std::vector<i64>& rev);
void fft_run(cplx* x, i64 n, const std::vector<cplx>& tw,
             const std::vector<i64>& rev, bool inverse);

// ------------------------------------------------------------- sdp core ---
double al_value(const Instance& I, const Mat& U, const Vec& p, double beta);
Mat al_gradient(const Instance& I, const Mat& U, const Vec& p, double beta);
struct GradOp {
  const Instance* I;
  Vec q, residual;
  GradOp(const Instance& inst, const Mat& U, const Vec& p, double beta);
  Mat apply(const Mat& V) const;
  Vec apply_vec(const Vec& v) const;
};
Mat project_ball(const Mat& U);
struct AlFn {
  const Instance* I;
  Vec p;
  double beta;
  double value(const Mat& U) const;
  Mat gradient(const Mat& U) const;
  std::pair<double, Mat> value_and_gradient(const Mat& U) const;
};

// ------------------------------------------------------------- subsolvers --
struct Smooth {
  std::function<double(const Mat&)> value;
  std::function<Mat(const Mat&)> gradient;
  std::function<std::pair<double, Mat>(const Mat&)> value_and_gradient;
  std::pair<double, Mat> eval(const Mat& x) const {
    if (value_and_gradient) return value_and_gradient(x);
    return {value(x), gradient(x)};
  }
};
struct FistaParams {
  double sigma = 0.3, chi = 0.5, mu = 0.5, L0 = 1.0;
  int max_iters = 0;
  void validate() const;
};
enum class FistaStatus { kSuccess = 0, kFailure = 1, kIterLimit = 2 };
struct FistaResult {
  FistaStatus status = FistaStatus::kFailure;
  Mat y, v;
  double L = 0, psi_y = 0;
  int iters = 0;
  Mat x_tilde;
  double A = 0;
};
FistaResult fista(const Smooth& psi, const Mat& x0, const FistaParams& prm);

struct AippParams {
  double lambda0 = 10.0, rho = 1e-4;
  FistaParams fista;
  int max_outer = 2000;
  double lambda_underflow = 1e-12;
  void validate() const;
};
enum class AippStatus { kConverged = 0, kIterLimit = 1, kLambdaUnderflow = 2 };
struct AippResult {
  AippStatus status = AippStatus::kConverged;
  Mat W, R;
  double R_norm = 0, g_value = 0, lambda = 0;
  int prox_iters = 0, fista_iters = 0;
};
AippResult aipp(const Smooth& g, const Mat& W_init, const AippParams& prm);

struct EigSettings {
  double tol = 1e-8;
  int max_iters = 5000;
  int block_restart = 30;
  u64 seed = 0;
  void validate() const;
};
struct EigResult {
  double lambda = 0.0;
  Vec v;
  double residual = 0.0;
  int matvecs = 0;
  bool converged = false;
};
using LinOp = std::function<Vec(const Vec&)>;
EigResult min_eigenpair(const LinOp& op, i64 n, const EigSettings& cfg);

// -------------------------------------------------------------------- hlr --
struct TraceEvent {
  int kind = 2;  // 0 stationary, 1 rank step, 2 outer
  int outer_iter = 0;
  double beta = 0, eps_inner = 0, gap = 0, theta = 0;
  i64 rank = 0;
  double al_value = 0, fw_alpha = 0, rel_pfeas = 0, rel_gap = 0, rel_dfeas = 0;
};
using Sink = std::function<void(const TraceEvent&)>;

struct HlrStats {
  int aipp_calls = 0;
  long aipp_iters = 0, fista_iters = 0, eig_products = 0;
  int fw_steps = 0;
};
enum class HlrStatus { kConverged = 0, kStepLimit = 1, kTimeLimit = 2 };
struct HlrSettings {
  EigSettings eig;
  AippParams aipp;
  int max_fw_steps = 500;
  int outer_iter = 0;
  std::optional<std::chrono::steady_clock::time_point> deadline;
};
struct HlrOutcome {
  Mat U;
  double theta = 0, gap = 0, lambda_min = 0, al_val = 0, cdot = 0;
  Vec residual;
  bool eig_trusted = true;
  HlrStats stats;
  HlrStatus status = HlrStatus::kConverged;
};
double fw_gap(const GradOp& G, const Mat& Y, double theta);
struct Escape {
  double theta = 0;
  Vec y;
  double lambda_min = 0, eig_residual = 0;
  int eig_products = 0;
  bool eig_trusted = true;
};
Escape escape_direction(const GradOp& G, i64 n, const EigSettings& cfg);
double fw_stepsize(const Instance& I, const Mat& Y, const Vec& y, double theta,
                   const Vec& p, double beta);
Mat rank_update(const Mat& Y, const Vec& y, double alpha);
HlrOutcome hlr_solve(const Instance& I, Mat U_init, const Vec& p, double beta,
                     double eps_t, const HlrSettings& hs, const Sink& sink);

// ----------------------------------------------------------------- solver --
struct SolverConfig {
  double eps = 1e-5, beta0 = 0.0, beta_growth = 2.0, eps0 = 0.0,
         eps_decay = 0.5, eps_floor = 0.0;
  int max_outer = 500;
  double time_limit = 3600.0;
  u64 seed = 0;
  EigSettings eig;
  AippParams aipp;
  int max_fw_steps = 500;
  void validate() const;
};
enum class SolveStatus { kOptimal = 0, kIterationLimit = 1, kTimeLimit = 2, kNumericalFailure = 3 };
struct SolveReport {
  SolveStatus status = SolveStatus::kIterationLimit;
  double pval = 0, dval = 0, dval_no_theta = 0, rel_pfeas = 0, rel_gap = 0,
         rel_dfeas = 0;
  i64 rank = 0;
  int outer_iters = 0, fw_steps = 0;
  long aipp_iters = 0, fista_iters = 0, eig_products = 0;
  double wall_seconds = 0;
  std::string message;
  Mat U;
  Vec p;
  double theta = 0, tau = 1.0;
};
struct Termination {
  double rel_pfeas = 0, rel_gap = 0, rel_dfeas = 0, pval = 0, dval = 0,
         dual_lambda_min = 0;
  long eig_products = 0;
  bool eig_trusted = true, done = false;
};
Instance scale_instance(const Instance& I, double* tau_orig);
Termination check_termination(const Instance& I, const Mat& U, const Vec& p,
                              double theta, const EigSettings& eig, double eps);
SolveReport solve(const Instance& I, const SolverConfig& cfg, const Sink& sink);
SolveReport solve_warm(const Instance& I, const SolverConfig& cfg,
                       const Mat& U0, const Vec& p0, const Sink& sink);

}  // namespace orc
