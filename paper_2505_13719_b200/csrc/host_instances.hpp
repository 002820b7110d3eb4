// Host-side instance construction for the B200 HALLaR product (C++).
// Bit-exact restatement of the reference generators so that constraint index
// sets, right-hand sides and start vectors are identical:
//   Rng            rng.cpp:9-80   (xoshiro256++, splitmix64 seeding, Box-Muller)
//   graphs         graph.cpp:56-148
//   theta          instances.cpp:63-112
//   matcomp        instances.cpp:117-234
//   phaseret       instances.cpp:239-389 (masks, hidden signal, b)
#pragma once

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace hallar_host {

struct InputError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

class Xoshiro {
 public:
  explicit Xoshiro(uint64_t seed);
  uint64_t next();
  double uniform();
  uint64_t below(uint64_t bound);
  double normal();
  void state(uint64_t out[4]) const {
    for (int i = 0; i < 4; ++i) out[i] = s_[i];
  }

 private:
  uint64_t s_[4];
  double spare_ = 0.0;
  bool has_spare_ = false;
};

// `count` consecutive standard normals of Xoshiro(seed) (gaussian_vector).
std::vector<double> gaussian_stream(uint64_t seed, int64_t count);

struct HostInst {
  int family = 0;  // 0 theta, 1 matcomp, 2 phaseret
  int64_t n = 0, m = 0, np = 0;
  bool has_trace = false;
  std::vector<int32_t> ei, ej;  // pair constraints, sorted by (ei, ej), ei < ej
  std::vector<double> b;        // length m, unscaled
  double tau = 1.0, norm_b1 = 0.0, norm_C1 = 0.0, nuclear = 0.0;
  int64_t n1 = 0;  // matcomp: rows of M (pair j = n1 + column)
  // phase retrieval
  int64_t nc = 0;
  int L = 0;
  std::vector<std::complex<double>> hidden_x, masks;  // masks nc x L column-major
  std::vector<std::complex<double>> twiddle;          // FftPlan forward twiddles
};

using Edges = std::vector<std::pair<int64_t, int64_t>>;

Edges edges_hypercube(int d);
Edges edges_cycle(int n);
Edges edges_petersen();
// load_graph: 0 edge-list, 1 matrix-market (pattern), 2 gset; returns n
Edges edges_from_file(const std::string& path, int fmt, int64_t* n_out);
// dedupe / drop self-loops / sort (EdgeAccumulator::finish)
Edges normalise_edges(int64_t n_hint, const Edges& raw, int64_t* n_out);

HostInst make_theta(int64_t n, const Edges& sorted_unique_edges);
int64_t matcomp_count(int64_t n1, int64_t n2, int r, bool offset);
// paper_draws > 0: the paper's sampling rule (that many draws with replacement,
// deduplicated) instead of instances.cpp:123-159
HostInst make_matcomp(int64_t n1, int64_t n2, int r, uint64_t seed, bool offset,
                      double tau_safety, int64_t paper_draws = 0);
// The host part of gen_matrix_completion that precedes the sample draws:
// hidden factors (column-major), the RNG state after them, the sample count
// (reference rule) and the nuclear norm / tau.  The draws themselves are made
// by devgen.cu (or by make_matcomp on the host).
struct McPrefix {
  int64_t m_target = 0;  // 0 under the paper rule
  std::vector<double> U, V;
  uint64_t state[4] = {0, 0, 0, 0};
  double nuclear = 0.0, tau = 0.0;
};
McPrefix matcomp_prefix(int64_t n1, int64_t n2, int r, uint64_t seed, bool offset, double tau_safety,
                        int64_t paper_draws);
HostInst make_phaseret(int64_t n, int L, uint64_t seed, double tau_slack);
// Gaussian-measurement phase retrieval (not in the
// reference): the signal x from Rng(seed) as make_phaseret draws it; the
// measurement vectors are generated on the device (devgen.cu gauss_fill).
HostInst make_gauss_pr(int64_t n, int64_t m, int parts, uint64_t seed, double tau_slack);

// Eigen LinearVectorized redux order (SSE2, 2 accumulators of 2 lanes).
double eigen_order_sum_sq(const double* x, int64_t n);
double eigen_order_sum_abs(const double* x, int64_t n);
// sum_i (x_i / tau)^2 in the same order (scale_instance, then squaredNorm)
double eigen_order_sum_sq_scaled(const double* x, int64_t n, double tau);

}  // namespace hallar_host
