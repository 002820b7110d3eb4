// Oracle support layer: reductions, Jacobi eigen-solver, parallel_for, RNG,
// graph builders.  TEST INFRASTRUCTURE ONLY (see orc.hpp).
#include <algorithm>
#include <atomic>
#include <fstream>
#include <sstream>
#include <thread>

#include "orc.hpp"

namespace orc {

// Eigen redux with a non-zero aligned start (first element 8 bytes past a
// 16-byte boundary): packets cover [start, start+aligned), then the peeled
// head element(s), then the tail (Eigen Redux.h LinearVectorizedTraversal).
double esum_block(const double* x, i64 n, int start_off) {
  if (start_off == 0 || n <= 0) return esum(x, n);
  const i64 st = std::min<i64>(start_off, n);
  const i64 rest = n - st;
  const i64 aligned = (rest / 2) * 2;
  if (aligned == 0) {
    double r = x[0];
    for (i64 i = 1; i < n; ++i) r = r + x[i];
    return r;
  }
  const double* y = x + st;
  double p0a = y[0], p0b = y[1];
  if (aligned > 2) {
    const i64 aligned2 = (rest / 4) * 4;
    double p1a = y[2], p1b = y[3];
    for (i64 i = 4; i < aligned2; i += 4) {
      p0a = p0a + y[i];
      p0b = p0b + y[i + 1];
      p1a = p1a + y[i + 2];
      p1b = p1b + y[i + 3];
    }
    p0a = p0a + p1a;
    p0b = p0b + p1b;
    if (aligned > aligned2) {
      p0a = p0a + y[aligned2];
      p0b = p0b + y[aligned2 + 1];
    }
  }
  double r = p0a + p0b;
  for (i64 i = 0; i < st; ++i) r = r + x[i];
  for (i64 i = st + aligned; i < n; ++i) r = r + x[i];
  return r;
}

bool all_finite(const Mat& m) {
  for (double v : m.a)
    if (!std::isfinite(v)) return false;
  return true;
}
bool all_finite(const Vec& v) {
  for (double x : v)
    if (!std::isfinite(x)) return false;
  return true;
}

// ---------------------------------------------------------------- Jacobi ---
// Tournament (circle-method) ordering: k' = k rounded up to even; in round r
// player positions rotate with player 0 fixed.  Within a round all pair
// rotations are applied to rows first, then to columns, then the pivots are
// zeroed.  The device eigensolver (csrc/solver.cuh jacobi_dev) uses the same
// rotation schedule and formulas with a looser stopping threshold (2 ulp of
// the largest entry); this checker keeps the tight one (over-converged, like
// Eigen's full-precision SelfAdjointEigenSolver).
void jacobi_eigh(int k, const double* H, double* evals, double* evecs) {
  std::vector<double> A(H, H + size_t(k) * k);
  std::vector<double> V(static_cast<size_t>(k) * k, 0.0);
  for (int i = 0; i < k; ++i) V[size_t(i) * k + i] = 1.0;
  auto a = [&](int i, int j) -> double& { return A[size_t(i) + size_t(j) * k]; };
  auto vv = [&](int i, int j) -> double& { return V[size_t(i) + size_t(j) * k]; };
  if (k > 1) {
    const int kp = k + (k & 1);
    double scale = 0.0;
    for (int j = 0; j < k; ++j)
      for (int i = 0; i < k; ++i) scale = std::max(scale, std::fabs(a(i, j)));
    const double thresh = scale * 1e-18;
    std::vector<int> P(kp), Q(kp / 2), R(kp / 2);
    std::vector<double> cs(kp / 2), sn(kp / 2);
    for (int sweep = 0; sweep < 40; ++sweep) {
      double off = 0.0;
      for (int j = 0; j < k; ++j)
        for (int i = 0; i < j; ++i) off = std::max(off, std::fabs(a(i, j)));
      if (off <= thresh || off == 0.0) break;
      for (int round = 0; round < kp - 1; ++round) {
        // positions: pos[0] = 0, pos[t] = 1 + (t - 1 + round) % (kp - 1)
        for (int t = 0; t < kp; ++t)
          P[t] = t == 0 ? 0 : 1 + (t - 1 + round) % (kp - 1);
        int np = 0;
        for (int t = 0; t < kp / 2; ++t) {
          int x = P[t], y = P[kp - 1 - t];
          if (x >= k || y >= k) continue;
          if (x > y) std::swap(x, y);
          Q[np] = x;
          R[np] = y;
          ++np;
        }
        for (int t = 0; t < np; ++t) {
          const int p = Q[t], q = R[t];
          const double apq = a(p, q);
          double c = 1.0, s = 0.0;
          if (apq != 0.0) {
            const double th = (a(q, q) - a(p, p)) / (2.0 * apq);
            double tn;
            if (std::fabs(th) > 1e150)
              tn = 0.5 / th;
            else
              tn = (th >= 0.0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
            c = 1.0 / std::sqrt(tn * tn + 1.0);
            s = tn * c;
          }
          cs[t] = c;
          sn[t] = s;
        }
        for (int t = 0; t < np; ++t) {  // rows p,q
          const int p = Q[t], q = R[t];
          const double c = cs[t], s = sn[t];
          if (s == 0.0) continue;
          for (int j = 0; j < k; ++j) {
            const double ap = a(p, j), aq = a(q, j);
            a(p, j) = c * ap - s * aq;
            a(q, j) = s * ap + c * aq;
          }
        }
        for (int t = 0; t < np; ++t) {  // columns p,q (and eigenvectors)
          const int p = Q[t], q = R[t];
          const double c = cs[t], s = sn[t];
          if (s == 0.0) continue;
          for (int i = 0; i < k; ++i) {
            const double ap = a(i, p), aq = a(i, q);
            a(i, p) = c * ap - s * aq;
            a(i, q) = s * ap + c * aq;
            const double vp = vv(i, p), vq = vv(i, q);
            vv(i, p) = c * vp - s * vq;
            vv(i, q) = s * vp + c * vq;
          }
        }
        for (int t = 0; t < np; ++t) {
          if (sn[t] == 0.0) continue;
          a(Q[t], R[t]) = 0.0;
          a(R[t], Q[t]) = 0.0;
        }
      }
    }
  }
  // ascending order (stable on ties), sign: largest-|.| component positive
  std::vector<int> ord(k);
  for (int i = 0; i < k; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(),
                   [&](int x, int y) { return a(x, x) < a(y, y); });
  for (int c = 0; c < k; ++c) {
    const int src = ord[c];
    evals[c] = a(src, src);
    int imax = 0;
    double best = -1.0;
    for (int i = 0; i < k; ++i)
      if (std::fabs(vv(i, src)) > best) {
        best = std::fabs(vv(i, src));
        imax = i;
      }
    const double sg = vv(imax, src) < 0.0 ? -1.0 : 1.0;
    for (int i = 0; i < k; ++i) evecs[size_t(i) + size_t(c) * k] = sg * vv(i, src);
  }
}

// -------------------------------------------------------------- parallel ---
// Same contract as the reference (parallel.cpp:22-47): fixed chunking by
// grain, chunks claimed from an atomic counter, threads spawned per call.
namespace {
std::atomic<int> g_threads{0};
}
void set_max_threads(int n) { g_threads.store(n < 0 ? 0 : n); }
int max_threads() {
  int n = g_threads.load();
  if (n == 0) n = int(std::thread::hardware_concurrency());
  return std::max(1, n);
}
void parallel_for(i64 n, i64 grain, const std::function<void(i64, i64)>& body) {
  if (n <= 0) return;
  grain = std::max<i64>(1, grain);
  const i64 chunks = (n + grain - 1) / grain;
  const int workers = int(std::min<i64>(chunks, max_threads()));
  if (workers <= 1) {
    body(0, n);
    return;
  }
  std::atomic<i64> next{0};
  auto run = [&] {
    for (i64 c; (c = next.fetch_add(1)) < chunks;) {
      const i64 lo = c * grain;
      body(lo, std::min(n, lo + grain));
    }
  };
  std::vector<std::thread> pool;
  for (int w = 1; w < workers; ++w) pool.emplace_back(run);
  run();
  for (auto& t : pool) t.join();
}

// ------------------------------------------------------------------- rng ---
// xoshiro256++ seeded by splitmix64 (reference rng.cpp:9-67).
static inline u64 rotl64(u64 x, int k) { return (x << k) | (x >> (64 - k)); }

Rng::Rng(u64 seed) {
  u64 z0 = seed;
  for (int w = 0; w < 4; ++w) {
    z0 += 0x9e3779b97f4a7c15ULL;
    u64 z = z0;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    s_[w] = z ^ (z >> 31);
  }
}
u64 Rng::next_u64() {
  const u64 out = rotl64(s_[0] + s_[3], 23) + s_[0];
  const u64 sh = s_[1] << 17;
  s_[2] ^= s_[0];
  s_[3] ^= s_[1];
  s_[1] ^= s_[2];
  s_[0] ^= s_[3];
  s_[2] ^= sh;
  s_[3] = rotl64(s_[3], 45);
  return out;
}
double Rng::uniform() { return double(next_u64() >> 11) * 0x1.0p-53; }
u64 Rng::uniform_below(u64 bound) {
  need(bound > 0, "uniform_below: bound must be positive");
  const u64 floor_ = (0 - bound) % bound;
  for (;;) {
    const u64 r = next_u64();
    if (r >= floor_) return r % bound;
  }
}
double Rng::normal() {
  if (has_cached_) {
    has_cached_ = false;
    return cached_;
  }
  double u1;
  do u1 = uniform();
  while (u1 <= 0.0);
  const double u2 = uniform();
  const double rad = std::sqrt(-2.0 * std::log(u1));
  const double ang = 2.0 * M_PI * u2;
  cached_ = rad * std::sin(ang);
  has_cached_ = true;
  return rad * std::cos(ang);
}
Mat gaussian_matrix(i64 rows, i64 cols, Rng& rng) {
  Mat M(rows, cols);
  for (auto& x : M.a) x = rng.normal();  // column by column
  return M;
}
Vec gaussian_vector(i64 n, Rng& rng) {
  Vec v(static_cast<size_t>(n));
  for (auto& x : v) x = rng.normal();
  return v;
}

// ----------------------------------------------------------------- graph ---
Graph graph_from_pairs(i64 n_hint, const std::vector<std::pair<i64, i64>>& raw) {
  Graph g;
  i64 vmax = 0;
  for (auto [u, v] : raw) {
    vmax = std::max({vmax, u, v});
    if (u == v) {
      ++g.dropped_self_loops;
      continue;
    }
    g.edges.emplace_back(std::min(u, v), std::max(u, v));
  }
  std::sort(g.edges.begin(), g.edges.end());
  g.edges.erase(std::unique(g.edges.begin(), g.edges.end()), g.edges.end());
  g.n_vertices = std::max(n_hint, vmax + 1);
  if (g.n_vertices <= 0 || g.edges.empty()) throw InputError("graph is empty");
  return g;
}

Graph make_cycle(int n) {
  need(n >= 3, "cycle graph needs n >= 3");
  Graph g;
  g.n_vertices = n;
  for (int v = 0; v + 1 < n; ++v) g.edges.emplace_back(v, v + 1);
  g.edges.emplace_back(0, n - 1);
  std::sort(g.edges.begin(), g.edges.end());
  return g;
}

Graph make_petersen() {
  Graph g;
  g.n_vertices = 10;
  for (int v = 0; v < 5; ++v) {
    const std::pair<i64, i64> es[3] = {
        {v, (v + 1) % 5}, {v, v + 5}, {v + 5, (v + 2) % 5 + 5}};
    for (auto e : es) g.edges.emplace_back(std::min(e.first, e.second),
                                            std::max(e.first, e.second));
  }
  std::sort(g.edges.begin(), g.edges.end());
  return g;
}

Graph make_hypercube(int d) {
  need(d >= 1 && d < 26, "hypercube dimension out of range");
  Graph g;
  g.n_vertices = i64(1) << d;
  for (i64 v = 0; v < g.n_vertices; ++v)
    for (int bit = 0; bit < d; ++bit) {
      const i64 u = v ^ (i64(1) << bit);
      if (v < u) g.edges.emplace_back(v, u);
    }
  std::sort(g.edges.begin(), g.edges.end());
  return g;
}

// Edge list / Matrix Market pattern / GSET reader (reference graph.cpp:56-109).
Graph load_graph(const std::string& path, int format) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open graph file '" + path + "'");
  std::vector<std::pair<i64, i64>> raw;
  std::string line;
  long lineno = 0;
  i64 n_hint = 0;
  bool header = false;
  auto fail = [&](const std::string& w) {
    throw InputError(path + ":" + std::to_string(lineno) + ": " + w);
  };
  while (std::getline(in, line)) {
    ++lineno;
    const auto f = line.find_first_not_of(" \t\r");
    if (f == std::string::npos) continue;
    const char c = line[f];
    if (c == '#') continue;
    if (format == 1 && c == '%') {
      if (line.find("%%MatrixMarket") != std::string::npos &&
          line.find("pattern") == std::string::npos)
        fail("expected a pattern matrix");
      continue;
    }
    std::istringstream ss(line.substr(f));
    if (!header && (format == 1 || format == 2)) {
      long n = 0, n2 = 0, nnz = 0;
      if (format == 2) {
        if (!(ss >> n >> nnz)) fail("bad GSET header");
      } else {
        if (!(ss >> n >> n2 >> nnz)) fail("bad Matrix Market size line");
        if (n != n2) fail("adjacency matrix must be square");
      }
      if (n <= 0) fail("non-positive vertex count");
      n_hint = n;
      header = true;
      continue;
    }
    long u = 0, v = 0;
    if (!(ss >> u >> v)) fail("expected two vertex indices");
    if (u < 1 || v < 1) fail("vertex indices are 1-based");
    if (n_hint > 0 && (u > n_hint || v > n_hint))
      fail("vertex index exceeds declared count");
    raw.emplace_back(u - 1, v - 1);
  }
  return graph_from_pairs(n_hint, raw);
}

}  // namespace orc
