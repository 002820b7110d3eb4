// Host-side instance construction (see host_instances.hpp).
#include "host_instances.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <sstream>

namespace hallar_host {

// ------------------------------------------------------------------- RNG ---
static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

Xoshiro::Xoshiro(uint64_t seed) {
  uint64_t st = seed;
  for (auto& w : s_) {
    st += 0x9e3779b97f4a7c15ULL;
    uint64_t z = st;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    w = z ^ (z >> 31);
  }
}
uint64_t Xoshiro::next() {
  const uint64_t r = rotl(s_[0] + s_[3], 23) + s_[0];
  const uint64_t t = s_[1] << 17;
  s_[2] ^= s_[0];
  s_[3] ^= s_[1];
  s_[1] ^= s_[2];
  s_[0] ^= s_[3];
  s_[2] ^= t;
  s_[3] = rotl(s_[3], 45);
  return r;
}
double Xoshiro::uniform() { return double(next() >> 11) * 0x1.0p-53; }
uint64_t Xoshiro::below(uint64_t bound) {
  if (bound == 0) throw InputError("uniform_below: bound must be positive");
  const uint64_t lim = (0 - bound) % bound;
  uint64_t r;
  do r = next();
  while (r < lim);
  return r % bound;
}
double Xoshiro::normal() {
  if (has_spare_) {
    has_spare_ = false;
    return spare_;
  }
  double u1 = uniform();
  while (u1 <= 0.0) u1 = uniform();
  const double u2 = uniform();
  const double rad = std::sqrt(-2.0 * std::log(u1));
  const double ang = 2.0 * M_PI * u2;
  spare_ = rad * std::sin(ang);
  has_spare_ = true;
  return rad * std::cos(ang);
}

std::vector<double> gaussian_stream(uint64_t seed, int64_t count) {
  Xoshiro g(seed);
  std::vector<double> v(static_cast<size_t>(count));
  for (auto& x : v) x = g.normal();
  return v;
}

// ----------------------------------------------------------- reductions ---
template <class F>
static double eigen_sum(int64_t n, F f) {
  if (n <= 0) return 0.0;
  const int64_t al = n / 2 * 2;
  if (al == 0) return f(0);
  double a0 = f(0), a1 = f(1);
  if (al > 2) {
    const int64_t al4 = n / 4 * 4;
    double b0 = f(2), b1 = f(3);
    for (int64_t i = 4; i < al4; i += 4) {
      a0 += f(i);
      a1 += f(i + 1);
      b0 += f(i + 2);
      b1 += f(i + 3);
    }
    a0 += b0;
    a1 += b1;
    if (al > al4) {
      a0 += f(al4);
      a1 += f(al4 + 1);
    }
  }
  double r = a0 + a1;
  for (int64_t i = al; i < n; ++i) r += f(i);
  return r;
}
double eigen_order_sum_sq(const double* x, int64_t n) {
  return eigen_sum(n, [x](int64_t i) { return x[i] * x[i]; });
}
double eigen_order_sum_sq_scaled(const double* x, int64_t n, double tau) {
  if (tau == 1.0) return eigen_order_sum_sq(x, n);
  return eigen_sum(n, [x, tau](int64_t i) {
    const double y = x[i] / tau;
    return y * y;
  });
}
double eigen_order_sum_abs(const double* x, int64_t n) {
  return eigen_sum(n, [x](int64_t i) { return std::fabs(x[i]); });
}

// ---------------------------------------------------------------- graphs ---
Edges normalise_edges(int64_t n_hint, const Edges& raw, int64_t* n_out) {
  Edges e;
  e.reserve(raw.size());
  int64_t vmax = 0;
  for (auto [u, v] : raw) {
    vmax = std::max({vmax, u, v});
    if (u != v) e.emplace_back(std::min(u, v), std::max(u, v));
  }
  std::sort(e.begin(), e.end());
  e.erase(std::unique(e.begin(), e.end()), e.end());
  *n_out = std::max(n_hint, vmax + 1);
  if (*n_out <= 0 || e.empty()) throw InputError("graph is empty");
  return e;
}

Edges edges_hypercube(int d) {
  if (d < 1 || d >= 26) throw InputError("hypercube dimension out of range");
  const int64_t n = int64_t(1) << d;
  Edges e;
  e.reserve(size_t(n) * d / 2);
  // (v, v ^ 2^bit) for v < u is produced in sorted order when bits ascend
  for (int64_t v = 0; v < n; ++v)
    for (int bit = 0; bit < d; ++bit) {
      const int64_t u = v ^ (int64_t(1) << bit);
      if (v < u) e.emplace_back(v, u);
    }
  return e;
}
Edges edges_cycle(int n) {
  if (n < 3) throw InputError("cycle graph needs n >= 3");
  Edges e;
  for (int i = 0; i + 1 < n; ++i) e.emplace_back(i, i + 1);
  e.emplace_back(0, n - 1);
  std::sort(e.begin(), e.end());
  return e;
}
Edges edges_petersen() {
  Edges e;
  for (int i = 0; i < 5; ++i) {
    const int64_t pr[3][2] = {{i, (i + 1) % 5}, {i, i + 5}, {i + 5, (i + 2) % 5 + 5}};
    for (auto& p : pr) e.emplace_back(std::min(p[0], p[1]), std::max(p[0], p[1]));
  }
  std::sort(e.begin(), e.end());
  return e;
}
Edges edges_from_file(const std::string& path, int fmt, int64_t* n_out) {
  std::ifstream in(path);
  if (!in) throw std::ios_base::failure("cannot open graph file '" + path + "'");
  Edges raw;
  std::string line;
  long ln = 0;
  int64_t n_hint = 0;
  bool header = false;
  auto bad = [&](const char* w) {
    throw InputError(path + ":" + std::to_string(ln) + ": " + w);
  };
  while (std::getline(in, line)) {
    ++ln;
    const auto f = line.find_first_not_of(" \t\r");
    if (f == std::string::npos || line[f] == '#') continue;
    if (fmt == 1 && line[f] == '%') {
      if (line.find("%%MatrixMarket") != std::string::npos &&
          line.find("pattern") == std::string::npos)
        bad("expected a pattern matrix");
      continue;
    }
    std::istringstream ss(line.substr(f));
    if (!header && (fmt == 1 || fmt == 2)) {
      long a = 0, b = 0, c = 0;
      if (fmt == 2) {
        if (!(ss >> a >> c)) bad("bad GSET header");
      } else {
        if (!(ss >> a >> b >> c)) bad("bad Matrix Market size line");
        if (a != b) bad("adjacency matrix must be square");
      }
      if (a <= 0) bad("non-positive vertex count");
      n_hint = a;
      header = true;
      continue;
    }
    long u = 0, v = 0;
    if (!(ss >> u >> v)) bad("expected two vertex indices");
    if (u < 1 || v < 1) bad("vertex indices are 1-based");
    if (n_hint > 0 && (u > n_hint || v > n_hint)) bad("vertex index exceeds declared count");
    raw.emplace_back(u - 1, v - 1);
  }
  return normalise_edges(n_hint, raw, n_out);
}

// ----------------------------------------------------------------- theta ---
HostInst make_theta(int64_t n, const Edges& edges) {
  if (n < 1 || edges.empty()) throw InputError("theta: graph is empty");
  if (n >= (int64_t(1) << 31)) throw InputError("theta: more than 2^31 vertices");
  HostInst h;
  h.family = 0;
  h.n = n;
  h.np = int64_t(edges.size());
  h.m = h.np + 1;
  h.has_trace = true;
  h.ei.resize(h.np);
  h.ej.resize(h.np);
  for (int64_t k = 0; k < h.np; ++k) {
    const auto [u, v] = edges[k];
    if (!(u >= 0 && v < n && u < v)) throw InputError("theta: bad edge");
    h.ei[k] = int32_t(u);
    h.ej[k] = int32_t(v);
  }
  h.b.assign(size_t(h.m), 0.0);
  h.b[h.m - 1] = 1.0;
  h.tau = 1.0;
  h.norm_b1 = 1.0;
  h.norm_C1 = double(n) * double(n);
  return h;
}

// ------------------------------------------------------ matrix completion ---
int64_t matcomp_count(int64_t n1, int64_t n2, int r, bool offset) {
  const double gamma = r * std::log(double(n1 + n2));
  const double base = double(offset ? n1 + n2 - r : n1 + n2);
  return int64_t(std::ceil(gamma * r * base));
}

namespace {
// open-addressing set of uint64 keys (key+1 stored; 0 = empty)
struct KeySet {
  std::vector<uint64_t> tab;
  uint64_t mask;
  explicit KeySet(uint64_t want) {
    uint64_t cap = 16;
    while (cap < want * 2) cap <<= 1;
    tab.assign(cap, 0);
    mask = cap - 1;
  }
  bool insert(uint64_t key) {
    const uint64_t v = key + 1;
    uint64_t h = key * 0x9E3779B97F4A7C15ULL;
    h ^= h >> 29;
    for (uint64_t i = h & mask;; i = (i + 1) & mask) {
      if (tab[i] == v) return false;
      if (tab[i] == 0) {
        tab[i] = v;
        return true;
      }
    }
  }
};

// LSD radix sort of uint64 keys (8 passes of 8 bits, skipping trivial passes)
void radix_sort(std::vector<uint64_t>& a) {
  std::vector<uint64_t> tmp(a.size());
  for (int sh = 0; sh < 64; sh += 8) {
    size_t cnt[257] = {0};
    for (uint64_t x : a) ++cnt[((x >> sh) & 255) + 1];
    bool trivial = false;
    for (int b = 1; b <= 256; ++b)
      if (cnt[b] == a.size()) trivial = true;
    if (trivial) continue;
    for (int b = 0; b < 256; ++b) cnt[b + 1] += cnt[b];
    for (uint64_t x : a) tmp[cnt[(x >> sh) & 255]++] = x;
    a.swap(tmp);
  }
}

// R factor of a tall n x r matrix (column-major) by Householder QR.
std::vector<double> house_r(std::vector<double> A, int64_t m, int r) {
  for (int k = 0; k < r; ++k) {
    double nrm = 0.0;
    for (int64_t i = k; i < m; ++i) nrm += A[i + k * m] * A[i + k * m];
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) continue;
    const double alpha = A[k + k * m] > 0 ? -nrm : nrm;
    std::vector<double> v(size_t(m - k));
    for (int64_t i = k; i < m; ++i) v[i - k] = A[i + k * m];
    v[0] -= alpha;
    double vn = 0.0;
    for (double x : v) vn += x * x;
    if (vn == 0.0) continue;
    for (int c = k; c < r; ++c) {
      double d = 0.0;
      for (int64_t i = k; i < m; ++i) d += v[i - k] * A[i + c * m];
      const double f = 2.0 * d / vn;
      for (int64_t i = k; i < m; ++i) A[i + c * m] -= f * v[i - k];
    }
  }
  std::vector<double> R(size_t(r) * r, 0.0);
  for (int c = 0; c < r; ++c)
    for (int i = 0; i <= c; ++i) R[i + c * r] = A[i + c * m];
  return R;
}
// sum of singular values of a small r x r matrix (one-sided Jacobi)
double nuclear_small(std::vector<double> A, int r) {
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < r; ++p)
      for (int q = p + 1; q < r; ++q) {
        double al = 0, be = 0, ga = 0;
        for (int i = 0; i < r; ++i) {
          al += A[i + p * r] * A[i + p * r];
          be += A[i + q * r] * A[i + q * r];
          ga += A[i + p * r] * A[i + q * r];
        }
        if (ga == 0.0) continue;
        off = std::max(off, std::fabs(ga) / std::sqrt(al * be));
        const double z = (be - al) / (2.0 * ga);
        const double t = (z >= 0 ? 1.0 : -1.0) / (std::fabs(z) + std::sqrt(1.0 + z * z));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (int i = 0; i < r; ++i) {
          const double x = A[i + p * r], y = A[i + q * r];
          A[i + p * r] = c * x - s * y;
          A[i + q * r] = s * x + c * y;
        }
      }
    if (off < 1e-16) break;
  }
  std::vector<double> sv(r);
  for (int c = 0; c < r; ++c) {
    double s = 0;
    for (int i = 0; i < r; ++i) s += A[i + c * r] * A[i + c * r];
    sv[c] = std::sqrt(s);
  }
  std::sort(sv.begin(), sv.end(), std::greater<double>());
  double nuc = 0;
  for (double x : sv) nuc += x;
  return nuc;
}
}  // namespace

namespace {
void matcomp_check(int64_t n1, int64_t n2, int r, double tau_safety, int64_t paper_draws) {
  if (!(n1 >= 1 && n2 >= n1)) throw InputError("matcomp: need n2 >= n1 >= 1");
  if (!(r >= 1 && r <= n1)) throw InputError("matcomp: need 1 <= r <= n1");
  if (!(tau_safety >= 1.0)) throw InputError("matcomp: tau_safety must be >= 1");
  if (n1 + n2 >= (int64_t(1) << 31)) throw InputError("matcomp: n1 + n2 >= 2^31");
  if (paper_draws < 0) throw InputError("matcomp: draws must be >= 0");
}
// ||M||_* of M = U V' from the R factors (instances.cpp:179-187)
double matcomp_nuclear(const std::vector<double>& U, const std::vector<double>& V, int64_t n1, int64_t n2,
                       int r) {
  const auto Ru = house_r(U, n1, r), Rv = house_r(V, n2, r);
  std::vector<double> core(size_t(r) * r);
  for (int a = 0; a < r; ++a)
    for (int b = 0; b < r; ++b) {
      double s = 0;
      for (int t = 0; t < r; ++t) s += Ru[a + t * r] * Rv[b + t * r];
      core[a + b * r] = s;
    }
  return nuclear_small(core, r);
}
}  // namespace

McPrefix matcomp_prefix(int64_t n1, int64_t n2, int r, uint64_t seed, bool offset, double tau_safety,
                        int64_t paper_draws) {
  matcomp_check(n1, n2, r, tau_safety, paper_draws);
  McPrefix p;
  p.m_target = paper_draws > 0 ? 0 : matcomp_count(n1, n2, r, offset);
  if (p.m_target > n1 * n2) throw InputError("matcomp: sample count exceeds matrix size");
  Xoshiro g(seed);
  p.U.resize(size_t(n1) * r);
  p.V.resize(size_t(n2) * r);
  for (auto& x : p.U) x = g.normal();  // column-major fills (rng.cpp:69-74)
  for (auto& x : p.V) x = g.normal();
  g.state(p.state);
  p.nuclear = matcomp_nuclear(p.U, p.V, n1, n2, r);
  p.tau = 2.0 * tau_safety * p.nuclear;
  return p;
}

HostInst make_matcomp(int64_t n1, int64_t n2, int r, uint64_t seed, bool offset,
                      double tau_safety, int64_t paper_draws) {
  matcomp_check(n1, n2, r, tau_safety, paper_draws);
  int64_t m = paper_draws > 0 ? 0 : matcomp_count(n1, n2, r, offset);
  if (m > n1 * n2) throw InputError("matcomp: sample count exceeds matrix size");
  Xoshiro g(seed);
  std::vector<double> U(size_t(n1) * r), V(size_t(n2) * r);  // column-major fills
  for (auto& x : U) x = g.normal();
  for (auto& x : V) x = g.normal();
  std::vector<uint64_t> keys;
  if (paper_draws > 0) {
    // the paper's rule: draws with replacement, deduplicated
    keys.resize(size_t(paper_draws));
    for (auto& key : keys) {
      const uint64_t i = g.below(uint64_t(n1));
      const uint64_t j = g.below(uint64_t(n2));
      key = i * uint64_t(n2) + j;
    }
    radix_sort(keys);
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    m = int64_t(keys.size());
  } else {
    keys.reserve(size_t(m));
    KeySet set(uint64_t(m) + 1);
    while (int64_t(keys.size()) < m) {
      const uint64_t i = g.below(uint64_t(n1));
      const uint64_t j = g.below(uint64_t(n2));
      const uint64_t key = i * uint64_t(n2) + j;
      if (set.insert(key)) keys.push_back(key);
    }
    radix_sort(keys);  // (i, j) lexicographic == key order
  }
  HostInst h;
  h.family = 1;
  h.n = n1 + n2;
  h.n1 = n1;
  h.m = m;
  h.np = m;
  h.ei.resize(m);
  h.ej.resize(m);
  h.b.resize(m);
  for (int64_t k = 0; k < m; ++k) {
    const int64_t i = int64_t(keys[k] / uint64_t(n2)), j = int64_t(keys[k] % uint64_t(n2));
    h.ei[k] = int32_t(i);
    h.ej[k] = int32_t(n1 + j);
    double d = U[i] * V[j];
    for (int t = 1; t < r; ++t) d = d + U[i + t * n1] * V[j + t * n2];
    h.b[k] = d;
  }
  h.nuclear = matcomp_nuclear(U, V, n1, n2, r);
  h.tau = 2.0 * tau_safety * h.nuclear;
  h.norm_b1 = eigen_order_sum_abs(h.b.data(), m);
  h.norm_C1 = 0.5 * double(h.n);
  return h;
}

// -------------------------------------------------------- phase retrieval ---
HostInst make_phaseret(int64_t n, int L, uint64_t seed, double tau_slack) {
  if (!(n >= 2 && (n & (n - 1)) == 0)) throw InputError("phaseret: n must be a power of two >= 2");
  if (L < 1) throw InputError("phaseret: L must be >= 1");
  if (!(tau_slack >= 1.0)) throw InputError("phaseret: tau_slack must be >= 1");
  HostInst h;
  h.family = 2;
  h.nc = n;
  h.L = L;
  h.n = 2 * n;
  h.m = n * L;
  Xoshiro g(seed);
  h.hidden_x.resize(n);
  for (int64_t j = 0; j < n; ++j) {
    const double im = g.normal();  // g++ evaluates the ctor args right to left
    const double re = g.normal();
    h.hidden_x[j] = {re / std::sqrt(2.0), im / std::sqrt(2.0)};
  }
  const std::complex<double> quads[4] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}};
  h.masks.resize(size_t(n) * L);
  for (int l = 0; l < L; ++l)
    for (int64_t j = 0; j < n; ++j) {
      const auto b1 = quads[g.below(4)];
      const double b2 = g.uniform() < 0.8 ? std::sqrt(2.0) / 2.0 : std::sqrt(3.0);
      h.masks[j + l * n] = {b1.real() * b2, b1.imag() * b2};
    }
  for (int64_t len = 2; len <= n; len <<= 1)
    for (int64_t k = 0; k < len / 2; ++k) {
      const double ang = -2.0 * M_PI * double(k) / double(len);
      h.twiddle.emplace_back(std::cos(ang), std::sin(ang));
    }
  // ||x||^2 in the oracle's reduction order (hidden_x.squaredNorm())
  const double sx = eigen_sum(n, [&](int64_t j) {
    const auto& z = h.hidden_x[j];
    return z.real() * z.real() + z.imag() * z.imag();
  });
  h.tau = tau_slack * sx;
  h.norm_C1 = double(2 * n);
  // b is computed on the device (map of the hidden signal) by the caller.
  return h;
}

HostInst make_gauss_pr(int64_t n, int64_t m, int parts, uint64_t seed, double tau_slack) {
  if (n < 1 || m < 1) throw InputError("gauss_pr: n and m must be >= 1");
  if (!(tau_slack >= 1.0)) throw InputError("gauss_pr: tau_slack must be >= 1");
  HostInst h;
  h.family = 2;
  h.nc = n;
  h.L = parts;
  h.n = 2 * n;
  h.m = m;
  Xoshiro g(seed);
  h.hidden_x.resize(n);
  for (int64_t j = 0; j < n; ++j) {
    const double im = g.normal();
    const double re = g.normal();
    h.hidden_x[j] = {re / std::sqrt(2.0), im / std::sqrt(2.0)};
  }
  const double sx = eigen_sum(n, [&](int64_t j) {
    const auto& z = h.hidden_x[j];
    return z.real() * z.real() + z.imag() * z.imag();
  });
  h.tau = tau_slack * sx;
  h.norm_C1 = double(2 * n);
  return h;
}

}  // namespace hallar_host
