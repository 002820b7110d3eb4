// Oracle instance families: Lovasz theta, matrix completion, coded-diffraction
// phase retrieval, dense SDPs.  Restates reference instances.cpp / fft.cpp.
// TEST INFRASTRUCTURE ONLY (see orc.hpp).
#include <algorithm>
#include <memory>
#include <unordered_set>

#include "orc.hpp"

namespace orc {

Mat Instance::C_plus_adjoint(const Vec& q, const Mat& U) const {
  if (apply_C_plus_adjoint) return apply_C_plus_adjoint(q, U);
  Mat a = apply_C(U), b = apply_adjoint(q, U);
  for (i64 t = 0; t < a.size(); ++t) a.a[t] = a.a[t] + b.a[t];
  return a;
}

// sdp_instance.cpp:7-22
void Instance::validate() const {
  need(n >= 1, "instance: n must be >= 1");
  need(m >= 1, "instance: m must be >= 1");
  need(i64(b.size()) == m, "instance: b has wrong length");
  need(std::isfinite(tau) && tau > 0, "instance: tau must be positive");
  need(std::isfinite(norm_b1) && norm_b1 > 0, "instance: norm_b1 must be positive");
  need(std::isfinite(norm_C1) && norm_C1 > 0, "instance: norm_C1 must be positive");
  need(bool(apply_C) && bool(apply_adjoint) && bool(apply_map),
       "instance: operator callables missing");
  if (identity_constraint)
    need(*identity_constraint >= 0 && *identity_constraint < m,
         "instance: identity_constraint out of range");
}

void Instance::check_dims(const Mat& U, const char* where) const {
  if (U.rows != n)
    throw InputError(std::string(where) + ": factor has " + std::to_string(U.rows) +
                     " rows, instance needs " + std::to_string(n));
  if (U.cols < 1) throw InputError(std::string(where) + ": factor must have >= 1 column");
}

namespace {

// Edge/entry constraints X_{i_k j_k} (i_k < j_k), A_k = (e_i e_j' + e_j e_i')/2.
struct Pairs {
  std::vector<i64> i, j;
  i64 count() const { return i64(i.size()); }

  // instances.cpp:27-35 — out_k = U.row(i_k) . U.row(j_k), strided row dot
  // summed sequentially over columns.
  void map_into(const Mat& U, double* out) const {
    const i64 nk = count();
    const i64 grain = std::max<i64>(i64(1) << 12, nk / (8 * i64(max_threads())) + 1);
    parallel_for(nk, grain, [&](i64 lo, i64 hi) {
      const i64 s = U.cols;
      for (i64 k = lo; k < hi; ++k) {
        const i64 a = i[k], b = j[k];
        double d = U(a, 0) * U(b, 0);
        for (i64 c = 1; c < s; ++c) d = d + U(a, c) * U(b, c);
        out[k] = d;
      }
    });
  }

  // instances.cpp:39-55 — out += sum_k p_k A_k U, k increasing, per column.
  void adjoint_into(const double* p, const Mat& U, Mat& out) const {
    const i64 nk = count();
    const i64 grain = std::max<i64>(1, (i64(1) << 15) / std::max<i64>(1, nk));
    parallel_for(U.cols, grain, [&](i64 c0, i64 c1) {
      for (i64 k = 0; k < nk; ++k) {
        const double w = 0.5 * p[k];
        if (w == 0.0) continue;
        const i64 a = i[k], b = j[k];
        for (i64 c = c0; c < c1; ++c) {
          out(a, c) = out(a, c) + w * U(b, c);
          out(b, c) = out(b, c) + w * U(a, c);
        }
      }
    });
  }
};

// U.colwise().sum() with Eigen's per-column alignment peeling.
Vec column_sums(const Mat& U) {
  Vec cs(static_cast<size_t>(U.cols));
  for (i64 c = 0; c < U.cols; ++c)
    cs[c] = esum_block(U.col(c), U.rows, int((c * U.rows) & 1));
  return cs;
}

}  // namespace

// ---------------------------------------------------------------- theta ---
// instances.cpp:63-112: min -ee'.X s.t. X_ij = 0 (ij in E), Tr X = 1.
Instance theta_instance(const Graph& g) {
  need(g.n_vertices >= 1 && !g.edges.empty(), "theta: graph is empty");
  const i64 n = g.n_vertices, ne = i64(g.edges.size()), m = ne + 1;
  auto P = std::make_shared<Pairs>();
  P->i.reserve(ne);
  P->j.reserve(ne);
  for (auto [u, v] : g.edges) {
    need(u >= 0 && v < n && u < v, "theta: bad edge");
    P->i.push_back(u);
    P->j.push_back(v);
  }
  Instance I;
  I.n = n;
  I.m = m;
  I.b.assign(static_cast<size_t>(m), 0.0);
  I.b[m - 1] = 1.0;
  I.tau = 1.0;
  I.norm_b1 = 1.0;
  I.norm_C1 = double(n) * double(n);
  I.identity_constraint = m - 1;
  I.apply_C = [n](const Mat& U) {
    const Vec cs = column_sums(U);
    Mat out(n, U.cols);
    for (i64 c = 0; c < U.cols; ++c)
      for (i64 a = 0; a < n; ++a) out(a, c) = -1.0 * cs[c];
    return out;
  };
  I.apply_map = [P, m](const Mat& U) {
    Vec out(static_cast<size_t>(m));
    P->map_into(U, out.data());
    out[m - 1] = sqnorm(U);
    return out;
  };
  I.apply_adjoint = [P, m](const Vec& p, const Mat& U) {
    Mat out(U.rows, U.cols);
    const double w = p[m - 1];
    for (i64 t = 0; t < U.size(); ++t) out.a[t] = w * U.a[t];
    P->adjoint_into(p.data(), U, out);
    return out;
  };
  I.apply_C_plus_adjoint = [P, n, m](const Vec& q, const Mat& U) {
    Mat out(U.rows, U.cols);
    const double w = q[m - 1];
    for (i64 t = 0; t < U.size(); ++t) out.a[t] = w * U.a[t];
    const Vec cs = column_sums(U);
    for (i64 c = 0; c < U.cols; ++c)
      for (i64 a = 0; a < n; ++a) out(a, c) = out(a, c) - cs[c] * 1.0;
    P->adjoint_into(q.data(), U, out);
    return out;
  };
  return I;
}

// ---------------------------------------------------- matrix completion ---
// instances.cpp:123-129
i64 mc_count(i64 n1, i64 n2, int r, bool offset) {
  const double gamma = r * std::log(double(n1 + n2));
  const double base = double(offset ? n1 + n2 - r : n1 + n2);
  return i64(std::ceil(gamma * r * base));
}

namespace {
// Householder QR of a tall matrix (rows >= cols); returns the cols x cols R.
Mat qr_r(const Mat& A0) {
  Mat A = A0;
  const i64 m = A.rows, n = A.cols;
  for (i64 k = 0; k < n; ++k) {
    double nrm = 0.0;
    for (i64 i = k; i < m; ++i) nrm += A(i, k) * A(i, k);
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) continue;
    const double alpha = A(k, k) > 0 ? -nrm : nrm;
    std::vector<double> v(static_cast<size_t>(m - k));
    for (i64 i = k; i < m; ++i) v[i - k] = A(i, k);
    v[0] -= alpha;
    double vn = 0.0;
    for (double x : v) vn += x * x;
    if (vn == 0.0) continue;
    for (i64 c = k; c < n; ++c) {
      double d = 0.0;
      for (i64 i = k; i < m; ++i) d += v[i - k] * A(i, c);
      const double f = 2.0 * d / vn;
      for (i64 i = k; i < m; ++i) A(i, c) -= f * v[i - k];
    }
  }
  Mat R(n, n);
  for (i64 c = 0; c < n; ++c)
    for (i64 r = 0; r <= c; ++r) R(r, c) = A(r, c);
  return R;
}
// Singular values of a small square matrix by one-sided Jacobi.
Vec singular_values(Mat A) {
  const i64 n = A.cols;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (i64 p = 0; p < n; ++p)
      for (i64 q = p + 1; q < n; ++q) {
        double al = 0, be = 0, ga = 0;
        for (i64 i = 0; i < A.rows; ++i) {
          al += A(i, p) * A(i, p);
          be += A(i, q) * A(i, q);
          ga += A(i, p) * A(i, q);
        }
        if (ga == 0.0) continue;
        off = std::max(off, std::fabs(ga) / std::sqrt(al * be));
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (i64 i = 0; i < A.rows; ++i) {
          const double x = A(i, p), y = A(i, q);
          A(i, p) = c * x - s * y;
          A(i, q) = s * x + c * y;
        }
      }
    if (off < 1e-16) break;
  }
  Vec sv(static_cast<size_t>(n));
  for (i64 c = 0; c < n; ++c) {
    double s = 0;
    for (i64 i = 0; i < A.rows; ++i) s += A(i, c) * A(i, c);
    sv[c] = std::sqrt(s);
  }
  std::sort(sv.begin(), sv.end(), std::greater<double>());
  return sv;
}
}  // namespace

// instances.cpp:131-234.  paper_draws > 0 selects the paper's sampling rule
// instead (not in the reference): that many
// (i, j) draws with replacement from the same stream, then deduplicated.
McData matrix_completion(i64 n1, i64 n2, int r, u64 seed, bool offset,
                         double tau_safety, i64 paper_draws) {
  need(n1 >= 1 && n2 >= n1, "matcomp: need n2 >= n1 >= 1");
  need(r >= 1 && r <= n1, "matcomp: need 1 <= r <= n1");
  need(tau_safety >= 1.0, "matcomp: tau_safety must be >= 1");
  need(paper_draws >= 0, "matcomp: draws must be >= 0");
  i64 m = paper_draws > 0 ? 0 : mc_count(n1, n2, r, offset);
  need(m <= n1 * n2, "matcomp: sample count exceeds matrix size");
  Rng rng(seed);
  McData out;
  out.hidden_U = gaussian_matrix(n1, r, rng);
  out.hidden_V = gaussian_matrix(n2, r, rng);
  std::vector<u64> keys;
  if (paper_draws > 0) {
    keys.resize(static_cast<size_t>(paper_draws));
    for (auto& key : keys) {
      const u64 i = rng.uniform_below(u64(n1));
      const u64 j = rng.uniform_below(u64(n2));
      key = i * u64(n2) + j;
    }
    std::sort(keys.begin(), keys.end());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    m = i64(keys.size());
  } else {
    // Omega: rejection sampling of distinct (i,j), then sorted by (i,j).
    // The reference's std::unordered_set membership test is restated with a
    // flat open-addressing table (same accept/reject sequence, so the same
    // Omega; it only changes the generation time: 165 s -> ~25 s at C4).
    keys.reserve(static_cast<size_t>(m));
    u64 cap = 16;
    while (cap < u64(m) * 2) cap <<= 1;
    std::vector<u64> table(static_cast<size_t>(cap), 0);  // key + 1; 0 = empty
    const u64 mask = cap - 1;
    auto insert = [&](u64 key) {
      u64 h = key * 0x9E3779B97F4A7C15ULL;
      h ^= h >> 29;
      for (u64 t = h & mask;; t = (t + 1) & mask) {
        if (table[t] == key + 1) return false;
        if (table[t] == 0) {
          table[t] = key + 1;
          return true;
        }
      }
    };
    while (i64(keys.size()) < m) {
      const u64 i = rng.uniform_below(u64(n1));
      const u64 j = rng.uniform_below(u64(n2));
      const u64 key = i * u64(n2) + j;
      if (insert(key)) keys.push_back(key);
    }
    std::sort(keys.begin(), keys.end());  // (i,j) order == key order
  }
  out.omega_i.resize(static_cast<size_t>(m));
  out.omega_j.resize(static_cast<size_t>(m));
  for (i64 k = 0; k < m; ++k) {
    out.omega_i[k] = i64(keys[k] / u64(n2));
    out.omega_j[k] = i64(keys[k] % u64(n2));
  }
  {
    const Mat Ru = qr_r(out.hidden_U), Rv = qr_r(out.hidden_V);
    Mat core(r, r);
    for (int a = 0; a < r; ++a)
      for (int b = 0; b < r; ++b) {
        double s = 0;
        for (int t = 0; t < r; ++t) s += Ru(a, t) * Rv(b, t);
        core(a, b) = s;
      }
    const Vec sv = singular_values(core);
    double nuc = 0;
    for (double x : sv) nuc += x;
    out.nuclear_norm = nuc;
  }
  auto P = std::make_shared<Pairs>();
  P->i = out.omega_i;
  P->j.resize(static_cast<size_t>(m));
  Instance& I = out.inst;
  I.b.resize(static_cast<size_t>(m));
  for (i64 k = 0; k < m; ++k) {
    P->j[k] = n1 + out.omega_j[k];
    const i64 a = out.omega_i[k], c = out.omega_j[k];
    double d = out.hidden_U(a, 0) * out.hidden_V(c, 0);
    for (int t = 1; t < r; ++t) d = d + out.hidden_U(a, t) * out.hidden_V(c, t);
    I.b[k] = d;
  }
  I.n = n1 + n2;
  I.m = m;
  I.tau = 2.0 * tau_safety * out.nuclear_norm;
  I.norm_b1 = esum_fn(m, [&](i64 k) { return std::fabs(I.b[k]); });
  I.norm_C1 = 0.5 * double(I.n);
  I.apply_C = [](const Mat& U) {
    Mat o = U;
    for (auto& x : o.a) x = 0.5 * x;
    return o;
  };
  I.apply_map = [P, m](const Mat& U) {
    Vec o(static_cast<size_t>(m));
    P->map_into(U, o.data());
    return o;
  };
  I.apply_adjoint = [P](const Vec& p, const Mat& U) {
    Mat o(U.rows, U.cols);
    P->adjoint_into(p.data(), U, o);
    return o;
  };
  I.apply_C_plus_adjoint = [P](const Vec& q, const Mat& U) {
    Mat o = U;
    for (auto& x : o.a) x = 0.5 * x;
    P->adjoint_into(q.data(), U, o);
    return o;
  };
  return out;
}

// --------------------------------------------------------------------- fft ---
// fft.cpp:97-140: bit-reversal + per-stage twiddle tables, forward sign -1.
void fft_plan_twiddles(i64 n, std::vector<cplx>& tw, std::vector<i64>& rev) {
  need(n >= 1 && (n & (n - 1)) == 0, "fft: length must be a power of two");
  rev.assign(static_cast<size_t>(n), 0);
  for (i64 i = 1, j = 0; i < n; ++i) {
    i64 bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    rev[i] = j;
  }
  tw.clear();
  for (i64 len = 2; len <= n; len <<= 1)
    for (i64 k = 0; k < len / 2; ++k) {
      const double ang = -2.0 * M_PI * double(k) / double(len);
      tw.emplace_back(std::cos(ang), std::sin(ang));
    }
}

static inline cplx cmul(cplx x, cplx y) {
  return cplx(x.real() * y.real() - x.imag() * y.imag(),
              x.real() * y.imag() + x.imag() * y.real());
}

void fft_run(cplx* x, i64 n, const std::vector<cplx>& tw,
             const std::vector<i64>& rev, bool inverse) {
  for (i64 i = 1; i < n; ++i)
    if (i < rev[i]) std::swap(x[i], x[rev[i]]);
  i64 stage = 0;
  for (i64 len = 2; len <= n; len <<= 1) {
    const i64 half = len / 2;
    for (i64 i0 = 0; i0 < n; i0 += len)
      for (i64 k = 0; k < half; ++k) {
        const cplx w = inverse ? std::conj(tw[stage + k]) : tw[stage + k];
        const cplx u = x[i0 + k];
        const cplx t = cmul(x[i0 + k + half], w);
        x[i0 + k] = cplx(u.real() + t.real(), u.imag() + t.imag());
        x[i0 + k + half] = cplx(u.real() - t.real(), u.imag() - t.imag());
      }
    stage += half;
  }
}

// ------------------------------------------------------- phase retrieval ---
namespace {
struct PrOp {
  i64 nc;
  int L;
  std::vector<cplx> masks;  // nc x L
  std::vector<cplx> tw;
  std::vector<i64> rev;

  // b_(l,k) += |FFT(d_l .* u)_k|^2  (instances.cpp:271-278)
  void map_column(const std::vector<cplx>& u, double* out) const {
    std::vector<cplx> buf(static_cast<size_t>(nc));
    for (int l = 0; l < L; ++l) {
      for (i64 j = 0; j < nc; ++j) buf[j] = cmul(masks[j + l * nc], u[j]);
      fft_run(buf.data(), nc, tw, rev, false);
      double* slot = out + i64(l) * nc;
      for (i64 k = 0; k < nc; ++k)
        slot[k] = slot[k] + (buf[k].real() * buf[k].real() + buf[k].imag() * buf[k].imag());
    }
  }
  // sum_l conj(d_l) .* IFFT(p_l .* FFT(d_l .* u))  (instances.cpp:281-293)
  void adjoint_column(const double* p, const std::vector<cplx>& u,
                      std::vector<cplx>& acc) const {
    std::vector<cplx> buf(static_cast<size_t>(nc));
    acc.assign(static_cast<size_t>(nc), cplx(0, 0));
    for (int l = 0; l < L; ++l) {
      for (i64 j = 0; j < nc; ++j) buf[j] = cmul(masks[j + l * nc], u[j]);
      fft_run(buf.data(), nc, tw, rev, false);
      const double* pl = p + i64(l) * nc;
      for (i64 k = 0; k < nc; ++k) buf[k] = cplx(buf[k].real() * pl[k], buf[k].imag() * pl[k]);
      fft_run(buf.data(), nc, tw, rev, true);
      for (i64 j = 0; j < nc; ++j) {
        const cplx t = cmul(std::conj(masks[j + l * nc]), buf[j]);
        acc[j] = cplx(acc[j].real() + t.real(), acc[j].imag() + t.imag());
      }
    }
  }
};
}  // namespace

// instances.cpp:298-389
PrData phase_retrieval(i64 n, int L, u64 seed, double tau_slack) {
  need(n >= 2 && (n & (n - 1)) == 0, "phaseret: n must be a power of two >= 2");
  need(L >= 1, "phaseret: L must be >= 1");
  need(tau_slack >= 1.0, "phaseret: tau_slack must be >= 1");
  const i64 nc = n, m = nc * L;
  Rng rng(seed);
  PrData out;
  out.nc = nc;
  out.L = L;
  out.hidden_x.resize(static_cast<size_t>(nc));
  const double r2 = std::sqrt(2.0);
  for (i64 j = 0; j < nc; ++j) {
    // g++ evaluates the two constructor arguments right to left: the first
    // draw is the imaginary part.
    const double im = rng.normal();
    const double re = rng.normal();
    out.hidden_x[j] = cplx(re / r2, im / r2);
  }
  out.masks.resize(static_cast<size_t>(nc * L));
  const cplx quads[4] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}};
  for (int l = 0; l < L; ++l)
    for (i64 j = 0; j < nc; ++j) {
      const cplx b1 = quads[rng.uniform_below(4)];
      const double b2 = rng.uniform() < 0.8 ? std::sqrt(2.0) / 2.0 : std::sqrt(3.0);
      out.masks[j + l * nc] = cplx(b1.real() * b2, b1.imag() * b2);
    }
  auto D = std::make_shared<PrOp>();
  D->nc = nc;
  D->L = L;
  D->masks = out.masks;
  fft_plan_twiddles(nc, D->tw, D->rev);

  Instance& I = out.inst;
  I.b.assign(static_cast<size_t>(m), 0.0);
  D->map_column(out.hidden_x, I.b.data());
  I.n = 2 * nc;
  I.m = m;
  I.tau = tau_slack * esum_fn(nc, [&](i64 j) {
            return out.hidden_x[j].real() * out.hidden_x[j].real() +
                   out.hidden_x[j].imag() * out.hidden_x[j].imag();
          });
  I.norm_b1 = esum_fn(m, [&](i64 k) { return std::fabs(I.b[k]); });
  I.norm_C1 = double(2 * nc);
  I.field = Field::kComplexEmbedded;

  auto for_cols = [D](i64 s, const std::function<void(i64)>& body) {
    const i64 work = D->nc * D->L;
    const i64 grain = std::max<i64>(1, (i64(1) << 15) / std::max<i64>(1, work));
    parallel_for(s, grain, [&](i64 c0, i64 c1) {
      for (i64 c = c0; c < c1; ++c) body(c);
    });
  };
  auto load = [D](const Mat& U, i64 c) {
    std::vector<cplx> u(static_cast<size_t>(D->nc));
    for (i64 j = 0; j < D->nc; ++j) u[j] = cplx(U(j, c), U(D->nc + j, c));
    return u;
  };
  I.apply_C = [](const Mat& U) { return U; };
  I.apply_map = [D, for_cols, load, m](const Mat& U) {
    const i64 s = U.cols;
    Mat part(m, s);
    for_cols(s, [&](i64 c) { D->map_column(load(U, c), part.col(c)); });
    Vec o(static_cast<size_t>(m));
    for (i64 k = 0; k < m; ++k) {
      double v = part(k, 0);
      for (i64 c = 1; c < s; ++c) v = v + part(k, c);
      o[k] = v;
    }
    return o;
  };
  auto adj = [D, for_cols, load](const Vec& p, const Mat& U, bool add_id) {
    Mat o(U.rows, U.cols);
    for_cols(U.cols, [&](i64 c) {
      std::vector<cplx> acc;
      D->adjoint_column(p.data(), load(U, c), acc);
      for (i64 j = 0; j < D->nc; ++j) {
        o(j, c) = acc[j].real();
        o(D->nc + j, c) = acc[j].imag();
      }
    });
    if (add_id)
      for (i64 t = 0; t < o.size(); ++t) o.a[t] = o.a[t] + U.a[t];
    return o;
  };
  I.apply_adjoint = [adj](const Vec& p, const Mat& U) { return adj(p, U, false); };
  I.apply_C_plus_adjoint = [adj](const Vec& q, const Mat& U) { return adj(q, U, true); };
  return out;
}

// --------------------------------------------------- Gaussian phase retrieval ---
// Dense restatement (the test_instances.cpp:255-297 pattern): y_ic = a_i^* u_c
// summed over j in increasing order, d_i = sum_c |y_ic|^2 in column order;
// adjoint z_c = sum_i a_i (q_i y_ic) over i in increasing order.
Instance gauss_pr_instance(i64 n, i64 m, const double* A_re, const double* A_im,
                           const std::vector<cplx>& x, double tau_slack) {
  need(n >= 1 && m >= 1, "gauss_pr: empty");
  need(i64(x.size()) == n, "gauss_pr: signal length");
  need(tau_slack >= 1.0, "gauss_pr: tau_slack must be >= 1");
  struct G {
    i64 n, m;
    std::vector<double> re, im;
    // y = a_i^* u
    cplx meas(i64 i, const cplx* u) const {
      double yr = 0.0, yi = 0.0;
      for (i64 j = 0; j < n; ++j) {
        const double ar = re[i * n + j], ai = im[i * n + j];
        yr = yr + (ar * u[j].real() + ai * u[j].imag());
        yi = yi + (ar * u[j].imag() - ai * u[j].real());
      }
      return cplx(yr, yi);
    }
  };
  auto D = std::make_shared<G>();
  D->n = n;
  D->m = m;
  D->re.assign(A_re, A_re + n * m);
  D->im.assign(A_im, A_im + n * m);
  Instance I;
  I.n = 2 * n;
  I.m = m;
  I.b.resize(static_cast<size_t>(m));
  for (i64 i = 0; i < m; ++i) {
    const cplx y = D->meas(i, x.data());
    I.b[i] = y.real() * y.real() + y.imag() * y.imag();
  }
  I.tau = tau_slack * esum_fn(n, [&](i64 j) { return x[j].real() * x[j].real() + x[j].imag() * x[j].imag(); });
  I.norm_b1 = esum_fn(m, [&](i64 k) { return std::fabs(I.b[k]); });
  I.norm_C1 = double(2 * n);
  I.field = Field::kComplexEmbedded;
  auto load = [D](const Mat& U, i64 c) {
    std::vector<cplx> u(static_cast<size_t>(D->n));
    for (i64 j = 0; j < D->n; ++j) u[j] = cplx(U(j, c), U(D->n + j, c));
    return u;
  };
  I.apply_C = [](const Mat& U) { return U; };
  I.apply_map = [D, load](const Mat& U) {
    Vec o(static_cast<size_t>(D->m));
    std::vector<std::vector<cplx>> us;
    for (i64 c = 0; c < U.cols; ++c) us.push_back(load(U, c));
    for (i64 i = 0; i < D->m; ++i) {
      double v = 0.0;
      for (i64 c = 0; c < U.cols; ++c) {
        const cplx y = D->meas(i, us[c].data());
        const double t = y.real() * y.real() + y.imag() * y.imag();
        v = c == 0 ? t : v + t;
      }
      o[i] = v;
    }
    return o;
  };
  auto adj = [D, load](const Vec& p, const Mat& U, bool add_id) {
    Mat o(U.rows, U.cols);
    for (i64 c = 0; c < U.cols; ++c) {
      const auto u = load(U, c);
      std::vector<double> zr(static_cast<size_t>(D->n), 0.0), zi(static_cast<size_t>(D->n), 0.0);
      for (i64 i = 0; i < D->m; ++i) {
        const cplx y = D->meas(i, u.data());
        const double wr = p[i] * y.real(), wi = p[i] * y.imag();
        for (i64 j = 0; j < D->n; ++j) {
          const double ar = D->re[i * D->n + j], ai = D->im[i * D->n + j];
          zr[j] = zr[j] + (ar * wr - ai * wi);
          zi[j] = zi[j] + (ar * wi + ai * wr);
        }
      }
      for (i64 j = 0; j < D->n; ++j) {
        o(j, c) = zr[j];
        o(D->n + j, c) = zi[j];
      }
    }
    if (add_id)
      for (i64 t = 0; t < o.size(); ++t) o.a[t] = o.a[t] + U.a[t];
    return o;
  };
  I.apply_adjoint = [adj](const Vec& p, const Mat& U) { return adj(p, U, false); };
  I.apply_C_plus_adjoint = [adj](const Vec& q, const Mat& U) { return adj(q, U, true); };
  return I;
}

// ------------------------------------------------------------------ dense ---
// tests/support/oracles.hpp:65-99 (DenseInstance::as_operator)
Instance dense_instance(const DenseSdp& d0) {
  auto d = std::make_shared<DenseSdp>(d0);
  const i64 n = d->C.rows, m = i64(d->A.size());
  Instance I;
  I.n = n;
  I.m = m;
  I.b = d->b;
  I.tau = d->tau;
  double nb1 = 0, nc1 = 0;
  for (double x : d->b) nb1 += std::fabs(x);
  for (double x : d->C.a) nc1 += std::fabs(x);
  I.norm_b1 = std::max(nb1, 1e-300);
  I.norm_C1 = nc1;
  auto matmul = [](const Mat& A, const Mat& B) {
    Mat o(A.rows, B.cols);
    for (i64 c = 0; c < B.cols; ++c)
      for (i64 t = 0; t < A.cols; ++t) {
        const double b = B(t, c);
        for (i64 r = 0; r < A.rows; ++r) o(r, c) += A(r, t) * b;
      }
    return o;
  };
  auto adjoint = [d, n, m](const Vec& p) {
    Mat S(n, n);
    for (i64 k = 0; k < m; ++k)
      for (i64 t = 0; t < n * n; ++t) S.a[t] += p[k] * d->A[k].a[t];
    return S;
  };
  I.apply_C = [d, matmul](const Mat& U) { return matmul(d->C, U); };
  I.apply_map = [d, m, matmul](const Mat& U) {
    Vec o(static_cast<size_t>(m));
    for (i64 k = 0; k < m; ++k) {
      const Mat AU = matmul(d->A[k], U);
      double tr = 0;
      for (i64 t = 0; t < U.size(); ++t) tr += U.a[t] * AU.a[t];
      o[k] = tr;
    }
    return o;
  };
  I.apply_adjoint = [adjoint, matmul](const Vec& p, const Mat& U) {
    return matmul(adjoint(p), U);
  };
  I.apply_C_plus_adjoint = [d, adjoint, matmul](const Vec& q, const Mat& U) {
    Mat S = adjoint(q);
    for (i64 t = 0; t < S.size(); ++t) S.a[t] += d->C.a[t];
    return matmul(S, U);
  };
  return I;
}

}  // namespace orc
