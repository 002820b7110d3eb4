// Parity mode (cuhallar_config.parity = 1): the HALLaR solve with every
// reduction in the checker's order, so the device takes the same decisions
// as the CPU oracle and reproduces its iteration counters.
//
// The fast solver (device.cuh / solver.cuh / solve.cuh) sums every norm, dot
// product and multiplier statistic in a fixed block/team tree: bitwise
// reproducible, but not the order of the reference binary, whose contiguous
// reductions are Eigen's LinearVectorized redux (two 2-wide packet
// accumulators = four interleaved partial sums) and whose
// Lanczos GEMVs are ordered dots.  FISTA's line search, AIPP's descent test
// and Lanczos' convergence test are knife-edge comparisons of such sums, so a
// 1-ulp difference can change the trajectory (H(12,2): 744 vs 18,611 FISTA
// iterations).  This path restates the oracle (oracle/src/algo.cpp, which
// restates adap_fista.cpp, adap_aipp.cpp, lanczos.cpp, hlr.cpp, solver.cpp
// statement by statement) with materialised vectors:
//   * the operator kernels are the fast path's bit-exact passes (map, fused
//     C + A*(q) row pass, gradient-operator pass);
//   * every scalar reduction is a "job": one CTA streams the terms through a
//     shared-memory ring (15 producer warps) while lanes 0..3 of warp 0 run
//     the four dependent partial-sum chains in Eigen order (or one ordered
//     chain for the CGS2 dots); the jobs of a phase run on different CTAs at
//     once and their results are broadcast through the team slots;
//   * factors stay row-major n x s in HBM; reductions over n x s visit them in
//     the reference's column-major order (index t -> row t % n, column t / n).
// Throughput is that of the dependent add chains (~latency of one FP64 add
// per term per chain); this mode is for parity runs on the BASELINE small
// configs, the fast mode for everything else.  Pair families, single GPU.
#pragma once

#include "solve.cuh"

namespace hallar {

enum PMode : int {
  kPmEigen = 0,   // Eigen redux, first element 16-byte aligned (esum_fn)
  kPmEigen1 = 1,  // Eigen redux, first element 8 bytes past alignment (esum_block, offset 1)
  kPmSeq = 2,     // s = 0.0; s = s + term(i), i increasing (ordered dot, algo.cpp cgs2)
};
constexpr int kPChunk = 512;  // terms per ring slot
constexpr int kPRing = 4;     // ring slots (producers run two chunks ahead)

// Layout of one reduction over term(i), i in [0, n): the Eigen packet chains
// cover [st, st + L4); the head (st = 1), the extra packet and the tail are
// at most 3 + 1 elements, folded at the end from the ring.
struct ChainLayout {
  int64_t n, st, aligned, aligned2, L4, nchunks;
  int mode;
  __device__ ChainLayout(int64_t n_, int mode_) : n(n_), st(0), aligned(0), aligned2(0), L4(0), mode(mode_) {
    if (mode != kPmSeq && n > 0) {
      st = mode == kPmEigen1 ? 1 : 0;
      const int64_t rest = n - st;
      aligned = (rest / 2) * 2;
      aligned2 = (rest / 4) * 4;
      L4 = aligned > 2 ? aligned2 : 0;
    }
    nchunks = n > 0 ? (n + kPChunk - 1) / kPChunk : 0;
  }
};

// warp 0: fold chunk ci (already in the ring) into the chain accumulators
__device__ __noinline__ void chain_consume(const ChainLayout& Lc, const double* ring, int64_t ci,
                                           double& acc, double& head) {
  const int lane = threadIdx.x & 31;
  const double* src = ring + (ci % kPRing) * kPChunk;
  const int64_t base = ci * kPChunk;
  const int cnt = (int)min((int64_t)kPChunk, Lc.n - base);
  if (Lc.mode == kPmSeq) {
    if (lane == 0)
      for (int i = 0; i < cnt; ++i) acc = acc + src[i];
    return;
  }
  if (ci == 0 && lane == 0 && Lc.st > 0) head = src[0];
  if (lane >= 4 || Lc.L4 == 0) return;
  // chain lane j owns i = st + j + 4t, t in [0, L4 / 4)
  const int64_t off = base - Lc.st - lane;  // i - base = 4t - off
  int64_t t = off > 0 ? (off + 3) / 4 : 0;
  const int64_t t_end = min(Lc.L4 / 4, (base + cnt - Lc.st - lane + 3) / 4);
  if (t == 0 && t < t_end) acc = src[-off], t = 1;  // p0a = y[0], p0b = y[1], p1a = y[2], p1b = y[3]
  for (; t < t_end; ++t) acc = acc + src[4 * t - off];
}

// warp 0 lane 0: p0a = y0 + y2 chains, p0b = y1 + y3, extra packet, lane
// sum, head, tail (orc::esum_fn / esum_block).  Elements past the chains sit
// in the last two chunks, still resident in the ring.
__device__ __noinline__ double chain_finish(const ChainLayout& Lc, const double* ring, double acc,
                                            double head) {
  const double a0 = __shfl_sync(0xffffffffu, acc, 0), a1 = __shfl_sync(0xffffffffu, acc, 1);
  const double a2 = __shfl_sync(0xffffffffu, acc, 2), a3 = __shfl_sync(0xffffffffu, acc, 3);
  auto at = [&](int64_t i) { return ring[((i / kPChunk) % kPRing) * kPChunk + i % kPChunk]; };
  if (Lc.mode == kPmSeq) return a0;
  const int64_t n = Lc.n, st = Lc.st;
  if (n <= 0) return 0.0;
  if (Lc.aligned == 0) {  // n <= 2: plain left-to-right
    double r = at(0);
    for (int64_t i = 1; i < n; ++i) r = r + at(i);
    return r;
  }
  double p0a, p0b;
  if (Lc.aligned > 2) {
    p0a = a0 + a2;
    p0b = a1 + a3;
    if (Lc.aligned > Lc.aligned2) {
      p0a = p0a + at(st + Lc.aligned2);
      p0b = p0b + at(st + Lc.aligned2 + 1);
    }
  } else {
    p0a = at(st);
    p0b = at(st + 1);
  }
  double r = p0a + p0b;
  if (st > 0) r = r + head;
  for (int64_t i = st + Lc.aligned; i < n; ++i) r = r + at(i);
  return r;
}

// One reduction by the whole CTA (all threads call).  Warps 1..15 evaluate
// term(i) into the ring two chunks ahead; warp 0 folds.  Returns the result
// in every thread.  Restates orc::esum_fn / esum_block (base.cpp:16-48,
// orc.hpp:67-96) and the ordered dot of algo.cpp:311-321.
template <class F>
__device__ double cta_chain(int64_t n, int mode, const F& term, double* ring, double* res) {
  const int tid = threadIdx.x, warp = tid >> 5;
  const ChainLayout Lc(n, mode);
  double acc = 0.0, head = 0.0;
  for (int64_t ci = -2; ci < Lc.nchunks; ++ci) {
    if (warp == 0) {
      if (ci >= 0) chain_consume(Lc, ring, ci, acc, head);
    } else if (ci + 2 < Lc.nchunks) {
      double* dst = ring + ((ci + 2) % kPRing) * kPChunk;
      const int64_t base = (ci + 2) * kPChunk;
      for (int e = tid - 32; e < kPChunk; e += kThreads - 32)
        if (base + e < n) dst[e] = term(base + e);
    }
    __syncthreads();
  }
  if (warp == 0) {
    const double r = chain_finish(Lc, ring, acc, head);
    if (tid == 0) *res = r;
  }
  __syncthreads();
  const double r = *res;
  __syncthreads();
  return r;
}

// A phase of K independent reductions: job j runs on CTA j % team (all of
// its threads), term(j, i) gives its i-th term.  Results land in
// c.rs.out[0..K) of every CTA.  Inputs must already be visible (team sync).
struct Jobs {
  int K = 0;
  int64_t len[kRedK];
  int mode[kRedK];
  __device__ int add(int64_t n, int m) {
    len[K] = n;
    mode[K] = m;
    return K++;
  }
};

template <class F>
__device__ __forceinline__ void par_jobs(Ctx& c, const Jobs& J, const F& term) {
  double* const ring = c.tw;
  double* const mine = c.t.slots + ((size_t)c.t.parity * c.t.lsize + c.t.lrank) * kRedK;
  for (int j = c.t.rank; j < J.K; j += c.t.size) {
    const double v = cta_chain(
        J.len[j], J.mode[j], [&](int64_t i) { return term(j, i); }, ring, c.rs.part);
    if (threadIdx.x == 0) mine[j] = v;
  }
  c.t.lsync();
  const double* base = c.t.slots + (size_t)c.t.parity * c.t.lsize * kRedK;
  if (threadIdx.x < (unsigned)J.K)
    c.rs.out[threadIdx.x] =
        __ldcg(base + (size_t)(threadIdx.x % c.t.lsize) * kRedK + threadIdx.x);
  c.t.parity ^= 1;
  __syncthreads();
  // cfg.trace >= 3: every job phase's results as debug events (kind 10)
  const Params& P = *c.Pp;
  if (P.cfg.trace >= 3 && P.trace && c.t.rank == 0 && threadIdx.x == 0) {
    const int i = *P.trace_count;
    if (i < P.trace_cap) {
      TraceEv ev{};
      ev.kind = 10;
      ev.outer_iter = i;
      ev.rank = J.K;
      const double* o = c.rs.out;
      ev.beta = o[0];
      ev.eps_inner = J.K > 1 ? o[1] : 0.0;
      ev.gap = J.K > 2 ? o[2] : 0.0;
      ev.theta = J.K > 3 ? o[3] : 0.0;
      ev.al_value = J.K > 4 ? o[4] : 0.0;
      ev.fw_alpha = J.K > 5 ? o[5] : 0.0;
      P.trace[i] = ev;
    }
    *P.trace_count = i + 1;
  }
}

// Parity-mode views of the instance: column-major index of an n x s factor
// stored row-major, m-vector terms with theta's trace constraint at k = np.
struct PView {
  int64_t n, np, m;
  int s;
  bool theta;
  __device__ __forceinline__ int64_t cm(int64_t t) const { return (t % n) * s + t / n; }
};

// Column sums + ||U||_F^2 of a factor (column_sums, families.cpp:83-88, and
// the trace constraint's sqnorm, :124): jobs [first, first + 1 + s).
__device__ __forceinline__ void jobs_stats(Jobs& J, const PView& v) {
  J.add(v.n * v.s, kPmEigen);
  for (int k = 0; k < v.s; ++k) J.add(v.n, ((int64_t)k * v.n) & 1 ? kPmEigen1 : kPmEigen);
}
__device__ __forceinline__ double term_stats(const PView& v, const double* U, int jrel, int64_t i) {
  if (jrel == 0) {
    const double u = U[v.cm(i)];
    return u * u;
  }
  return U[i * v.s + (jrel - 1)];
}

// Residual r = A(UU') - b into r_out (edge order), the trace entry aside.
__device__ __forceinline__ void p_map_r(Ctx& c, const Params& P, const double* U, int s,
                                        double* r_out) {
  double dummy[2] = {0.0, 0.0};
  map_pass<0>(c, P, U, s, kMapROut, nullptr, r_out, nullptr, dummy);
}

// ---------------------------------------------------------------- al_value --
// al_value (algo.cpp:47-56, sdp_instance.cpp:50-60) of U (visible), p, beta;
// r written to r_scr.  Leaves cs (theta) in dst_cs.
__device__ __noinline__ bool p_al_value(Ctx& c, const Params& P, const PView& v, const double* U,
                                        double beta, double* r_scr, double* dst_cs, double* val) {
  const DevPairs& I = P.I;
  const double pt = c.p_trace;
  p_map_r(c, P, U, v.s, r_scr);
  Jobs J;
  jobs_stats(J, v);
  par_jobs(c, J, [&](int j, int64_t i) { return term_stats(v, U, j, i); });
  const double sq = c.rs.out[0];
  if (threadIdx.x < (unsigned)v.s) dst_cs[threadIdx.x] = c.rs.out[1 + threadIdx.x];
  __syncthreads();
  const double rt = sq - I.b_trace;
  Jobs K;
  K.add(v.n * v.s, kPmEigen);  // <CU, U>
  K.add(v.m, kPmEigen);        // p.r
  K.add(v.m, kPmEigen);        // r.r
  par_jobs(c, K, [&](int j, int64_t i) -> double {
    if (j == 0) {
      const double u = U[v.cm(i)];
      return v.theta ? (-1.0 * dst_cs[i / v.n]) * u : (0.5 * u) * u;
    }
    const double r = i < v.np ? r_scr[i] : rt;
    if (j == 1) return (i < v.np ? P.p_up[i] : pt) * r;
    return r * r;
  });
  const double v_ = c.rs.out[0] + c.rs.out[1] + 0.5 * beta * c.rs.out[2];
  __syncthreads();
  if (!isfinite(v_)) {
    fail(c, kErrNumerical, kMsgAlValue);
    return false;
  }
  *val = v_;
  return true;
}

// -------------------------------------------------------------- ADAP-FISTA --
// fista (algo.cpp:124-201) on psi(u) = lambda g(u) + 0.5||u - W||^2 from
// x0 = W (prox_objective, algo.cpp:212-230).  Buffers: R.x, R.y, R.xt, R.gt,
// R.yn, R.v, h = buf[11].  Scratch m-vectors: r_up (r at x~), r_lo (r at y+).
struct PFista {
  int status;  // 0 success, 1 failure, 2 iteration limit
  double L, psi_y, dist0;
  int iters;
};

// cfg.trace >= 2: one debug event per fista() call (kind 9), matching the
// checker's ORC_DEBUG_FISTA record (algo.cpp dbg_fista).
__device__ __forceinline__ void p_dbg_fista(const Params& P, Ctx& c, double L0, const PFista& o,
                                            int cap) {
  if (P.cfg.trace < 2) return;
  TraceEv ev{};
  ev.kind = 9;
  ev.eps_inner = L0;
  ev.rank = o.status;
  ev.outer_iter = o.iters;
  ev.gap = o.L;
  ev.theta = o.status == 2 ? 0.0 : o.psi_y;
  ev.fw_alpha = cap;
  emit_trace(P, c, ev);
}

__device__ __noinline__ bool p_fista(Ctx& c, const Params& P, const PView& v, Roles& R,
                                     double lambda, double L0, PFista& out) {
  const DevPairs& I = P.I;
  const Cfg& cf = P.cfg;
  const int s = v.s;
  const double mu = cf.fista_mu, chi = cf.fista_chi, sigma = cf.fista_sigma;
  const double beta = c.beta, pt = c.p_trace;
  const bool theta = v.theta;
  double* const csx = c.cs;          // column sums of x~
  double* const csy = c.cs + kSMax;  // column sums of y+
  double* const H = P.buf[11];
  double* const rx = P.r_up;
  double* const ry = P.r_lo;
  double A = 0.0, tau = 1.0, L = L0;
  {
    const double* W = P.buf[R.wp];
    double* X = P.buf[R.x];
    double* Y = P.buf[R.y];
    for (int64_t o = c.rl * s + threadIdx.x; o < c.rh * s; o += kThreads) {
      X[o] = W[o];
      Y[o] = W[o];
    }
    __syncthreads();  // x~ below reads them with the same element map, but keep the CTA ordered
  }
  for (int it = 0;; ++it) {
    const int cap = cf.fista_max_iters > 0
                        ? cf.fista_max_iters
                        : 50 + (int)(10.0 * sqrt(L / mu) * log2(4.0 + L / L0));
    if (it >= cap) {
      out.status = 2;
      out.L = L;
      out.iters = it;
      p_dbg_fista(P, c, L0, out, cap);
      return true;
    }
    double a, psi_t, psi_n, dsq, dist0, sq_y;
    const double* W = P.buf[R.wp];
    double* XT = P.buf[R.xt];
    double* GT = P.buf[R.gt];
    double* YN = P.buf[R.yn];
    for (;;) {
      a = fista_a(tau, A, L, mu);
      {
        const double* X = P.buf[R.x];
        const double* Y = P.buf[R.y];
        for (int64_t o = c.rl * s + threadIdx.x; o < c.rh * s; o += kThreads)
          XT[o] = (A * Y[o] + a * X[o]) / (A + a);
      }
      c.t.sync();
      // psi.eval(x~): AlFunction::value_and_gradient (algo.cpp:102-113) + prox terms
      double dd;
      {
        Jobs J;
        jobs_stats(J, v);
        J.add(v.n * s, kPmEigen);  // ||x~ - W||^2 (sqnorm(d), algo.cpp:225)
        par_jobs(c, J, [&](int j, int64_t i) -> double {
          if (j <= s) return term_stats(v, XT, j, i);
          const int64_t o = v.cm(i);
          const double d = XT[o] - W[o];
          return d * d;
        });
        if (threadIdx.x < (unsigned)s) csx[threadIdx.x] = c.rs.out[1 + threadIdx.x];
        dd = c.rs.out[1 + s];
        const double sqx = c.rs.out[0];
        __syncthreads();
        const double rt = sqx - I.b_trace;
        const double qt = pt + beta * rt;
        p_map_r(c, P, XT, s, rx);
        double sums[3] = {0.0, 0.0, 0.0};
        auto epi = [&](int64_t row, int cc, double h, double xo) {
          const int64_t o = row * s + cc;
          H[o] = h;
          GT[o] = lambda * (2.0 * h) + (xo - W[o]);
        };
        row_pass<0, false>(c, P, XT, s, P.p_up, P.p_lo, beta, theta ? qt : 0.5,
                           theta ? csx : nullptr, false, sums, epi);
        c.t.sync();
        Jobs K;
        K.add(v.m, kPmEigen);      // q.(r + b)
        K.add(v.n * s, kPmEigen);  // <h, U>
        K.add(v.m, kPmEigen);      // p.r
        K.add(v.m, kPmEigen);      // r.r
        K.add(v.n * s, kPmEigen);  // ||z||^2, z = x~ - g~/L (project_ball)
        par_jobs(c, K, [&](int j, int64_t i) -> double {
          if (j == 1) {
            const int64_t o = v.cm(i);
            return H[o] * XT[o];
          }
          if (j == 4) {
            const int64_t o = v.cm(i);
            const double z = XT[o] - GT[o] / L;
            return z * z;
          }
          const bool tr = i >= v.np;
          const double r = tr ? rt : rx[i];
          const double pk = tr ? pt : P.p_up[i];
          if (j == 0) {
            const double bk = tr ? I.b_trace : (I.b_up ? I.b_up[i] : 0.0);
            const double q = pk + beta * r;
            return q * (r + bk);
          }
          if (j == 2) return pk * r;
          return r * r;
        });
        const double cdot = c.rs.out[1] - c.rs.out[0];
        const double val = cdot + c.rs.out[2] + 0.5 * beta * c.rs.out[3];
        const double zz = c.rs.out[4];
        __syncthreads();
        if (!isfinite(val)) {
          fail(c, kErrNumerical, kMsgAlValGrad);
          return false;
        }
        psi_t = lambda * val + 0.5 * dd;
        // y+ = project_ball(z) (algo.cpp:90-97)
        if (!isfinite(zz)) {
          fail(c, kErrInput, kMsgProjectBall);
          return false;
        }
        const double nrm = sqrt(zz);
        const bool scale = !(nrm <= 1.0);
        for (int64_t o = c.rl * s + threadIdx.x; o < c.rh * s; o += kThreads) {
          const double z = XT[o] - GT[o] / L;
          YN[o] = scale ? z / nrm : z;
        }
        c.t.sync();
      }
      // psi.value(y+) = lambda al_value(y+) + 0.5||y+ - W||^2; dsq; <g~, y+ - x~>
      {
        p_map_r(c, P, YN, s, ry);
        Jobs J;
        jobs_stats(J, v);
        J.add(v.n * s, kPmEigen);  // ||y+ - W||^2
        J.add(v.n * s, kPmEigen);  // ||y+ - x~||^2
        J.add(v.n * s, kPmEigen);  // <g~, y+ - x~>
        par_jobs(c, J, [&](int j, int64_t i) -> double {
          if (j <= s) return term_stats(v, YN, j, i);
          const int64_t o = v.cm(i);
          if (j == s + 1) {
            const double d = YN[o] - W[o];
            return d * d;
          }
          const double d = YN[o] - XT[o];
          return j == s + 2 ? d * d : GT[o] * d;
        });
        sq_y = c.rs.out[0];
        if (threadIdx.x < (unsigned)s) csy[threadIdx.x] = c.rs.out[1 + threadIdx.x];
        dist0 = c.rs.out[s + 1];
        dsq = c.rs.out[s + 2];
        const double lin_s = c.rs.out[s + 3];
        __syncthreads();
        const double rt = sq_y - I.b_trace;
        Jobs K;
        K.add(v.n * s, kPmEigen);  // <CU, U>
        K.add(v.m, kPmEigen);      // p.r
        K.add(v.m, kPmEigen);      // r.r
        par_jobs(c, K, [&](int j, int64_t i) -> double {
          if (j == 0) {
            const double u = YN[v.cm(i)];
            return theta ? (-1.0 * csy[i / v.n]) * u : (0.5 * u) * u;
          }
          const bool tr = i >= v.np;
          const double r = tr ? rt : ry[i];
          if (j == 1) return (tr ? pt : P.p_up[i]) * r;
          return r * r;
        });
        const double val = c.rs.out[0] + c.rs.out[1] + 0.5 * beta * c.rs.out[2];
        __syncthreads();
        if (!isfinite(val)) {
          fail(c, kErrNumerical, kMsgAlValue);
          return false;
        }
        psi_n = lambda * val + 0.5 * dist0;
        const double lin = psi_t + lin_s;
        const double noise = 1e-14 * (fabs(psi_n) + fabs(psi_t) + 1.0);
        if (lin + (1.0 - chi) * L / 4.0 * dsq >= psi_n - noise) break;
      }
      L *= 2.0;
      if (L > 1e18) {
        fail(c, kErrNumerical, kMsgFistaDiverged);
        return false;
      }
    }
    const double A_next = A + a;
    tau += a * mu;
    if (dist0 < chi * A_next * L * dsq) {
      out.status = 1;
      out.L = L;
      out.psi_y = psi_n;
      out.iters = it + 1;
      out.dist0 = dist0;
      p_dbg_fista(P, c, L0, out, -1);
      return true;
    }
    // gy = psi.gradient(y+); v = gy - g~ + L (x~ - y+); x update (algo.cpp:165-170)
    {
      double* X = P.buf[R.x];
      double* V = P.buf[R.v];
      const double qt = pt + beta * (sq_y - I.b_trace);
      double sums[3] = {0.0, 0.0, 0.0};
      auto epi = [&](int64_t row, int cc, double h, double yo) {
        const int64_t o = row * s + cc;
        const double gy = lambda * (2.0 * h) + (yo - W[o]);
        const double xt = XT[o];
        V[o] = gy - GT[o] + L * (xt - yo);
        const double sd = (L - mu) * (xt - yo);
        X[o] = (mu * a * yo + (tau - a * mu) * X[o] - a * sd) / tau;
      };
      row_pass<0, false>(c, P, YN, s, P.p_up, P.p_lo, beta, theta ? qt : 0.5,
                         theta ? csy : nullptr, false, sums, epi);
      c.t.sync();
      Jobs J;
      J.add(v.n * s, kPmEigen);
      par_jobs(c, J, [&](int, int64_t i) -> double {
        const double x = V[v.cm(i)];
        return x * x;
      });
      const double vv = c.rs.out[0];
      __syncthreads();
      if (!isfinite(vv)) {
        fail(c, kErrNumerical, kMsgAlGrad);
        return false;
      }
      if (sqrt(vv) <= sigma * sqrt(dist0)) {
        out.status = 0;
        out.L = L;
        out.psi_y = psi_n;
        out.iters = it + 1;
        out.dist0 = dist0;
        p_dbg_fista(P, c, L0, out, -1);
        return true;
      }
    }
    A = A_next;
    const int tmp = R.y;
    R.y = R.yn;
    R.yn = tmp;
  }
}

// ---------------------------------------------------------------- ADAP-AIPP --
// aipp (algo.cpp:233-300) from buffers[R.yt].
__device__ __noinline__ bool p_aipp(Ctx& c, const Params& P, const PView& v, Roles& R, double rho,
                                    AippOut& out) {
  const Cfg& cf = P.cfg;
  const int s = v.s;
  double lambda = cf.aipp_lambda0, M_bar = 1.0;
  {
    const double* Y = P.buf[R.yt];
    double* W = P.buf[R.wp];
    for (int64_t o = c.rl * s + threadIdx.x; o < c.rh * s; o += kThreads) W[o] = Y[o];
  }
  c.t.sync();
  double g_prev;
  if (!p_al_value(c, P, v, P.buf[R.wp], c.beta, P.r_up, c.cs, &g_prev)) return false;
  out.w_buf = R.yt;
  out.R_norm = INFINITY;
  out.g_value = g_prev;
  out.lambda = lambda;
  out.prox_iters = 0;
  out.fista_iters = 0;
  bool have_best = false;
  for (int j = 1; j <= cf.aipp_max_outer; ++j) {
    double L_out = 0.0, g_W = 0.0, Rn2 = 0.0;
    for (;;) {
      if (lambda < cf.aipp_lambda_underflow * cf.aipp_lambda0) {
        out.status = 2;
        if (have_best) out.w_buf = R.best;
        return true;
      }
      PFista fo;
      if (!p_fista(c, P, v, R, lambda, fmax(1.0, M_bar / 2.0), fo)) return false;
      out.fista_iters += fo.iters;
      if (fo.status == 0) {
        const double step_sq = fo.dist0;  // sqdist(res.y, Wp): the same sum as dist0
        g_W = (fo.psi_y - 0.5 * step_sq) / lambda;
        const double descent = lambda * g_prev - (lambda * g_W + 0.5 * step_sq);
        const double* V = P.buf[R.v];
        const double* Wp = P.buf[R.wp];
        const double* Yn = P.buf[R.yn];
        Jobs J;
        J.add(v.n * s, kPmEigen);  // <v, W_prev - y>
        J.add(v.n * s, kPmEigen);  // ||(v + W_prev - y)/lambda||^2
        par_jobs(c, J, [&](int j2, int64_t i) -> double {
          const int64_t o = v.cm(i);
          if (j2 == 0) return V[o] * (Wp[o] - Yn[o]);
          const double r = (V[o] + Wp[o] - Yn[o]) / lambda;
          return r * r;
        });
        const double vw = c.rs.out[0], rn2 = c.rs.out[1];
        __syncthreads();
        if (descent >= vw) {
          L_out = fo.L;
          Rn2 = rn2;
          break;
        }
      }
      lambda /= 2.0;
    }
    M_bar = L_out;
    const double R_norm = sqrt(Rn2);
    ++out.prox_iters;
    if (R_norm <= rho) {
      out.status = 0;
      out.w_buf = R.yn;
      out.R_norm = R_norm;
      out.g_value = g_W;
      out.lambda = lambda;
      return true;
    }
    if (R_norm < out.R_norm) {
      const double* src = P.buf[R.yn];
      double* dst = P.buf[R.best];
      for (int64_t o = c.rl * s + threadIdx.x; o < c.rh * s; o += kThreads) dst[o] = src[o];
      have_best = true;
      out.w_buf = R.best;
      out.R_norm = R_norm;
      out.g_value = g_W;
      out.lambda = lambda;
    }
    const int tmp = R.wp;
    R.wp = R.yn;
    R.yn = tmp;
    g_prev = g_W;
    __syncthreads();
  }
  out.status = 1;
  return true;
}

// ------------------------------------------------------------------ Lanczos --
// min_eigenpair (algo.cpp:339-455) of op = C + A*(q) with q fixed (GOp), B = -op.
struct PLz {
  const Params* P;
  int64_t n;
  unsigned long long used = 0ull;
  __device__ int alloc() {
    for (int sl = 0; sl < P->nslot; ++sl)
      if (!((used >> sl) & 1ull)) {
        used |= 1ull << sl;
        return sl;
      }
    return -1;
  }
  __device__ void release(int sl) {
    if (sl >= 0) used &= ~(1ull << sl);
  }
};

// w = applyB(x) = -(C x + A*(q) x), x visible; theta needs sum(x) first.
__device__ __noinline__ void p_applyB(Ctx& c, const Params& P, const GOp& g, const double* x,
                                      double* w) {
  const DevPairs& I = P.I;
  double csum = 0.0;
  if (is_theta(I)) {
    Jobs J;
    J.add(I.n, kPmEigen);  // column_sums of the n x 1 factor (offset 0)
    par_jobs(c, J, [&](int, int64_t i) { return x[i]; });
    csum = c.rs.out[0];
    __syncthreads();
  }
  double sums[3] = {0.0, 0.0, 0.0};
  auto epi = [&](int64_t a, int, double h, double) { w[a] = -h; };
  row_pass<1, true>(c, P, x, 1, g.qup, g.qlo, 0.0, theta_alpha_or_half(I, g.qt),
                    is_theta(I) ? &csum : nullptr, false, sums, epi);
  c.t.sync();
}

// cgs2 (algo.cpp:311-335): ordered dots h = V'w, w -= V h, twice; h += h2.
__device__ __noinline__ void p_cgs2(Ctx& c, const Params& P, int k, double* w, double* hh,
                                    double* hh2) {
  for (int pass = 0; pass < 2; ++pass) {
    double* h = pass == 0 ? hh : hh2;
    Jobs J;
    for (int t = 0; t < k; ++t) J.add(P.I.n, kPmSeq);
    par_jobs(c, J, [&](int t, int64_t i) { return slot_ptr(P, c.col[t])[i] * w[i]; });
    if (threadIdx.x < (unsigned)k) h[threadIdx.x] = c.rs.out[threadIdx.x];
    __syncthreads();
    for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads)
      w[a] = w[a] - lz_row_dot(c, P, k, a, h);
    c.t.sync();
  }
  if (threadIdx.x < (unsigned)k) hh[threadIdx.x] = hh[threadIdx.x] + hh2[threadIdx.x];
  __syncthreads();
}

__device__ __forceinline__ double p_norm(Ctx& c, int64_t n, const double* x) {
  Jobs J;
  J.add(n, kPmEigen);
  par_jobs(c, J, [&](int, int64_t i) { return x[i] * x[i]; });
  const double r = sqrt(c.rs.out[0]);
  __syncthreads();
  return r;
}

__device__ __noinline__ bool p_lanczos(Ctx& c, const Params& P, const GOp& g, double tol,
                                       int max_iters, int block_restart, LzOut& best) {
  const int64_t n = P.I.n;
  const int kmax = (int)min((int64_t)block_restart, n);
  const int keep = max(1, kmax / 3);
  PLz S{&P, n};
  double* hh = c.hh;
  double* hh2 = c.hh2;
  const int wsl = S.alloc(), fsl = S.alloc();
  double* w = slot_ptr(P, wsl);
  int refill = 0;
  {
    const double nv = p_norm(c, n, P.lz_rand);
    const int s0 = S.alloc();
    if (threadIdx.x == 0) c.col[0] = s0;
    double* v0 = slot_ptr(P, s0);
    for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) v0[a] = P.lz_rand[a] / nv;
    c.t.sync();
  }
  for (int idx = threadIdx.x; idx < kHLd * kHLd; idx += kThreads) c.H[idx] = 0.0;
  __syncthreads();
  int matvecs = 0, basis = 1, filled = 0;
  double beta = 0.0;
  best = LzOut();
  best.residual = INFINITY;
  best.matvecs = 0;
  for (;;) {
    bool breakdown = false;
    while (filled < basis && matvecs < max_iters) {
      const int j = filled;
      p_applyB(c, P, g, slot_ptr(P, c.col[j]), w);
      ++matvecs;
      p_cgs2(c, P, basis, w, hh, hh2);
      if (threadIdx.x < (unsigned)basis) {
        c.H[threadIdx.x + j * kHLd] = hh[threadIdx.x];
        c.H[j + threadIdx.x * kHLd] = hh[threadIdx.x];
      }
      __syncthreads();
      ++filled;
      beta = p_norm(c, n, w);
      double hmax = 0.0;
      for (int t = 0; t < basis; ++t) hmax = fmax(hmax, fabs(hh[t]));
      if (beta <= 1e-13 * fmax(1.0, hmax)) {
        breakdown = true;
        break;
      }
      if (basis < kmax) {
        const int sl = S.alloc();
        double* vb = slot_ptr(P, sl);
        for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) vb[a] = w[a] / beta;
        if (threadIdx.x == 0) {
          c.col[basis] = sl;
          c.H[basis + j * kHLd] = beta;
          c.H[j + basis * kHLd] = beta;
        }
        c.t.sync();
        ++basis;
      }
    }
    const int f = filled;
    jacobi_dev(c, c.H, kHLd, f, true);
    const int top = f - 1;
    const double mu = c.ev[top];
    const double res_est = breakdown ? 0.0 : beta * fabs(c.E[(f - 1) + top * f]);
    const bool budget_left = matvecs + 1 < max_iters;
    if (res_est <= tol * fmax(1.0, fabs(mu)) || !budget_left || (breakdown && filled >= n)) {
      // measure(ritz(top)) (algo.cpp:364-380)
      const int xs = S.alloc(), bs = S.alloc();
      double* x = slot_ptr(P, xs);
      double* Bx = slot_ptr(P, bs);
      for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads)
        x[a] = lz_row_dot(c, P, f, a, c.E + top * f);
      c.t.sync();
      const double nx = p_norm(c, n, x);
      for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) x[a] = x[a] / nx;
      c.t.sync();
      p_applyB(c, P, g, x, Bx);
      ++matvecs;
      Jobs J;
      J.add(n, kPmEigen);
      par_jobs(c, J, [&](int, int64_t i) { return x[i] * Bx[i]; });
      const double mux = c.rs.out[0];
      __syncthreads();
      Jobs K;
      K.add(n, kPmEigen);
      par_jobs(c, K, [&](int, int64_t i) {
        const double d = Bx[i] - mux * x[i];
        return d * d;
      });
      const double res = sqrt(c.rs.out[0]);
      __syncthreads();
      S.release(bs);
      LzOut o;
      o.lambda = -mux;
      o.residual = res;
      o.matvecs = matvecs;
      o.converged = o.residual <= tol * fmax(1.0, fabs(o.lambda));
      o.vslot = xs;
      if (o.residual < best.residual) {
        S.release(best.vslot);
        best = o;
      } else {
        S.release(xs);
      }
      if (best.converged || matvecs >= max_iters || (breakdown && filled >= n)) return true;
    }
    // thick restart (algo.cpp:436-453)
    const int l = min(keep, f - 1 > 0 ? f - 1 : 1);
    int newcol[kLanczosMax];
    for (int t = 0; t < l; ++t) newcol[t] = S.alloc();
    if (newcol[l - 1] < 0) {
      fail(c, kErrCapacity, kMsgRefillCap);
      return false;
    }
    for (int t = 0; t < l; ++t) {
      double* d = slot_ptr(P, newcol[t]);
      for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads)
        d[a] = lz_row_dot(c, P, f, a, c.E + (f - 1 - t) * f);
    }
    for (int t = 0; t < basis; ++t) S.release(c.col[t]);
    for (int idx = threadIdx.x; idx < kHLd * kHLd; idx += kThreads) c.H[idx] = 0.0;
    __syncthreads();
    if (threadIdx.x < (unsigned)l) {
      c.H[threadIdx.x + threadIdx.x * kHLd] = c.ev[f - 1 - threadIdx.x];
      c.col[threadIdx.x] = newcol[threadIdx.x];
    }
    __syncthreads();
    c.t.sync();
    const int sl = S.alloc();
    double* vl = slot_ptr(P, sl);
    if (breakdown) {
      ++refill;
      double* fr = slot_ptr(P, fsl);
      const double* rnd = lz_refill(c, P, refill);
      if (!rnd) {
        fail(c, kErrCapacity, kMsgRefillCap);
        return false;
      }
      for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) fr[a] = __ldcv(rnd + a);
      c.t.sync();
      p_cgs2(c, P, l, fr, hh, hh2);
      const double fn = p_norm(c, n, fr);
      if (fn <= 1e-13) return true;
      for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) vl[a] = fr[a] / fn;
    } else {
      for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) vl[a] = w[a] / beta;
    }
    if (threadIdx.x == 0) c.col[l] = sl;
    c.t.sync();
    basis = l + 1;
    filled = l;
  }
}

// ---------------------------------------------------------------------- HLR --
// hlr_solve (algo.cpp:511-591) from buffers[R.yt] (rank s).  On exit r_up /
// r_lo hold the residual of the last GradientOperator and out.rt its trace
// entry; out.pr / out.rr are p.r and r.r in the reference's order.
__device__ __noinline__ bool p_hlr(Ctx& c, const Params& P, Roles& R, int s, double beta,
                                   double eps_t, int outer_iter, unsigned long long deadline_ns,
                                   HlrOut& out) {
  const DevPairs& I = P.I;
  const Cfg& cf = P.cfg;
  out = HlrOut();
  for (int step = 0;; ++step) {
    PView v{I.n, I.np, I.m, s, is_theta(I)};
    AippOut ao;
    if (!p_aipp(c, P, v, R, eps_t, ao)) return false;
    out.aipp_iters += ao.prox_iters;
    out.fista_iters += ao.fista_iters;
    const int ybuf = ao.w_buf;
    const double* Y = P.buf[ybuf];
    c.t.sync();
    // GradientOperator(Y) (algo.cpp:71-78)
    double* const csY = c.cs;
    Jobs J;
    jobs_stats(J, v);
    par_jobs(c, J, [&](int j, int64_t i) { return term_stats(v, Y, j, i); });
    const double sqY = c.rs.out[0];
    if (threadIdx.x < (unsigned)s) csY[threadIdx.x] = c.rs.out[1 + threadIdx.x];
    __syncthreads();
    const double rt = sqY - I.b_trace;
    const double qt = c.p_trace + beta * rt;
    {
      double sums[2] = {0.0, 0.0};
      bool bad = false;
      gradop_pass<0>(c, P, Y, s, beta, sums, &bad);
      double fl[1] = {bad ? 1.0 : 0.0};
      team_sum<1>(c.t, c.rs, fl);
      if (fl[0] != 0.0 || (is_theta(I) && !isfinite(qt))) {
        fail(c, kErrNumerical, kMsgGradOp);
        return false;
      }
    }
    const GOp g{P.q_up, P.q_lo, qt};
    LzOut lz;
    if (!p_lanczos(c, P, g, 0.1 * eps_t, cf.eig_max_iters, cf.eig_block_restart, lz)) return false;
    out.eig_products += lz.matvecs;
    const double theta = lz.lambda < 0 ? -lz.lambda : 0.0;
    // fw_gap (algo.cpp:459-461): <G Y, Y> + theta
    double gap;
    {
      double* Hm = P.buf[11];
      double sums[3] = {0.0, 0.0, 0.0};
      auto epi = [&](int64_t a, int cc, double h, double) { Hm[a * s + cc] = h; };
      row_pass<0, true>(c, P, Y, s, g.qup, g.qlo, 0.0, theta_alpha_or_half(I, qt),
                        is_theta(I) ? csY : nullptr, false, sums, epi);
      c.t.sync();
      Jobs K;
      K.add(v.n * s, kPmEigen);
      par_jobs(c, K, [&](int, int64_t i) {
        const int64_t o = v.cm(i);
        return Hm[o] * Y[o];
      });
      gap = c.rs.out[0] + theta;
      __syncthreads();
    }
    {
      TraceEv ev{};
      ev.kind = 0;
      ev.outer_iter = outer_iter;
      ev.beta = beta;
      ev.eps_inner = eps_t;
      ev.gap = gap;
      ev.theta = theta;
      ev.rank = s;
      ev.al_value = ao.g_value;
      emit_trace(P, c, ev);
    }
    const bool done = gap <= eps_t;
    const bool no_steps = step >= cf.max_fw_steps;
    const bool no_time = team_now(c) >= (double)deadline_ns;
    if (done || no_steps || no_time || !lz.converged) {
      Jobs K;
      K.add(v.m, kPmEigen);  // p.r
      K.add(v.m, kPmEigen);  // r.r
      par_jobs(c, K, [&](int j, int64_t i) -> double {
        const bool tr = i >= v.np;
        const double r = tr ? rt : P.r_up[i];
        return j == 0 ? (tr ? c.p_trace : P.p_up[i]) * r : r * r;
      });
      out.pr = c.rs.out[0];
      out.rr = c.rs.out[1];
      __syncthreads();
      out.y_buf = ybuf;
      out.s = s;
      out.theta = theta;
      out.gap = gap;
      out.lambda_min = lz.lambda;
      out.al_val = ao.g_value;
      out.rt = rt;
      out.cdot = ao.g_value - out.pr - 0.5 * beta * out.rr;
      out.eig_trusted = lz.converged;
      out.status = done ? 0 : (no_time ? 2 : 1);
      if (!lz.converged && !done) out.status = 1;
      return true;
    }
    // fw_stepsize (algo.cpp:480-494): numer = the same fw_gap of the rebuilt G
    const double* yv = theta > 0 ? slot_ptr(P, lz.vslot) : nullptr;
    double denom;
    {
      double sqy = 0.0;  // A(yy')_{m-1} = sqnorm(y) (theta trace constraint)
      if (yv && v.theta) {
        Jobs Q;
        Q.add(v.n, kPmEigen);
        par_jobs(c, Q, [&](int, int64_t i) { return yv[i] * yv[i]; });
        sqy = c.rs.out[0];
        __syncthreads();
      }
      Jobs K;
      K.add(v.m, kPmEigen);
      par_jobs(c, K, [&](int, int64_t i) -> double {
        double my, rb;
        if (i < v.np) {
          const int64_t a = I.ei[i], b = I.ej[i];
          my = yv ? yv[a] * yv[b] : 0.0;
          rb = P.r_up[i] + (I.b_up ? I.b_up[i] : 0.0);
        } else {
          my = yv ? sqy : 0.0;
          rb = rt + I.b_trace;
        }
        const double d = rb - my;
        return d * d;
      });
      denom = beta * c.rs.out[0];
      __syncthreads();
    }
    const double numer = gap;
    double alpha;
    if (denom <= 1e-14)
      alpha = numer > 0 ? 1.0 : 0.0;
    else
      alpha = fmin(fmax(numer / denom, 0.0), 1.0);
    int s_new = s;
    if (theta > 0 && alpha != 1.0 && s + 1 > kSMax) {
      fail(c, kErrCapacity, kMsgRankCap);
      return false;
    }
    {
      double* dst = P.buf[R.tmp];
      rank_update_dev<0>(c, P, Y, s, yv, alpha, theta > 0, dst, &s_new);
      const int t = R.yt;
      R.yt = R.tmp;
      R.tmp = t;
    }
    s = s_new;
    ++out.fw_steps;
    if (cf.trace) {
      PView v2{I.n, I.np, I.m, s, is_theta(I)};
      double al;
      if (!p_al_value(c, P, v2, P.buf[R.yt], beta, P.r_lo, c.cs + kSMax, &al)) return false;
      TraceEv ev{};
      ev.kind = 1;
      ev.outer_iter = outer_iter;
      ev.beta = beta;
      ev.eps_inner = eps_t;
      ev.gap = gap;
      ev.theta = theta;
      ev.rank = s;
      ev.fw_alpha = alpha;
      ev.al_value = al;
      emit_trace(P, c, ev);
    }
  }
}

// -------------------------------------------------------- outer AL driver --
// check_termination (algo.cpp:617-639) with multiplier (p_up/p_lo, pt).
__device__ __noinline__ bool p_check_termination(Ctx& c, const Params& P, const PView& v,
                                                 const double* U, double pt, double theta,
                                                 double eig_tol, Term& t) {
  const DevPairs& I = P.I;
  const Cfg& cf = P.cfg;
  p_map_r(c, P, U, v.s, P.r_up);
  Jobs J;
  jobs_stats(J, v);
  par_jobs(c, J, [&](int j, int64_t i) { return term_stats(v, U, j, i); });
  const double sq = c.rs.out[0];
  double* const cs = c.cs;
  if (threadIdx.x < (unsigned)v.s) cs[threadIdx.x] = c.rs.out[1 + threadIdx.x];
  __syncthreads();
  const double rt = sq - I.b_trace;
  Jobs K;
  K.add(v.m, kPmEigen);        // r.r
  K.add(v.n * v.s, kPmEigen);  // <CU, U>
  K.add(v.m, kPmEigen);        // b.p
  par_jobs(c, K, [&](int j, int64_t i) -> double {
    if (j == 1) {
      const double u = U[v.cm(i)];
      return v.theta ? (-1.0 * cs[i / v.n]) * u : (0.5 * u) * u;
    }
    const bool tr = i >= v.np;
    if (j == 0) {
      const double r = tr ? rt : P.r_up[i];
      return r * r;
    }
    const double bk = tr ? I.b_trace : (I.b_up ? I.b_up[i] : 0.0);
    return bk * (tr ? pt : P.p_up[i]);
  });
  t.rel_pfeas = sqrt(c.rs.out[0]) / (1.0 + I.norm_b1);
  t.pval = c.rs.out[1];
  t.dval = -c.rs.out[2] - theta;
  __syncthreads();
  t.rel_gap = fabs(t.pval - t.dval) / (1.0 + fabs(t.pval) + fabs(t.dval));
  LzOut lz;
  const GOp g{P.p_up, P.p_lo, pt};
  if (!p_lanczos(c, P, g, eig_tol, cf.eig_max_iters, cf.eig_block_restart, lz)) return false;
  t.dual_lambda_min = lz.lambda;
  t.eig_products = lz.matvecs;
  t.eig_trusted = lz.converged;
  t.rel_dfeas = fmax(0.0, -t.dual_lambda_min) / (1.0 + I.norm_C1);
  t.done = t.eig_trusted && t.rel_pfeas <= cf.eps && t.rel_gap <= cf.eps && t.rel_dfeas <= cf.eps;
  return true;
}

// certify (algo.cpp:648-675)
__device__ __noinline__ bool p_certify(Ctx& c, const Params& P, const PView& v, const double* U,
                                       double pt, double theta, double eig_tol, Cert& ct) {
  const DevPairs& I = P.I;
  ct.pt = pt;
  ct.theta = theta;
  if (v.theta && theta > 0) {
    ct.pt = ct.pt + theta;
    ct.theta = 0.0;
  }
  if (!p_check_termination(c, P, v, U, ct.pt, ct.theta, eig_tol, ct.t)) return false;
  if (!ct.t.eig_trusted) return true;
  Term& t = ct.t;
  if (v.theta) {
    if (t.dual_lambda_min < 0) {
      ct.pt = ct.pt - t.dual_lambda_min;
      t.dval = t.dval + t.dual_lambda_min * I.b_trace;
      t.dual_lambda_min = 0.0;
      t.rel_dfeas = 0.0;
    }
  } else {
    const double tight = fmax(0.0, -t.dual_lambda_min);
    t.dval = t.dval + (ct.theta - tight);
    ct.theta = tight;
  }
  t.rel_gap = fabs(t.pval - t.dval) / (1.0 + fabs(t.pval) + fabs(t.dval));
  t.done = t.rel_pfeas <= P.cfg.eps && t.rel_gap <= P.cfg.eps && t.rel_dfeas <= P.cfg.eps;
  return true;
}

// b.p over all m constraints (dot(si.b, rep.p), algo.cpp:740/771)
__device__ __forceinline__ double p_bdotp(Ctx& c, const Params& P, const PView& v, double pt) {
  const DevPairs& I = P.I;
  Jobs J;
  J.add(v.m, kPmEigen);
  par_jobs(c, J, [&](int, int64_t i) -> double {
    if (i >= v.np) return I.b_trace * pt;
    return (I.b_up ? I.b_up[i] : 0.0) * P.p_up[i];
  });
  const double r = c.rs.out[0];
  __syncthreads();
  return r;
}

// solve_warm (algo.cpp:691-808) from buffers[0] (rank P.s_in), multiplier in
// p_up / p_lo / P.p_trace.
__device__ __noinline__ void p_solve(Ctx& c, const Params& P, SolveOut* so) {
  const DevPairs& I = P.I;
  const Cfg& cf = P.cfg;
  const double t0 = team_now(c);
  const double deadline = t0 + cf.time_limit * 1e9;
  const double nb1 = I.norm_b1, nb2 = I.nb2;
  const double eps_floor = cf.eps_floor > 0 ? cf.eps_floor : cf.eps * (1.0 + nb1) / 10.0;
  double eps_t = cf.eps0 > 0 ? cf.eps0 : 1e-2 * (1.0 + nb1);
  eps_t = fmax(eps_t, eps_floor);
  double beta = cf.beta0 > 0 ? cf.beta0 : 10.0 * fmax(1.0, nb2 > 0 ? 1.0 / nb2 : 1.0);
  const double eig_term_tol = fmin(cf.eig_tol, 1e-7);
  Roles R{0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10};
  int s = P.s_in;
  double theta = 0.0;
  c.p_trace = P.p_trace;
  SolveOut o{};
  bool have_cert = false;
  Cert fc;
  double prev_pfeas = INFINITY;
  int status = 1;
  bool nan_report = false;
  for (int t = 1; t <= cf.max_outer; ++t) {
    if (team_now(c) >= deadline) {
      status = 2;
      break;
    }
    {
      const double* src = P.buf[R.rep];
      double* dst = P.buf[R.yt];
      for (int64_t q = c.rl * s + threadIdx.x; q < c.rh * s; q += kThreads) dst[q] = src[q];
    }
    c.t.sync();
    c.beta = beta;
    HlrOut ho;
    if (!p_hlr(c, P, R, s, beta, eps_t, t, (unsigned long long)deadline, ho)) {
      if (c.status == kErrNumerical) {
        c.status = kOk;
        status = 3;
      }
      break;
    }
    o.outer_iters = t;
    o.fw_steps += ho.fw_steps;
    o.aipp_iters += ho.aipp_iters;
    o.fista_iters += ho.fista_iters;
    o.eig_products += ho.eig_products;
    {
      const int tb = R.rep;
      R.rep = ho.y_buf;
      if (R.yt == ho.y_buf) R.yt = tb;
      else if (R.wp == ho.y_buf) R.wp = tb;
      else if (R.best == ho.y_buf) R.best = tb;
      else if (R.x == ho.y_buf) R.x = tb;
      else if (R.y == ho.y_buf) R.y = tb;
      else if (R.xt == ho.y_buf) R.xt = tb;
      else if (R.gt == ho.y_buf) R.gt = tb;
      else if (R.yn == ho.y_buf) R.yn = tb;
      else if (R.v == ho.y_buf) R.v = tb;
      else if (R.tmp == ho.y_buf) R.tmp = tb;
      s = ho.s;
    }
    // rep.p += beta * residual (algo.cpp:763); finiteness of U and p
    double bad = 0.0;
    {
      for (int64_t k = c.kl + threadIdx.x; k < c.kh; k += kThreads) {
        const double pn = P.p_up[k] + beta * P.r_up[k];
        P.p_up[k] = pn;
        if (!isfinite(pn)) bad = 1.0;
      }
      const int64_t lo0 = I.lo_ptr[c.rl], lo_n = I.lo_ptr[c.rh] - lo0;
      for (int64_t e = threadIdx.x; e < lo_n; e += kThreads)
        P.p_lo[lo0 + e] = P.p_lo[lo0 + e] + beta * P.r_lo[lo0 + e];
      const double* U = P.buf[R.rep];
      for (int64_t q = c.rl * s + threadIdx.x; q < c.rh * s; q += kThreads)
        if (!isfinite(U[q])) bad = 1.0;
      double v[1] = {bad};
      team_sum<1>(c.t, c.rs, v);
      bad = v[0];
    }
    c.p_trace = c.p_trace + beta * ho.rt;
    theta = ho.theta;
    if (is_theta(I) && !isfinite(c.p_trace)) bad = 1.0;
    if (bad != 0.0) {
      c.msg = kMsgNonFinite;
      status = 3;
      nan_report = true;
      break;
    }
    const PView v{I.n, I.np, I.m, s, is_theta(I)};
    const double rel_pfeas = sqrt(ho.rr) / (1.0 + nb1);
    const double pval = ho.cdot;
    const double dval = -p_bdotp(c, P, v, c.p_trace) - ho.theta;
    const double rel_gap = fabs(pval - dval) / (1.0 + fabs(pval) + fabs(dval));
    const double lam = is_theta(I) ? ho.lambda_min + ho.theta : ho.lambda_min;
    const double rel_dfeas_est = fmax(0.0, -lam) / (1.0 + I.norm_C1);
    {
      TraceEv ev{};
      ev.kind = 2;
      ev.outer_iter = t;
      ev.beta = beta;
      ev.eps_inner = eps_t;
      ev.gap = ho.gap;
      ev.theta = ho.theta;
      ev.rank = s;
      ev.al_value = ho.al_val;
      ev.rel_pfeas = rel_pfeas;
      ev.rel_gap = rel_gap;
      ev.rel_dfeas = rel_dfeas_est;
      emit_trace(P, c, ev);
    }
    if (ho.eig_trusted && rel_pfeas <= cf.eps && rel_gap <= cf.eps && rel_dfeas_est <= cf.eps) {
      Cert ct;
      if (!p_certify(c, P, v, P.buf[R.rep], c.p_trace, theta, eig_term_tol, ct)) break;
      o.eig_products += ct.t.eig_products;
      if (ct.t.done) {
        fc = ct;
        have_cert = true;
        status = 0;
        break;
      }
    }
    if (rel_pfeas > 0.9 * prev_pfeas) beta *= cf.beta_growth;
    prev_pfeas = rel_pfeas;
    eps_t = fmax(eps_floor, eps_t * cf.eps_decay);
  }
  if (c.status != kOk) {
    if (c.t.rank == 0 && threadIdx.x == 0) {
      so->status = c.status;
      so->msg = c.msg;
    }
    return;
  }
  const PView v{I.n, I.np, I.m, s, is_theta(I)};
  if (!have_cert && !nan_report) {
    Cert ct;
    if (!p_certify(c, P, v, P.buf[R.rep], c.p_trace, theta, eig_term_tol, ct)) {
      if (c.t.rank == 0 && threadIdx.x == 0) {
        so->status = c.status;
        so->msg = c.msg;
      }
      return;
    }
    o.eig_products += ct.t.eig_products;
    fc = ct;
    have_cert = true;
  }
  o.out_buf = R.rep;
  o.rank = s;
  o.msg = c.msg;
  if (nan_report) {
    o.status = 3;
    o.pval = o.dval = o.dval_no_theta = NAN;
    o.rel_pfeas = o.rel_gap = o.rel_dfeas = NAN;
    o.theta = theta;
    o.p_trace = c.p_trace;
  } else {
    o.status = status;
    o.theta = fc.theta;
    o.p_trace = fc.pt;
    o.rel_pfeas = fc.t.rel_pfeas;
    o.rel_gap = fc.t.rel_gap;
    o.rel_dfeas = fc.t.rel_dfeas;
    o.pval = fc.t.pval;
    o.dval = fc.t.dval;
    o.dval_no_theta = -p_bdotp(c, P, v, fc.pt);
  }
  if (c.t.rank == 0 && threadIdx.x == 0) *so = o;
}

// Parity-mode entry points of the persistent kernel: the solve and the two
// sub-solver parity ops (Lanczos on G, AIPP).
__device__ __noinline__ void p_dispatch(Ctx& c, const Params& P, SolveOut* so) {
  const DevPairs& I = P.I;
  const int s = P.s_in;
  c.beta = P.beta_in;
  c.p_trace = P.p_trace;
  if (P.op == kOpSolve) {
    p_solve(c, P, so);
    return;
  }
  const PView v{I.n, I.np, I.m, s, is_theta(I)};
  if (P.op == kOpMinEigG) {
    const double* U = P.buf[0];
    c.t.sync();
    Jobs J;
    jobs_stats(J, v);
    par_jobs(c, J, [&](int j, int64_t i) { return term_stats(v, U, j, i); });
    const double qt = P.p_trace + P.beta_in * (c.rs.out[0] - I.b_trace);
    __syncthreads();
    double sums[2] = {0.0, 0.0};
    bool bad = false;
    gradop_pass<0>(c, P, U, s, P.beta_in, sums, &bad);
    double fl[1] = {bad ? 1.0 : 0.0};
    team_sum<1>(c.t, c.rs, fl);
    if (fl[0] != 0.0) {
      fail(c, kErrNumerical, kMsgGradOp);
    } else {
      const GOp g{P.q_up, P.q_lo, qt};
      LzOut lz;
      if (p_lanczos(c, P, g, P.rho_in, P.cfg.eig_max_iters, P.cfg.eig_block_restart, lz)) {
        if (lz.vslot >= 0) {
          const double* x = slot_ptr(P, lz.vslot);
          for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) P.out_vec[a] = x[a];
        }
        if (c.t.rank == 0 && threadIdx.x == 0) {
          P.scalars[0] = lz.lambda;
          P.scalars[1] = lz.residual;
          P.iscalars[0] = lz.matvecs;
          P.iscalars[1] = lz.converged ? 1 : 0;
        }
      }
    }
  } else if (P.op == kOpAipp) {
    Roles R{10, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9};
    AippOut ao;
    c.t.sync();
    if (p_aipp(c, P, v, R, P.rho_in, ao)) {
      const double* W = P.buf[ao.w_buf];
      for (int64_t q = c.rl * s + threadIdx.x; q < c.rh * s; q += kThreads) P.out_mat[q] = W[q];
      if (c.t.rank == 0 && threadIdx.x == 0) {
        P.scalars[0] = ao.R_norm;
        P.scalars[1] = ao.g_value;
        P.scalars[2] = ao.lambda;
        P.iscalars[0] = ao.status;
        P.iscalars[1] = ao.prox_iters;
        P.iscalars[2] = ao.fista_iters;
      }
    }
  }
  if (c.t.rank == 0 && threadIdx.x == 0) {
    so->status = c.status;
    so->msg = c.msg;
  }
}

}  // namespace hallar
