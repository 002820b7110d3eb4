// Device Lanczos (with the CTA-parallel Jacobi eigen-solver), HLR inner
// method, outer AL driver and certificate, and the op dispatcher of the
// persistent kernel.  Continues device.cuh.
#pragma once

#include "device.cuh"

namespace hallar {

#define HALLAR_DISPATCH_S(s, CALL)        \
  switch (s) {                            \
    case 1: { constexpr int S_ = 1; CALL; } break; \
    case 2: { constexpr int S_ = 2; CALL; } break; \
    case 3: { constexpr int S_ = 3; CALL; } break; \
    case 4: { constexpr int S_ = 4; CALL; } break; \
    default: { constexpr int S_ = 0; CALL; } break; \
  }

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Team-consistent clock: CTA 0's timer, broadcast through a reduction.
inline __device__ __noinline__ double team_now(Ctx& c) {
  double v[1] = {(c.t.rank == 0 && threadIdx.x == 0) ? (double)globaltimer_ns() : 0.0};
  team_sum<1>(c.t, c.rs, v);
  return v[0];
}

inline __device__ void emit_trace(const Params& P, Ctx& c, const TraceEv& ev) {
  if (!P.cfg.trace || c.t.rank != 0 || threadIdx.x != 0 || !P.trace) return;
  const int i = *P.trace_count;
  if (i < P.trace_cap) P.trace[i] = ev;
  *P.trace_count = i + 1;
}

// ---------------------------------------------------------------- Jacobi ---
// Same rotation schedule and formulas as oracle/src/base.cpp jacobi_eigh
// (threshold 2 ulp of the largest entry here, tighter in the checker):
// tournament rounds (circle method); per round every thread
// owns one (pair, row/column) item, computes its pair's rotation from the
// round-start snapshot, applies the row rotation, then the column rotation
// (and eigenvector update), zeroing the pivot — three barriers per round.
// Input H column-major with leading dim ldh; outputs ascending c.ev[0..k)
// and c.E (column-major, ld k), signs normalised.
inline __device__ __noinline__ void jacobi_dev(Ctx& c, const double* H, int ldh, int k, bool tight = false) {
  double* const A = c.JA;
  double* const V = c.JV;
  double* const red = c.rs.part;  // scratch [kWarps]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int idx = tid; idx < k * k; idx += kThreads) {
    const int i = idx % k, j = idx / k;
    A[idx] = H[i + j * ldh];
    V[idx] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  auto block_max = [&](double v) -> double {
    v = warp_max(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double m = red[0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) m = fmax(m, red[w]);
    __syncthreads();
    return m;
  };
  if (k > 1) {
    const int kp = k + (k & 1);
    const int half = kp / 2;
    // item = (pair t, index r): one per thread (kp/2 <= 16, k <= 32)
    const int t = tid / k, r = tid % k;
    const bool active = t < half;
    double mloc = 0.0;
    for (int idx = tid; idx < k * k; idx += kThreads) mloc = fmax(mloc, fabs(A[idx]));
    // 2 ulp of the largest entry: below this a pivot is rounding noise (a
    // tighter bound never triggers and costs ~3x more sweeps, measured)
    // parity mode (tight): the checker's threshold and pivot test (base.cpp jacobi_eigh)
    const double thresh = block_max(mloc) * (tight ? 1e-18 : 4e-16);
    for (int sweep = 0; sweep < 40; ++sweep) {
      double oloc = 0.0;
      for (int idx = tid; idx < k * k; idx += kThreads) {
        const int i = idx % k, j = idx / k;
        if (i < j) oloc = fmax(oloc, fabs(A[idx]));
      }
      const double off = block_max(oloc);
      if (off <= thresh) break;
      for (int round = 0; round < kp - 1; ++round) {
        int p = 0, q = 0;
        bool ok = false;
        double cc = 1.0, ss = 0.0;
        if (active) {
          const int pa = t == 0 ? 0 : 1 + (t - 1 + round) % (kp - 1);
          const int tb = kp - 1 - t;
          const int pb = 1 + (tb - 1 + round) % (kp - 1);
          p = min(pa, pb);
          q = max(pa, pb);
          ok = q < k;
          if (ok) {
            const double apq = A[p + q * k];
            if (tight ? apq != 0.0 : fabs(apq) > thresh) {
              const double th = (A[q + q * k] - A[p + p * k]) / (2.0 * apq);
              double tn;
              if (fabs(th) > 1e150)
                tn = 0.5 / th;
              else
                tn = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
              cc = 1.0 / sqrt(tn * tn + 1.0);
              ss = tn * cc;
            }
          }
        }
        const bool rot = ok && ss != 0.0;
        __syncthreads();
        if (rot) {  // rows p, q at column r
          const double ap = A[p + r * k], aq = A[q + r * k];
          A[p + r * k] = cc * ap - ss * aq;
          A[q + r * k] = ss * ap + cc * aq;
        }
        __syncthreads();
        if (rot) {  // columns p, q at row r, eigenvectors, pivot zeroed
          const double ap = A[r + p * k], aq = A[r + q * k];
          A[r + p * k] = (r == q) ? 0.0 : cc * ap - ss * aq;
          A[r + q * k] = (r == p) ? 0.0 : ss * ap + cc * aq;
          const double vp = V[r + p * k], vq = V[r + q * k];
          V[r + p * k] = cc * vp - ss * vq;
          V[r + q * k] = ss * vp + cc * vq;
        }
        __syncthreads();
      }
    }
  }
  // stable ascending ranks; sign: largest-|.| (first on ties) positive
  if (tid < k) {
    const double d = A[tid + tid * k];
    int rk = 0;
    for (int j = 0; j < k; ++j) {
      const double dj = A[j + j * k];
      if (dj < d || (dj == d && j < tid)) ++rk;
    }
    int imax = 0;
    double best = -1.0;
    for (int i = 0; i < k; ++i)
      if (fabs(V[i + tid * k]) > best) {
        best = fabs(V[i + tid * k]);
        imax = i;
      }
    const double sg = V[imax + tid * k] < 0.0 ? -1.0 : 1.0;
    c.ev[rk] = d;
    for (int i = 0; i < k; ++i) c.E[i + rk * k] = sg * V[i + tid * k];
  }
  __syncthreads();
}

// --------------------------------------------------------------- Lanczos ---
struct GOp {
  const double* qup;
  const double* qlo;
  double qt;
};
struct LzOut {
  double lambda = 0.0, residual = INFINITY;
  int matvecs = 0;
  bool converged = false;
  int vslot = -1;
};

__device__ __forceinline__ double* slot_ptr(const Params& P, int sl) {
  return P.vslot + (size_t)sl * P.I.n;
}

// A Lanczos vector that exists only as (src / scale): materialised into its
// slot by the matvec that consumes it, so normalisation costs no barrier.
struct Pending {
  const double* src;
  double scale;
  double sum;  // column sum of src / scale (theta C-term)
  int dst;     // slot receiving src / scale (-1: none)
};

// out = -(C v + A*(q) v) with v = pend.src / pend.scale gathered on the fly
// (apply_B, lanczos.cpp:38); also writes v into slot pend.dst for own rows.
// The caller has team-synchronised after pend.src was written.
__device__ __forceinline__ void lz_apply(Ctx& c, const Params& P, const GOp& g, const Pending& pv,
                                         double* out) {
  const DevPairs& I = P.I;
  double* vdst = pv.dst >= 0 ? slot_ptr(P, pv.dst) : nullptr;
  auto epi = [&](int64_t a, int, double h, double va) {
    out[a] = -h;
    if (vdst) vdst[a] = va;
  };
  double sums[3] = {0.0, 0.0, 0.0};
  const double sumv = pv.sum;
  if (is_pr(I)) {
    const UScaled v{pv.src, pv.scale};
    pr_forward(P, c.t.rank, c.t.size, c.X, v, 1);
    c.t.sync();
    pr_inverse<true>(P, c.t.rank, c.t.size, c.X, 1, g.qup, nullptr, 0.0, sums);
    c.t.sync();
    pr_combine(P, c.rl, c.rh, v, 1, true, epi);
    return;
  }
  row_pass_t<1, true>(c, P, UScaled{pv.src, pv.scale}, 1, g.qup, g.qlo, 0.0,
                      theta_alpha_or_half(I, g.qt), is_theta(I) ? &sumv : nullptr, false, sums,
                      epi);
}

// sum_i V_i(a) e_i in increasing i, with the loads issued in batches of 8
__device__ __forceinline__ double lz_row_dot(const Ctx& c, const Params& P, int k, int64_t a,
                                             const double* e) {
  double s = 0.0;
  int i = 0;
  for (; i + 8 <= k; i += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = slot_ptr(P, c.col[i + u])[a];
#pragma unroll
    for (int u = 0; u < 8; ++u) s = s + v[u] * e[i + u];
  }
  for (; i < k; ++i) s = s + slot_ptr(P, c.col[i])[a] * e[i];
  return s;
}

// h[i] = V_i . w for i < k  (result in c.rs.out[0..k)).  Lane i owns basis
// vector i and walks the warp's 32-row chunk sequentially (rows broadcast by
// shuffle): no per-vector warp reductions, fixed summation order.
// Small instances (<= 32 rows per CTA): warp w owns basis vectors w, w+16,
// lanes own rows; the owning warp's sum lands in rs.part[w][i], zeros elsewhere.
__device__ __forceinline__ void lz_dot_small(Ctx& c, const Params& P, int k, const double* wv,
                                             int64_t R) {
  const int lane = c.lane, warp = c.warp;
  const int64_t a = c.rl + lane;
  const bool ok = lane < R;
  const double wa = ok ? wv[a] : 0.0;
  for (int i = lane; i < k; i += 32) c.rs.part[warp * kRedK + i] = 0.0;
  __syncwarp();
  for (int i = warp; i < k; i += kWarps) {
    double t = ok ? slot_ptr(P, c.col[i])[a] * wa : 0.0;
    t = warp_sum(t);
    if (lane == 0) c.rs.part[warp * kRedK + i] = t;
  }
  team_reduce_smem(c.t, c.rs, k);
}

// Large instances: h[i] = V_i . w' over this CTA's rows with a thread per
// row, so basis vector i is read coalesced (consecutive threads, consecutive
// rows); the basis is taken 8 vectors at a time (8 partial sums per thread in
// registers, w re-read per group), optionally after w' = w - V_k hs (same
// thread, same rows: lz_row_dot order).  Partials are reduced warp -> CTA ->
// team in a fixed tree (deterministic).
template <bool SUB>
__device__ __forceinline__ void lz_dot_rows(Ctx& c, const Params& P, int k, double* w,
                                            const double* hs) {
  if (SUB)
    for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) w[a] = w[a] - lz_row_dot(c, P, k, a, hs);
  for (int g = 0; g < k; g += 8) {
    const double* v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = slot_ptr(P, c.col[g + u < k ? g + u : g]);
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.0;
    // two rows per step: 16 independent loads in flight per thread
    int64_t a = c.rl + threadIdx.x;
    for (; a + kThreads < c.rh; a += 2 * kThreads) {
      const double wa = w[a], wb = w[a + kThreads];
      double va[8], vb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        va[u] = g + u < k ? v[u][a] : 0.0;
        vb[u] = g + u < k ? v[u][a + kThreads] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] = (acc[u] + va[u] * wa) + vb[u] * wb;
    }
    if (a < c.rh) {
      const double wa = w[a];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (g + u < k) acc[u] = acc[u] + v[u][a] * wa;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (g + u < k) {
        const double x = warp_sum(acc[u]);
        if (c.lane == 0) c.rs.part[c.warp * kRedK + g + u] = x;
      }
  }
  team_reduce_smem(c.t, c.rs, k);
}

__device__ __forceinline__ void lz_dot(Ctx& c, const Params& P, int k, const double* w) {
  const int lane = c.lane;
  const int64_t rl = c.rl, rh = c.rh;
  if (rh - rl <= 32) {
    lz_dot_small(c, P, k, w, rh - rl);
    return;
  }
  if (rh - rl >= kRtMinRows) {
    lz_dot_rows<false>(c, P, k, const_cast<double*>(w), nullptr);
    return;
  }
  const double* vi = slot_ptr(P, c.col[lane < k ? lane : 0]);
  double mine = 0.0;
  for (int64_t a0 = rl + c.warp * 32; a0 < rh; a0 += kWarps * 32) {
    const int cnt = (int)min((int64_t)32, rh - a0);
    const double wl = lane < cnt ? w[a0 + lane] : 0.0;
#pragma unroll 8
    for (int r = 0; r < 32; ++r) {
      const double wr = __shfl_sync(kFull, wl, r);
      if (r < cnt && lane < k) mine = mine + vi[a0 + r] * wr;
    }
  }
  team_sum_lanes(c.t, c.rs, mine, k);
}
// w -= V_k h (thread per row, ordered over the basis); then h2 = V_k' w
// (dot_after) or (||w||^2, sum w) into rs.out[0..2)
__device__ __forceinline__ void lz_sub(Ctx& c, const Params& P, int k, double* w, const double* h,
                                       bool dot_after) {
  const int lane = c.lane;
  const int64_t rl = c.rl, rh = c.rh;
  if (rh - rl <= 32) {
    // small instances: partial sums over basis subsets per warp, combined in
    // warp order per row, then the dot (or the norm) on the new w
    const int64_t R = rh - rl;
    double* scr = c.tw;  // [kWarps][32] partials, then [32] new w
    {
      const int64_t a = rl + lane;
      double part = 0.0;
      if (lane < R)
        for (int i = c.warp; i < k; i += kWarps) part = part + slot_ptr(P, c.col[i])[a] * h[i];
      scr[c.warp * 32 + lane] = part;
    }
    __syncthreads();
    double* wn_s = scr + kWarps * 32;
    if (threadIdx.x < R) {
      double sacc = scr[threadIdx.x];
      for (int wv = 1; wv < kWarps; ++wv) sacc = sacc + scr[wv * 32 + threadIdx.x];
      const int64_t a = rl + threadIdx.x;
      const double wn = w[a] - sacc;
      w[a] = wn;
      wn_s[threadIdx.x] = wn;
    }
    __syncthreads();
    if (dot_after) {
      lz_dot_small(c, P, k, w, R);
    } else {
      double v[2] = {0.0, 0.0};
      if (threadIdx.x < R) {
        const double wn = wn_s[threadIdx.x];
        v[0] = wn * wn;
        v[1] = wn;
      }
      team_sum<2>(c.t, c.rs, v);
    }
    return;
  }
  if (dot_after && rh - rl >= kRtMinRows) {
    lz_dot_rows<true>(c, P, k, w, h);
    return;
  }
  const double* vi = slot_ptr(P, c.col[lane < k ? lane : 0]);
  double mine = 0.0, ssum = 0.0;
  for (int64_t a0 = rl + c.warp * 32; a0 < rh; a0 += kWarps * 32) {
    const int64_t a = a0 + lane;
    const int cnt = (int)min((int64_t)32, rh - a0);
    double wn = 0.0;
    if (a < rh) {
      wn = w[a] - lz_row_dot(c, P, k, a, h);
      w[a] = wn;
    }
    if (dot_after) {
#pragma unroll 8
      for (int r = 0; r < 32; ++r) {
        const double wr = __shfl_sync(kFull, wn, r);
        if (r < cnt && lane < k) mine = mine + vi[a0 + r] * wr;
      }
    } else {
      mine = mine + wn * wn;
      ssum = ssum + wn;
    }
  }
  if (dot_after) {
    team_sum_lanes(c.t, c.rs, mine, k);
  } else {
    double v[2] = {mine, ssum};
    team_sum<2>(c.t, c.rs, v);
  }
}
// orthogonalize (lanczos.cpp:22-28): h <- V'w; w -= Vh; h2 <- V'w; w -= Vh2;
// h += h2.  Returns ||w||^2 (and *wsum = sum w); h left in hh[0..k).
inline __device__ __noinline__ double lz_cgs2(Ctx& c, const Params& P, int k, double* w, double* hh,
                                       double* hh2, double* wsum) {
  lz_dot(c, P, k, w);
  if (threadIdx.x < (unsigned)k) hh[threadIdx.x] = c.rs.out[threadIdx.x];
  __syncthreads();
  lz_sub(c, P, k, w, hh, true);
  if (threadIdx.x < (unsigned)k) hh2[threadIdx.x] = c.rs.out[threadIdx.x];
  __syncthreads();
  lz_sub(c, P, k, w, hh2, false);
  const double ww = c.rs.out[0];
  *wsum = c.rs.out[1];
  __syncthreads();
  if (threadIdx.x < (unsigned)k) hh[threadIdx.x] = hh[threadIdx.x] + hh2[threadIdx.x];
  __syncthreads();
  return ww;
}
// slot dst = V_f e (e in smem, column of c.E); returns ||.||^2 and the sum
__device__ __forceinline__ double lz_combine(Ctx& c, const Params& P, int f, const double* e, int dst,
                                          double* sum) {
  double* d = slot_ptr(P, dst);
  double v[2] = {0.0, 0.0};
  for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) {
    const double s = lz_row_dot(c, P, f, a, e);
    d[a] = s;
    v[0] = v[0] + s * s;
    v[1] = v[1] + s;
  }
  team_sum<2>(c.t, c.rs, v);
  *sum = v[1];
  return v[0];
}

// Lanczos breakdown refill j (1-based, lanczos.cpp:127-130): the j-th next
// gaussian_vector of the start-vector stream.  The first n_refill are
// pre-drawn in HBM; later ones come from the launch's host service thread
// (capi.cu RefillService): CTA 0 posts the index to host-mapped memory and
// waits for the staged vector; the team barrier then releases every CTA to
// read its rows (uncached loads: the staging buffer is reused).  Returns null
// when no service is attached or the host does not answer within 60 s.
inline __device__ const double* lz_refill(Ctx& c, const Params& P, int j) {
  if (j <= P.n_refill) return P.lz_rand + (size_t)j * P.I.n;
  if (!P.svc_req || c.t.mw) return nullptr;
  if (c.t.rank == 0 && threadIdx.x == 0) {
    *(volatile int*)P.svc_req = j;
    __threadfence_system();
    const unsigned long long t0 = globaltimer_ns();
    int ok = 1;
    while (*(volatile const int*)P.svc_ready != j) {
      if (globaltimer_ns() - t0 > 60000000000ull) {
        ok = 0;
        break;
      }
      __nanosleep(1000);
    }
    __threadfence_system();
    *(volatile int*)P.svc_err = ok ? 0 : 1;
  }
  c.t.sync();
  if (*(volatile const int*)P.svc_err) return nullptr;
  return P.svc_buf;
}

// min_eigenpair (lanczos.cpp:32-141) of op = C + A*(q), i.e. B = -op.
// Per matvec: one gather pass (no barrier) + three all-reduces (CGS2).
inline __device__ __noinline__ bool lanczos_dev(Ctx& c, const Params& P, const GOp& g, double tol,
                                         int max_iters, int block_restart, LzOut& best) {
  const DevPairs& I = P.I;
  const int64_t n = I.n;
  const int kmax = (int)min((int64_t)block_restart, n);
  const int keep = max(1, kmax / 3);
  double* hh = c.hh;
  double* hh2 = c.hh2;
  unsigned long long used = 0ull;
  auto alloc = [&]() -> int {
    for (int sl = 0; sl < P.nslot; ++sl)
      if (!((used >> sl) & 1ull)) {
        used |= 1ull << sl;
        return sl;
      }
    return -1;
  };
  auto release = [&](int sl) {
    if (sl >= 0) used &= ~(1ull << sl);
  };
  int refill = 0;
  const int wslot[2] = {alloc(), alloc()};  // ping-pong w buffers
  int wc = 0;
  Pending pend;
  {
    // V(:,0) = v0/|v0|
    double v[2] = {0.0, 0.0};
    for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) {
      const double x = P.lz_rand[a];
      v[0] = v[0] + x * x;
      v[1] = v[1] + x;
    }
    team_sum<2>(c.t, c.rs, v);
    const int s0 = alloc();
    if (threadIdx.x == 0) c.col[0] = s0;
    const double nv = sqrt(v[0]);
    pend = Pending{P.lz_rand, nv, v[1] / nv, s0};
  }
  for (int idx = threadIdx.x; idx < kHLd * kHLd; idx += kThreads) c.H[idx] = 0.0;
  __syncthreads();
  int matvecs = 0, basis = 1, filled = 0;
  double beta = 0.0;
  best = LzOut();
  best.residual = INFINITY;
  double* w = slot_ptr(P, wslot[wc]);

  for (;;) {
    bool breakdown = false;
    while (filled < basis && matvecs < max_iters) {
      if (c.t.xfailed) {
        fail(c, kErrFabric, kMsgFabric);
        return false;
      }
      const int j = filled;
      w = slot_ptr(P, wslot[wc]);
      lz_apply(c, P, g, pend, w);  // materialises V(:, j) = pending column
      prof_mark(c, P, kPfLzApply);
      if (threadIdx.x == 0) c.vsum[pend.dst] = pend.sum;
      ++matvecs;
      double wsum;
      const double ww = lz_cgs2(c, P, basis, w, hh, hh2, &wsum);
      prof_mark(c, P, kPfLzCgs);
      if (threadIdx.x < (unsigned)basis) {
        c.H[threadIdx.x + j * kHLd] = hh[threadIdx.x];
        c.H[j + threadIdx.x * kHLd] = hh[threadIdx.x];
      }
      __syncthreads();
      ++filled;
      beta = sqrt(ww);
      double hmax = 0.0;
      for (int t = 0; t < basis; ++t) hmax = fmax(hmax, fabs(hh[t]));
      if (beta <= 1e-13 * fmax(1.0, hmax)) {
        breakdown = true;
        break;
      }
      if (basis < kmax) {
        const int sl = alloc();
        if (threadIdx.x == 0) {
          c.col[basis] = sl;
          c.H[basis + j * kHLd] = beta;
          c.H[j + basis * kHLd] = beta;
        }
        __syncthreads();
        pend = Pending{w, beta, wsum / beta, sl};
        wc ^= 1;
        ++basis;
      }
    }
    const int f = filled;
    jacobi_dev(c, c.H, kHLd, f);
    prof_mark(c, P, kPfJacobi);
    const int top = f - 1;
    const double mu = c.ev[top];
    const double res_est = breakdown ? 0.0 : beta * fabs(c.E[(f - 1) + top * f]);
    const bool budget_left = matvecs + 1 < max_iters;
    if (res_est <= tol * fmax(1.0, fabs(mu)) || !budget_left || (breakdown && filled >= n)) {
      // measure(V_f * e_top) (lanczos.cpp:61-74)
      const int xr = alloc();  // raw Ritz vector
      double xsum;
      const double nx2 = lz_combine(c, P, f, c.E + top * f, xr, &xsum);
      const double nx = sqrt(nx2);
      const int xs = alloc();  // normalised copy, materialised by the matvec
      const int bs = alloc();
      double* Bx = slot_ptr(P, bs);
      lz_apply(c, P, g, Pending{slot_ptr(P, xr), nx, xsum / nx, xs}, Bx);
      ++matvecs;
      release(xr);
      const double* x = slot_ptr(P, xs);
      double v1[1] = {0.0};
      for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) v1[0] = v1[0] + x[a] * Bx[a];
      team_sum<1>(c.t, c.rs, v1);
      const double mux = v1[0];
      double v2[1] = {0.0};
      for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) {
        const double d = Bx[a] - mux * x[a];
        v2[0] = v2[0] + d * d;
      }
      team_sum<1>(c.t, c.rs, v2);
      release(bs);
      LzOut o;
      o.lambda = -mux;
      o.residual = sqrt(v2[0]);
      o.matvecs = matvecs;
      o.converged = o.residual <= tol * fmax(1.0, fabs(o.lambda));
      o.vslot = xs;
      if (o.residual < best.residual) {
        release(best.vslot);
        best = o;
      } else {
        release(xs);
      }
      // best keeps the matvec count of its own measure (lanczos.cpp:70, :110-114)
      prof_mark(c, P, kPfLzMeasure);
      if (best.converged || matvecs >= max_iters || (breakdown && filled >= n)) return true;
    }
    // thick restart (lanczos.cpp:117-139)
    const int l = min(keep, f - 1 > 0 ? f - 1 : 1);
    int newcol[kLanczosMax];
    {
      for (int t = 0; t < l; ++t) newcol[t] = alloc();
      if (newcol[l - 1] < 0) {
        fail(c, kErrCapacity, kMsgRefillCap);
        return false;
      }
      double mine = 0.0;
      for (int64_t a0 = c.rl + c.warp * 32; a0 < c.rh; a0 += kWarps * 32) {
        const int64_t a = a0 + c.lane;
        const bool ok = a < c.rh;
        for (int t = 0; t < l; ++t) {
          double s = 0.0;
          if (ok) {
            s = lz_row_dot(c, P, f, a, c.E + (f - 1 - t) * f);
            slot_ptr(P, newcol[t])[a] = s;
          }
          const double ts = warp_sum(s);
          if (c.lane == t) mine = mine + ts;
        }
      }
      team_sum_lanes(c.t, c.rs, mine, l);
      if (threadIdx.x < (unsigned)l) c.vsum[newcol[threadIdx.x]] = c.rs.out[threadIdx.x];
      __syncthreads();
    }
    for (int t = 0; t < basis; ++t) release(c.col[t]);
    for (int idx = threadIdx.x; idx < kHLd * kHLd; idx += kThreads) c.H[idx] = 0.0;
    __syncthreads();
    if (threadIdx.x < (unsigned)l) {
      c.H[threadIdx.x + threadIdx.x * kHLd] = c.ev[f - 1 - threadIdx.x];
      c.col[threadIdx.x] = newcol[threadIdx.x];
    }
    __syncthreads();
    const int sl = alloc();
    if (threadIdx.x == 0) c.col[l] = sl;
    __syncthreads();
    const int w_idx = (w == slot_ptr(P, wslot[0])) ? 0 : 1;  // buffer holding the last w
    if (breakdown) {
      ++refill;
      // fresh direction: next gaussian_vector of the same stream, orthogonalised
      double* fr = slot_ptr(P, wslot[1 - w_idx]);
      const double* rnd = lz_refill(c, P, refill);
      if (!rnd) {
        fail(c, kErrCapacity, kMsgRefillCap);
        return false;
      }
      for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) fr[a] = __ldcv(rnd + a);
      __syncthreads();
      double fsum;
      const double fn2 = lz_cgs2(c, P, l, fr, hh, hh2, &fsum);
      const double fn = sqrt(fn2);
      if (fn <= 1e-13) return true;
      pend = Pending{fr, fn, fsum / fn, sl};
      wc = w_idx;
    } else {
      pend = Pending{w, beta, 0.0, sl};
      // sum of w/beta: w is the last CGS output
      double v[1] = {0.0};
      for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) v[0] = v[0] + w[a];
      team_sum<1>(c.t, c.rs, v);
      pend.sum = v[0] / beta;
      wc = 1 - w_idx;
    }
    basis = l + 1;
    filled = l;
    prof_mark(c, P, kPfLzRestart);
  }
}

// -------------------------------------------------------------------- HLR ---
struct HlrOut {
  int y_buf = 0, s = 1;
  double theta = 0, gap = 0, lambda_min = 0, al_val = 0, cdot = 0;
  double pr = 0, rr = 0, rt = 0;  // residual stats at exit (incl. trace)
  bool eig_trusted = true;
  int status = 0;
  long long aipp_iters = 0, fista_iters = 0, eig_products = 0;
  int fw_steps = 0;
};

// GradientOperator(Y): writes q/r arrays; returns p.r, ||r||^2 (incl. trace),
// and the trace residual / multiplier.
template <int S>
__device__ __noinline__ bool gradop_dev(Ctx& c, const Params& P, const double* Y, int s, double beta,
                           double* pr, double* rr, double* rt, double* qt) {
  const DevPairs& I = P.I;
  double ny2;
  factor_stats<S>(c, P, Y, s, &ny2);
  double sums[2] = {0.0, 0.0};
  bool bad = false;
  if (is_pr(I)) {
    // GradientOperator (sdp_instance.cpp:73-83): residual = map - b, q = p + beta residual
    pr_forward(P, c.t.rank, c.t.size, c.X, UPlain{Y}, s);
    c.t.sync();
    pr_map_combine(P, c.kl, c.kh, s, [&](int64_t k, double d) {
      const double r = d - I.b_up[k];
      const double pk = P.p_up[k];
      const double q = pk + beta * r;
      if (!isfinite(q)) bad = true;
      P.r_up[k] = r;
      P.q_up[k] = q;
      sums[0] = sums[0] + pk * r;
      sums[1] = sums[1] + r * r;
    });
  } else {
    if (!gradop_sell<S>(c, P, Y, beta, sums, &bad)) gradop_pass<S>(c, P, Y, s, beta, sums, &bad);
  }
  double v[3] = {sums[0], sums[1], bad ? 1.0 : 0.0};
  team_sum<3>(c.t, c.rs, v);
  double p_r = v[0], r_r = v[1];
  double r_t = 0.0, q_t = 0.0;
  if (is_theta(I)) {
    r_t = ny2 - I.b_trace;
    q_t = c.p_trace + beta * r_t;
    p_r = p_r + c.p_trace * r_t;
    r_r = r_r + r_t * r_t;
    if (!isfinite(q_t)) v[2] = 1.0;
  }
  *pr = p_r;
  *rr = r_r;
  *rt = r_t;
  *qt = q_t;
  if (v[2] != 0.0) {
    fail(c, kErrNumerical, kMsgGradOp);
    return false;
  }
  return true;
}

// <G Y, Y> with G = C + A*(q) stored (fw_gap, hlr.cpp:8-10)
template <int S>
__device__ __noinline__ double fw_gap_dev(Ctx& c, const Params& P, const double* Y, int s, const GOp& g) {
  const DevPairs& I = P.I;
  double ny2;
  factor_stats<S>(c, P, Y, s, &ny2);
  double gs = 0.0;
  auto epi = [&](int64_t, int, double h, double yo) { gs = gs + h * yo; };
  double sums[3] = {0.0, 0.0, 0.0};
  if (is_pr(I)) {
    pr_forward(P, c.t.rank, c.t.size, c.X, UPlain{Y}, s);
    c.t.sync();
    pr_inverse<true>(P, c.t.rank, c.t.size, c.X, s, g.qup, nullptr, 0.0, sums);
    c.t.sync();
    pr_combine(P, c.rl, c.rh, UPlain{Y}, s, true, epi);
  } else {
    row_pass<S, true>(c, P, Y, s, g.qup, g.qlo, 0.0, theta_alpha_or_half(I, g.qt),
                      is_theta(I) ? c.cs : nullptr, false, sums, epi);
  }
  double v[1] = {gs};
  team_sum<1>(c.t, c.rs, v);
  return v[0];
}

// rank_update / shrink (hlr.cpp:46-53, 127-134) into buffer dst.
template <int S>
__device__ __noinline__ void rank_update_dev(Ctx& c, const Params& P, const double* Y, int s, const double* y,
                                double alpha, bool theta_pos, double* dst, int* s_new) {
  if (theta_pos) {
    if (alpha == 1.0) {
      for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) dst[a] = y[a];
      *s_new = 1;
    } else {
      const double sa = sqrt(1.0 - alpha), sb = sqrt(alpha);
      const int s1 = s + 1;
      for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) {
        for (int k = 0; k < s; ++k) dst[a * s1 + k] = sa * Y[a * s + k];
        dst[a * s1 + s] = sb * y[a];
      }
      *s_new = s1;
    }
  } else {
    if (alpha == 1.0) {
      for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) dst[a] = 0.0;
      *s_new = 1;
    } else {
      const double sa = sqrt(1.0 - alpha);
      for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads)
        for (int k = 0; k < s; ++k) dst[a * s + k] = sa * Y[a * s + k];
      *s_new = s;
    }
  }
  c.t.sync();
}

// hlr_solve (hlr.cpp:55-151).  Input buffers[R.yt] with rank s.
inline __device__ __noinline__ bool hlr_dev(Ctx& c, const Params& P, Roles& R, int s, double beta, double eps_t,
                        int outer_iter, unsigned long long deadline_ns, HlrOut& out) {
  const DevPairs& I = P.I;
  const Cfg& cf = P.cfg;
  out = HlrOut();
  for (int step = 0;; ++step) {
    if (c.t.xfailed) {
      fail(c, kErrFabric, kMsgFabric);
      return false;
    }
    AippOut ao;
    bool ok = true;
    HALLAR_DISPATCH_S(s, ok = aipp_dev<S_>(c, P, R, s, eps_t, ao));
    if (!ok) return false;
    out.aipp_iters += ao.prox_iters;
    out.fista_iters += ao.fista_iters;
    const int ybuf = ao.w_buf;
    const double* Y = P.buf[ybuf];
    double pr = 0, rr = 0, rt = 0, qt = 0;
    HALLAR_DISPATCH_S(s, ok = gradop_dev<S_>(c, P, Y, s, beta, &pr, &rr, &rt, &qt));
    if (!ok) return false;
    prof_mark(c, P, kPfGradop);
    const GOp g{P.q_up, P.q_lo, qt};
    LzOut lz;
    if (!lanczos_dev(c, P, g, 0.1 * eps_t, cf.eig_max_iters, cf.eig_block_restart, lz))
      return false;
    out.eig_products += lz.matvecs;
    const double theta = lz.lambda < 0 ? -lz.lambda : 0.0;
    double gap;
    HALLAR_DISPATCH_S(s, gap = fw_gap_dev<S_>(c, P, Y, s, g));
    gap = gap + theta;
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
    prof_mark(c, P, kPfGap);
    if (done || no_steps || no_time || !lz.converged) {
      out.y_buf = ybuf;
      out.s = s;
      out.theta = theta;
      out.gap = gap;
      out.lambda_min = lz.lambda;
      out.al_val = ao.g_value;
      out.pr = pr;
      out.rr = rr;
      out.rt = rt;
      out.cdot = ao.g_value - pr - 0.5 * beta * rr;
      out.eig_trusted = lz.converged;
      out.status = done ? 0 : (no_time ? 2 : 1);
      if (!lz.converged && !done) out.status = 1;
      return true;
    }
    // fw_stepsize (hlr.cpp:31-44): numer = gap (same G, same Y)
    const double* yv = theta > 0 ? slot_ptr(P, lz.vslot) : nullptr;
    double denom;
    {
      double v[2] = {0.0, 0.0};
      if (yv)
        for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) v[0] = v[0] + yv[a] * yv[a];
      if (yv) publish_rows(c.t, yv, c.rl, c.rh, 1);
      if (is_pr(I)) {
        // A(yy') of the (n x 1) eigenvector; the spectrum cache is free here
        if (yv) {
          pr_forward(P, c.t.rank, c.t.size, c.X, UPlain{yv}, 1);
          c.t.sync();
        }
        pr_map_combine(P, c.kl, c.kh, yv ? 1 : 0, [&](int64_t k, double d) {
          const double t = (P.r_up[k] + I.b_up[k]) - d;
          v[1] = v[1] + t * t;
        });
      } else {
        for (int64_t k = c.kl + threadIdx.x; k < c.kh; k += kThreads) {
          const double d = yv ? yv[I.ei[k]] * yv[I.ej[k]] : 0.0;
          const double bk = I.b_up ? I.b_up[k] : 0.0;
          const double t = (P.r_up[k] + bk) - d;
          v[1] = v[1] + t * t;
        }
      }
      team_sum<2>(c.t, c.rs, v);
      double sq = v[1];
      if (is_theta(I)) {
        const double t = (rt + I.b_trace) - v[0];
        sq = sq + t * t;
      }
      denom = beta * sq;
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
      HALLAR_DISPATCH_S(s, rank_update_dev<S_>(c, P, Y, s, yv, alpha, theta > 0, dst, &s_new));
      const int t = R.yt;
      R.yt = R.tmp;
      R.tmp = t;
    }
    s = s_new;
    ++out.fw_steps;
    prof_mark(c, P, kPfFwStep);
    if (cf.trace) {
      double al;
      HALLAR_DISPATCH_S(s, ok = al_value_dev<S_>(c, P, P.buf[R.yt], s, P.p_up, c.p_trace, beta,
                                                 &al, nullptr));
      if (!ok) return false;
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

}  // namespace hallar
