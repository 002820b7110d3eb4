// Device-resident HALLaR for pair-constraint instances (Lovasz theta on any
// graph, matrix completion).  The whole solve — outer AL loop, HLR, ADAP-AIPP,
// ADAP-FISTA, thick-restart Lanczos, certificate — runs inside ONE persistent
// cooperative kernel; scalars are reduced deterministically and replicated in
// every thread, so the control flow never leaves the GPU.
//
// Reference statements are cited as file:line into /root/reference/proj/src.
// Arithmetic is compiled with -fmad=false so element-wise expressions round
// exactly like the reference's SSE2 build (no FMA contraction).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"
#include "team.cuh"
#include "pr.cuh"

namespace hallar {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kTileLd = 33;  // padded fold tile stride (conflict-free)
constexpr int kHLd = kLanczosMax + 1;

enum Msg : int {
  kMsgNone = 0,
  kMsgFistaDiverged = 1,
  kMsgAlValue = 2,
  kMsgAlValGrad = 3,
  kMsgAlGrad = 4,
  kMsgGradOp = 5,
  kMsgProjectBall = 6,
  kMsgNonFinite = 7,
  kMsgRankCap = 8,
  kMsgRefillCap = 9,
  kMsgRank32 = 10,
  kMsgFabric = 11,
};

struct Ctx {
  Team t;
  RedSmem rs;
  int64_t* vlo;   // tile engine: [kTileRows+1] lower row pointers of the tile
  int64_t* vup;   // [kTileRows+1] upper row pointers
  double* tw;     // [kTileEntries] w per entry
  int32_t* tcol;  // [kTileEntries] gathered row per entry
  double* tterm;  // [kTileEntries * 4] w * U(b, c), c < 4
  double2* X;     // phase retrieval transform buffer (aliases the tile arrays)
  // launch-long cache of the CTA's static pair structure (small instances)
  bool cached = false;
  int32_t* ccol;   // [kCacheEnt] lower columns of the CTA's rows, then upper columns
  int32_t* crlo;   // [kCacheRows+1] lo_ptr[r] - lo_ptr[rl]
  int32_t* crup;   // [kCacheRows+1] up_ptr[r] - up_ptr[rl]
  int32_t* ctr;    // [kCacheTiles+1] tile_row[t] - rl
  int64_t clo0 = 0, cup0 = 0;  // lo_ptr[rl], up_ptr[rl]
  int32_t cnlo = 0;            // lower entries of the CTA's rows
  double* cs;     // [kSMax] column sums of the gathered factor (theta C-term)
  double* H;      // [kHLd][kHLd] Lanczos projected matrix (column-major)
  double* JA;     // [32*32] Jacobi work
  double* JV;     // [32*32]
  double* E;      // [32*32] sorted eigenvectors
  double* ev;     // [32] sorted eigenvalues
  double* jcs;    // [32] rotation cos/sin pairs
  int* jpq;       // [32] pair indices
  double* vsum;   // [nslot] column sums of Lanczos slots (theta)
  int* col;       // [kHLd+1] Lanczos basis -> slot
  int64_t tl, th;  // row tiles owned by this CTA
  int64_t rl, rh;  // rows owned by this CTA (= its tiles' rows)
  int64_t kl, kh;  // edges owned by this CTA
  double* hh;     // [32] Lanczos CGS coefficients
  double* hh2;    // [32]
  int warp, lane;
  int status = kOk;
  int msg = kMsgNone;
  unsigned long long prof_last = 0;
  const Params* Pp = nullptr;  // launch parameters (debug hooks)
  double deadline = 1e300;  // solve: t0 + time_limit (team_now ns), see fista_dev
  bool timed_out = false;
  double beta = 0.0;     // current AL penalty (replicated)
  double p_trace = 0.0;  // current p[m-1] (theta trace multiplier)
};

__device__ __forceinline__ bool is_theta(const DevPairs& I) { return I.has_trace != 0; }

__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void prof_mark(Ctx& c, const Params& P, int cat) {
  if (P.prof && c.t.rank == 0 && threadIdx.x == 0) {
    const unsigned long long now = gtimer_ns();
    P.prof[cat] += now - c.prof_last;
    P.prof[kProfCats + cat] += 1;
    c.prof_last = now;
  }
}

__device__ __forceinline__ void fail(Ctx& c, int status, int msg) {
  if (c.status == kOk) {
    c.status = status;
    c.msg = msg;
  }
}

// ------------------------------------------------------------------ layout --
// Rows are split so that (lower + upper entries + 8) is balanced per CTA.
inline __device__ int64_t work_prefix(const DevPairs& I, int64_t a) {
  return I.lo_ptr[a] + I.up_ptr[a] + 8 * a;
}
inline __device__ int64_t row_split(const DevPairs& I, int rank, int size) {
  if (rank <= 0) return 0;
  if (rank >= size) return I.n;
  const int64_t total = work_prefix(I, I.n);
  const int64_t target = (int64_t)((__int128)total * rank / size);
  int64_t lo = 0, hi = I.n;  // first a with prefix >= target
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (work_prefix(I, mid) < target) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------- tile engine ---
// The CTA walks its tiles (host-precomputed runs of consecutive rows with
// <= kTileEntries entries and <= kTileRows rows).  Per tile:
//   1. row pointers of the tile -> smem;
//   2. every thread takes entries v = tid, tid+512, ... of the tile's merged
//      (lower-then-upper per row) entry list: loads col / multiplier / b,
//      gathers U_b (and U_a), computes w_v = 0.5 q_v and the products
//      w_v U(b_v, c) for c < 4 into smem — all entries in flight at once;
//   3. one thread per (row, column) folds the products of its row in entry
//      (= increasing constraint k) order and runs the epilogue.
// The fold adds the same rounded products in the same order as the reference
// adjoint_into (instances.cpp:45-52), so the pair adjoint stays bit-exact.
// Column index of a thread in phase 3 is fixed (tid % s), so per-column
// epilogue accumulators are plain registers.
//
// For every row a owned by this CTA and column c:
//   h(a,c) = init(a,c) (+)fold_k 0.5 q_k U(b_k,c),  init = alpha*U(a,c) - cs[c] | 0
// q_k = P_k (FIXED) or P_k + beta (U_a.U_b - b_k) (!FIXED); !FIXED also
// accumulates over upper entries (each constraint once):
//   sums[0] += p r, sums[1] += r^2, sums[2] += q (r + b).
// epi(a, c, h, U(a,c)) is called once per (row, column).
struct UPlain {
  const double* __restrict__ U;
  __device__ __forceinline__ double operator()(int64_t o) const { return U[o]; }
  __device__ __forceinline__ const double* base() const { return U; }
  __device__ __forceinline__ double xf(double raw) const { return raw; }
};
struct UScaled {  // Lanczos: v = src / scale, materialised on the fly
  const double* __restrict__ src;
  double sc;
  __device__ __forceinline__ double operator()(int64_t o) const { return src[o] / sc; }
  __device__ __forceinline__ const double* base() const { return src; }
  __device__ __forceinline__ double xf(double raw) const { return raw / sc; }
};

__device__ __forceinline__ void group_sync(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(kGT) : "memory");
}

// cp.async (LDGSTS): global -> shared copies that hold no registers in flight
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cpa4(void* d, const void* s) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(d)), "l"(s) : "memory");
}
__device__ __forceinline__ void cpa8(void* d, const void* s) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(d)), "l"(s) : "memory");
}
// the same copies with an L2 evict-first hint: streamed once per pass, they
// must not push the gathered factor rows out of L2
__device__ __forceinline__ unsigned long long l2_evict_first() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void cpa4s(void* d, const void* s, unsigned long long pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(smem_u32(d)), "l"(s),
               "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cpa8s(void* d, const void* s, unsigned long long pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(smem_u32(d)), "l"(s),
               "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait_group1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }


// ------------------------------- row-thread engine, fixed-q (cp.async) -----
// Fixed-multiplier passes (Lanczos matvec, fw_gap, operator calls): as the
// row-thread engine below, but the row's entries form one merged stream of
// batches of B.  A batch's column indices, multipliers and
// right-hand sides are brought into the thread's private shared-memory slot
// with cp.async (LDGSTS) one batch ahead (the first batch of the next row
// during the last batch of this one; row pointers one row ahead), so per
// batch only its B independent gathers U(b, :) sit on the critical path and
// no registers are spent on prefetched data.  Slots are [stage][u][thread]
// (conflict-free); each thread reads only what it copied itself, so no
// barrier is needed.  Arithmetic is the v1 engine's term for term, so the
// results are bit-identical.
constexpr int kRtB = 8;  // staging depth per batch (B <= kRtB)

template <int S, bool FIXED, class UA, class Epi>
__device__ __forceinline__ void row_pass_rt_async(Ctx& c, const Params& P, const UA& U,
                                            const double* __restrict__ Pup,
                                            const double* __restrict__ Plo, double beta,
                                            double alpha, const double* cs, bool zero_init,
                                            double (&sums)[3], Epi& epi) {
  static_assert(S >= 1 && S <= 4, "row-thread engine: ranks 1..4");
  constexpr int B = S <= 2 ? 8 : 4;
  static_assert(B <= kRtB, "batch above the staging depth");
  const DevPairs& I = P.I;
  const bool has_b = !FIXED && I.b_up != nullptr;
  const int t = threadIdx.x;
  // staging slots inside the pass scratch: col [2][kRtB][512] int32, p and b [2][kRtB][512]
  int32_t* const colS = reinterpret_cast<int32_t*>(c.tw);
  double* const pS = c.tw + kRtB * kThreads;
  double* const bS = pS + 2 * kRtB * kThreads;
  double csr[S];
#pragma unroll
  for (int k = 0; k < S; ++k) csr[k] = cs ? cs[k] : 0.0;

  struct Row {
    int64_t lo0, up0;  // first lower / upper entry
    int nlo, nv;       // lower entries, all entries
  };
  auto load_row = [&](int64_t a) {
    Row r;
    r.lo0 = __ldg(I.lo_ptr + a);
    r.up0 = __ldg(I.up_ptr + a);
    r.nlo = (int)(__ldg(I.lo_ptr + a + 1) - r.lo0);
    r.nv = r.nlo + (int)(__ldg(I.up_ptr + a + 1) - r.up0);
    return r;
  };
  // batch [v0, v0 + B) of a row's merged stream -> stage slot (async)
  auto issue = [&](int st, const Row& r, int v0) {
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int v = v0 + u;
      if (v < r.nv) {
        const bool up = v >= r.nlo;
        const int64_t e = up ? r.up0 + (v - r.nlo) : r.lo0 + v;
        const int slot = (st * kRtB + u) * kThreads + t;
        cpa4(colS + slot, (up ? I.ej : I.lo_col) + e);
        cpa8(pS + slot, (up ? Pup : Plo) + e);
        if (has_b) cpa8(bS + slot, (up ? I.b_up : I.b_lo) + e);
      }
    }
  };

  int64_t a = c.rl + t;
  Row R{}, Rn{};
  if (a < c.rh) R = load_row(a);
  int64_t an = a + kThreads;
  if (an < c.rh) Rn = load_row(an);
  int st = 0;
  bool pref = false;  // the current row's first batch is already in flight in stage st
  while (a < c.rh) {
    if (!pref) {
      issue(st, R, 0);
      cpa_commit();
    }
    pref = false;
    double ua[S], acc[S];
#pragma unroll
    for (int k = 0; k < S; ++k) {
      ua[k] = U(a * S + k);
      acc[k] = 0.0;
      if (!zero_init) {
        acc[k] = alpha * ua[k];
        if (cs) acc[k] = acc[k] - csr[k];
      }
    }
#pragma unroll 1
    for (int v0 = 0; v0 < R.nv; v0 += B) {
      // next batch of this row, or the first batch of the next row, in flight
      if (v0 + B < R.nv) {
        issue(st ^ 1, R, v0 + B);
      } else if (an < c.rh) {
        issue(st ^ 1, Rn, 0);
        pref = true;
      }
      cpa_commit();
      cpa_wait_group1();  // this batch (all but the newest group) has landed
      double ub[B][S], pk[B], bk[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int slot = (st * kRtB + u) * kThreads + t;
        const bool ok = v0 + u < R.nv;
        const int64_t bcol = ok ? (int64_t)colS[slot] : a;
        pk[u] = ok ? pS[slot] : 0.0;
        bk[u] = (ok && has_b) ? bS[slot] : 0.0;
#pragma unroll
        for (int k = 0; k < S; ++k) ub[u][k] = U(bcol * S + k);
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int v = v0 + u;
        if (v >= R.nv) break;
        const bool upper = v >= R.nlo;
        double w;
        if (FIXED) {
          w = 0.5 * pk[u];
        } else {
          double d = 0.0;
#pragma unroll
          for (int k = 0; k < S; ++k) {
            const double tt = ua[k] * ub[u][k];
            d = (k == 0) ? tt : d + tt;
          }
          const double rr = d - bk[u];
          const double q = pk[u] + beta * rr;
          w = 0.5 * q;
          if (upper) {
            sums[0] = sums[0] + pk[u] * rr;
            sums[1] = sums[1] + rr * rr;
            sums[2] = sums[2] + q * (rr + bk[u]);
          }
        }
        // skipped terms (w == 0, instances.cpp:47): x + (-0.0) == x exactly
#pragma unroll
        for (int k = 0; k < S; ++k) acc[k] = acc[k] + ((w != 0.0) ? w * ub[u][k] : -0.0);
      }
      st ^= 1;
    }
#pragma unroll
    for (int k = 0; k < S; ++k) epi(a, k, acc[k], ua[k]);
    a = an;
    R = Rn;
    an += kThreads;
    if (an < c.rh) Rn = load_row(an);
  }
  cpa_wait_all();
  __syncthreads();
}

// ------------------------------------------------- row-thread engine ------
// Large instances (many rows per CTA), ranks 1..4: one thread owns a whole
// row and walks its lower then upper entries — increasing constraint k, the
// reference's adjoint_into order (instances.cpp:45-52) — with the column
// accumulators in registers.  Entries are taken in batches of B: the B
// column indices and multipliers (contiguous per row) are loaded first, then
// the B gathered rows U(b, :), then the batch is folded in order.  No shared
// memory, no barriers and no entry->row search: every thread keeps B
// independent gathers in flight (the v1 tile engine, which spreads one row's
// entries over threads, is kept for instances with few rows per CTA).
// Arithmetic is the v1 engine's term for term, so results are bit-identical.
template <int S, bool FIXED, class UA, class Epi>
__device__ __forceinline__ void row_pass_rt(Ctx& c, const Params& P, const UA& U,
                                            const double* __restrict__ Pup,
                                            const double* __restrict__ Plo, double beta,
                                            double alpha, const double* cs, bool zero_init,
                                            double (&sums)[3], Epi& epi) {
  static_assert(S >= 1 && S <= 4, "row-thread engine: ranks 1..4");
  constexpr int B = S <= 2 ? 8 : 4;
  const DevPairs& I = P.I;
  const bool has_b = !FIXED && I.b_up != nullptr;
  double csr[S];
#pragma unroll
  for (int k = 0; k < S; ++k) csr[k] = cs ? cs[k] : 0.0;
  for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) {
    double ua[S], acc[S];
#pragma unroll
    for (int k = 0; k < S; ++k) {
      ua[k] = U(a * S + k);
      acc[k] = 0.0;
      if (!zero_init) {
        acc[k] = alpha * ua[k];
        if (cs) acc[k] = acc[k] - csr[k];
      }
    }
#pragma unroll 1
    for (int part = 0; part < 2; ++part) {
      const bool upper = part == 1;
      const int64_t e0 = upper ? __ldg(I.up_ptr + a) : __ldg(I.lo_ptr + a);
      const int64_t e1 = upper ? __ldg(I.up_ptr + a + 1) : __ldg(I.lo_ptr + a + 1);
      const int32_t* __restrict__ colp = upper ? I.ej : I.lo_col;
      const double* __restrict__ pp = upper ? Pup : Plo;
      const double* __restrict__ bp = upper ? I.b_up : I.b_lo;
#pragma unroll 1
      for (int64_t e = e0, step = B; e < e1; e += step) {
        int64_t bc[B];
        double pk[B], bk[B];
        // matrix completion (long rows, three streams per entry): an odd start is
        // peeled as a one-entry batch so full batches load their column indices,
        // multipliers and right-hand sides as 8/16-byte pairs (fewer load
        // instructions: these passes are load-queue throttled); order unchanged
        step = (has_b && (e & 1)) ? 1 : B;
        const int lim = (int)min((int64_t)step, e1 - e);
        if (has_b && lim == B) {
#pragma unroll
          for (int u = 0; u < B; u += 2) {
            const int2 cv = __ldg(reinterpret_cast<const int2*>(colp + e + u));
            const double2 pv = __ldg(reinterpret_cast<const double2*>(pp + e + u));
            const double2 bv = __ldg(reinterpret_cast<const double2*>(bp + e + u));
            bc[u] = cv.x;
            bc[u + 1] = cv.y;
            pk[u] = pv.x;
            pk[u + 1] = pv.y;
            bk[u] = bv.x;
            bk[u + 1] = bv.y;
          }
        } else {
#pragma unroll
          for (int u = 0; u < B; ++u) {
            const bool ok = u < lim;
            bc[u] = ok ? (int64_t)__ldg(colp + e + u) : a;
            pk[u] = ok ? __ldg(pp + e + u) : 0.0;
            bk[u] = (ok && has_b) ? __ldg(bp + e + u) : 0.0;
          }
        }
        double ub[B][S];
#pragma unroll
        for (int u = 0; u < B; ++u)
#pragma unroll
          for (int k = 0; k < S; ++k) ub[u][k] = U(bc[u] * S + k);
#pragma unroll
        for (int u = 0; u < B; ++u) {
          if (u >= lim) break;
          double w;
          if (FIXED) {
            w = 0.5 * pk[u];
          } else {
            double d = 0.0;
#pragma unroll
            for (int k = 0; k < S; ++k) {
              const double t = ua[k] * ub[u][k];
              d = (k == 0) ? t : d + t;
            }
            const double rr = d - bk[u];
            const double q = pk[u] + beta * rr;
            w = 0.5 * q;
            if (upper) {
              sums[0] = sums[0] + pk[u] * rr;
              sums[1] = sums[1] + rr * rr;
              sums[2] = sums[2] + q * (rr + bk[u]);
            }
          }
          // skipped terms (w == 0, instances.cpp:47): x + (-0.0) == x exactly
#pragma unroll
          for (int k = 0; k < S; ++k) acc[k] = acc[k] + ((w != 0.0) ? w * ub[u][k] : -0.0);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < S; ++k) epi(a, k, acc[k], ua[k]);
  }
  __syncthreads();
}

// ------------------------------------------------------- SELL engine ------
// Single-GPU row passes of large instances: the same one-thread-per-row fold
// as the row-thread engine (lower then upper entries, increasing k, the
// reference's adjoint_into order, so results are bit-identical), but a warp
// owns the 32 rows of one SELL slice (DevPairs::s_*), so the stream loads of
// entry v (column index, multiplier, right-hand side) are 32 consecutive
// slots: one or two cache lines per warp load instead of 32.  The gathered
// factor rows are read with the widest aligned vector load (s = 2: 128-bit,
// s = 4: 256-bit, s = 3: 64 + 128-bit), so a gathered row costs one L1
// wavefront per entry; the streams are read evict-first (__ldcs) so the
// gathered factor stays L2-resident.
// A rank-3 factor copied to rows of 4 doubles (P.pad): one 256-bit load per
// gathered row instead of a 64-bit + a 128-bit one (the gathers are
// L1-wavefront bound).  Filled by pad_rows before a pass, read-only in it.
struct UPad4 {
  const double* __restrict__ U;
  __device__ __forceinline__ double operator()(int64_t o) const { return U[(o / 3) * 4 + o % 3]; }
  __device__ __forceinline__ const double* base() const { return U; }
  __device__ __forceinline__ double xf(double raw) const { return raw; }
};
template <class UA>
struct URowStride {
  static constexpr int v = 0;  // the rank
};
template <>
struct URowStride<UPad4> {
  static constexpr int v = 4;
};

template <int S, class UA>
__device__ __forceinline__ void sell_row(const UA& U, int64_t b, double (&o)[S]) {
  constexpr int ST = URowStride<UA>::v ? URowStride<UA>::v : S;
  const double* p = U.base() + b * ST;
  if constexpr (ST == 4 && S == 3) {
    double t0, t1, t2, t3;
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(t0), "=d"(t1), "=d"(t2), "=d"(t3)
                 : "l"(p));
    (void)t3;
    o[0] = t0;
    o[1] = t1;
    o[2] = t2;
  } else if constexpr (S == 1) {
    o[0] = U.xf(p[0]);
  } else if constexpr (S == 2) {
    const double2 v = *reinterpret_cast<const double2*>(p);
    o[0] = U.xf(v.x);
    o[1] = U.xf(v.y);
  } else if constexpr (S == 3) {
    if (b & 1) {
      const double2 v = *reinterpret_cast<const double2*>(p + 1);
      o[0] = U.xf(p[0]);
      o[1] = U.xf(v.x);
      o[2] = U.xf(v.y);
    } else {
      const double2 v = *reinterpret_cast<const double2*>(p);
      o[0] = U.xf(v.x);
      o[1] = U.xf(v.y);
      o[2] = U.xf(p[2]);
    }
  } else {
    double t0, t1, t2, t3;
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(t0), "=d"(t1), "=d"(t2), "=d"(t3)
                 : "l"(p));
    o[0] = U.xf(t0);
    o[1] = U.xf(t1);
    o[2] = U.xf(t2);
    o[3] = U.xf(t3);
  }
}
template <int S>
__device__ __forceinline__ bool sell_aligned(const double* base) {
  const unsigned long long a = reinterpret_cast<unsigned long long>(base);
  return S == 1 || (S == 4 ? (a & 31) == 0 : (a & 15) == 0);
}

// rows [rl, rh) of a rank-3 factor -> P.pad (stride 4), then a team barrier
// (the pass that follows gathers every row)
template <class UA>
__device__ __forceinline__ void pad_rows3(Ctx& c, const Params& P, const UA& U) {
  for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) {
    const double u0 = U(a * 3), u1 = U(a * 3 + 1), u2 = U(a * 3 + 2);
    double* d = P.pad + a * 4;
    *reinterpret_cast<double2*>(d) = make_double2(u0, u1);
    d[2] = u2;
  }
  c.t.sync();
}

template <int S, bool FIXED, class UA, class Epi>
__device__ __forceinline__ void row_pass_sell(Ctx& c, const Params& P, const UA& U,
                                              const double* __restrict__ Ps, double beta,
                                              double alpha, const double* cs, bool zero_init,
                                              double (&sums)[3], Epi& epi) {
  static_assert(S >= 1 && S <= 4, "SELL engine: ranks 1..4");
  constexpr int B = S <= 2 ? 8 : 4;
  const DevPairs& I = P.I;
  const bool has_b = !FIXED && I.s_b != nullptr;
  double csr[S];
#pragma unroll
  for (int k = 0; k < S; ++k) csr[k] = cs ? cs[k] : 0.0;
  const int64_t sl0 = c.rl >> 5, sl1 = (c.rh + 31) >> 5;
  for (int64_t sl = sl0 + c.warp; sl < sl1; sl += kWarps) {
    const int64_t a = (sl << 5) + c.lane;
    const bool mine = a >= c.rl && a < c.rh;
    const int64_t s_beg = __ldg(I.s_off + sl);
    const int L = (int)((__ldg(I.s_off + sl + 1) - s_beg) >> 5);
    const int64_t base = s_beg + c.lane;
    const int nv = mine ? __ldg(I.s_nv + a) : 0;
    const int nlo = mine ? __ldg(I.s_nlo + a) : 0;
    double ua[S], acc[S];
    if (mine) {
      sell_row<S>(U, a, ua);
    } else {
#pragma unroll
      for (int k = 0; k < S; ++k) ua[k] = 0.0;
    }
#pragma unroll
    for (int k = 0; k < S; ++k) {
      acc[k] = 0.0;
      if (!zero_init) {
        acc[k] = alpha * ua[k];
        if (cs) acc[k] = acc[k] - csr[k];
      }
    }
#pragma unroll 1
    for (int v0 = 0; v0 < L; v0 += B) {
      int32_t bc[B];
      double pk[B], bk[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const bool ok = v0 + u < nv;
        const int64_t slot = base + (int64_t)(v0 + u) * 32;
        bc[u] = ok ? __ldcs(I.s_col + slot) : 0;
        pk[u] = ok ? __ldcs(Ps + slot) : 0.0;
        bk[u] = (ok && has_b) ? __ldcs(I.s_b + slot) : 0.0;
      }
      double ub[B][S];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        if (v0 + u < nv) {
          sell_row<S>(U, bc[u], ub[u]);
        } else {
#pragma unroll
          for (int k = 0; k < S; ++k) ub[u][k] = 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int v = v0 + u;
        if (v >= nv) break;
        const bool upper = v >= nlo;
        double w;
        if (FIXED) {
          w = 0.5 * pk[u];
        } else {
          double d = 0.0;
#pragma unroll
          for (int k = 0; k < S; ++k) {
            const double t = ua[k] * ub[u][k];
            d = (k == 0) ? t : d + t;
          }
          const double rr = d - bk[u];
          const double q = pk[u] + beta * rr;
          w = 0.5 * q;
          if (upper) {
            sums[0] = sums[0] + pk[u] * rr;
            sums[1] = sums[1] + rr * rr;
            sums[2] = sums[2] + q * (rr + bk[u]);
          }
        }
        // skipped terms (w == 0, instances.cpp:47): x + (-0.0) == x exactly
#pragma unroll
        for (int k = 0; k < S; ++k) acc[k] = acc[k] + ((w != 0.0) ? w * ub[u][k] : -0.0);
      }
    }
    if (mine) {
#pragma unroll
      for (int k = 0; k < S; ++k) epi(a, k, acc[k], ua[k]);
    }
  }
  __syncthreads();
}

// mbarrier + 1-D bulk copy (TMA) helpers
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_inval(unsigned long long* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes,
                                            unsigned long long* bar, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// Pipelined SELL engine: entry v of a slice's 32 rows is 32 consecutive
// slots, so a batch of B entries of every stream (column index, multiplier,
// right-hand side) is one contiguous block per stream.  Lane 0 of each warp
// streams the NEXT batch's blocks into a shared-memory stage with 1-D bulk
// copies (TMA, L2 evict-first, completion on a per-warp mbarrier) while the
// warp gathers and folds the current batch: per batch only the gathers of
// factor rows sit on the critical path (the passes are latency-bound at 16
// warps per SM), and the streams cost no per-lane load instructions.  Same
// fold as row_pass_sell, so results are bit-identical.
template <int S, bool FIXED, bool HB, class UA, class Epi, bool GOP = false>
__device__ __forceinline__ void row_pass_sell_async(Ctx& c, const Params& P, const UA& U,
                                                    const double* __restrict__ Ps, double beta,
                                                    double alpha, const double* cs, bool zero_init,
                                                    double (&sums)[3], Epi& epi) {
  static_assert(S >= 1 && S <= 4, "SELL engine: ranks 1..4");
  // GOP: the GradientOperator build (sdp_instance.cpp:73-83) instead of a row
  // fold: per entry r = U_a.U_b - b, q = p + beta r written in SELL order and,
  // for upper entries, in edge order (edge id streamed from s_eid); sums[0] =
  // p.r, sums[1] = r.r over upper entries, sums[2] counts non-finite q
  // per warp and stage: B x 32 x (4 [+ 4] + 8 [+ 8]) bytes; two stages per warp
  constexpr int B = GOP ? (HB ? 5 : 7) : (HB ? 6 : 8);
  constexpr int kStageInts = B * 32;
  constexpr int kInts = GOP ? 2 : 1;  // int32 streams (column, [edge id]) in doubles of B x 512
  // layout in doubles: kInts x B x kThreads (int32 streams, both stages), 2 x B x
  // kThreads per f64 stream, then the 2 x kWarps barriers
  static_assert((kInts + (HB ? 4 : 2)) * B * kThreads + 2 * kWarps <= kPassScratch,
                "SELL stages exceed the pass scratch");
  const DevPairs& I = P.I;
  const int lane = c.lane, warp = c.warp;
  // scratch: [warp][stage] col blocks (int32), [edge-id blocks], p blocks, b blocks, barriers
  int32_t* const colW = reinterpret_cast<int32_t*>(c.tw) + warp * 2 * kStageInts;
  uint32_t* const eidW = reinterpret_cast<uint32_t*>(c.tw + B * kThreads) + warp * 2 * kStageInts;
  double* const pW = c.tw + kInts * B * kThreads + warp * 2 * kStageInts;
  double* const bW = c.tw + (kInts + 2) * B * kThreads + warp * 2 * kStageInts;
  unsigned long long* const bar =
      reinterpret_cast<unsigned long long*>(c.tw + (kInts + (HB ? 4 : 2)) * B * kThreads) + warp * 2;
  double csr[S];
#pragma unroll
  for (int k = 0; k < S; ++k) csr[k] = cs ? cs[k] : 0.0;
  const int64_t sl1 = (c.rh + 31) >> 5;
  struct Sl {
    int64_t a, s_beg;
    int L, nv, nlo;
    bool mine;
  };
  auto slice = [&](int64_t sl) {
    Sl x;
    x.a = (sl << 5) + lane;
    x.mine = x.a >= c.rl && x.a < c.rh;
    x.s_beg = __ldg(I.s_off + sl);
    x.L = (int)((__ldg(I.s_off + sl + 1) - x.s_beg) >> 5);
    x.nv = x.mine ? __ldg(I.s_nv + x.a) : 0;
    x.nlo = x.mine ? __ldg(I.s_nlo + x.a) : 0;
    return x;
  };
  const unsigned long long pol = l2_evict_first();
  auto issue = [&](int st, const Sl& x, int v0) {  // lane 0 only
    const int ne = min(B, x.L - v0) * 32;
    const int64_t g = x.s_beg + (int64_t)v0 * 32;
    mbar_expect_tx(bar + st, (unsigned)ne * ((HB ? 20u : 12u) + (GOP ? 4u : 0u)));
    tma_load_1d(colW + st * kStageInts, I.s_col + g, ne * 4, bar + st, pol);
    if (GOP) tma_load_1d(eidW + st * kStageInts, I.s_eid + g, ne * 4, bar + st, pol);
    tma_load_1d(pW + st * kStageInts, Ps + g, ne * 8, bar + st, pol);
    if (HB) tma_load_1d(bW + st * kStageInts, I.s_b + g, ne * 8, bar + st, pol);
  };
  int64_t sl = (c.rl >> 5) + warp;
  if (sl < sl1) {
    if (lane == 0) {
      mbar_init(bar, 1);
      mbar_init(bar + 1, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    Sl X = slice(sl);
    int st = 0;
    unsigned phase = 0;  // bit st: parity of stage st's next completion
    if (lane == 0 && X.L > 0) issue(0, X, 0);
    while (true) {
      double ua[S], acc[S];
      if (X.mine) {
        sell_row<S>(U, X.a, ua);
      } else {
#pragma unroll
        for (int k = 0; k < S; ++k) ua[k] = 0.0;
      }
#pragma unroll
      for (int k = 0; k < S; ++k) {
        acc[k] = 0.0;
        if (!zero_init) {
          acc[k] = alpha * ua[k];
          if (cs) acc[k] = acc[k] - csr[k];
        }
      }
      const int64_t sln = sl + kWarps;
      const bool have_next = sln < sl1;
      Sl XN{};
      if (have_next) XN = slice(sln);
#pragma unroll 1
      for (int v0 = 0; v0 < X.L; v0 += B) {
        // the next batch (this slice, or the next slice's first) in flight
        if (lane == 0) {
          if (v0 + B < X.L)
            issue(st ^ 1, X, v0 + B);
          else if (have_next && XN.L > 0)
            issue(st ^ 1, XN, 0);
        }
        mbar_wait(bar + st, (phase >> st) & 1u);
        phase ^= 1u << st;
        int32_t bc[B];
        uint32_t ek[B];
        double pk[B], bk[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
          const bool ok = v0 + u < X.nv;
          bc[u] = ok ? colW[st * kStageInts + u * 32 + lane] : 0;
          ek[u] = (ok && GOP) ? eidW[st * kStageInts + u * 32 + lane] : 0u;
          pk[u] = ok ? pW[st * kStageInts + u * 32 + lane] : 0.0;
          bk[u] = (ok && HB) ? bW[st * kStageInts + u * 32 + lane] : 0.0;
        }
        __syncwarp();  // stage st is refilled by the next-but-one issue
        double ub[B][S];
#pragma unroll
        for (int u = 0; u < B; ++u) {
          if (v0 + u < X.nv) {
            sell_row<S>(U, bc[u], ub[u]);
          } else {
#pragma unroll
            for (int k = 0; k < S; ++k) ub[u][k] = 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
          const int v = v0 + u;
          if (v >= X.nv) break;
          const bool upper = v >= X.nlo;
          if constexpr (GOP) {
            double d = 0.0;
#pragma unroll
            for (int k = 0; k < S; ++k) {
              const double tt = ua[k] * ub[u][k];
              d = (k == 0) ? tt : d + tt;
            }
            const double rr = d - bk[u];
            const double q = pk[u] + beta * rr;
            const int64_t slot = X.s_beg + 32 * (int64_t)v + lane;
            P.r_sell[slot] = rr;
            P.q_sell[slot] = q;
            if (!isfinite(q)) sums[2] = sums[2] + 1.0;
            if (upper) {
              P.r_up[ek[u]] = rr;
              P.q_up[ek[u]] = q;
              sums[0] = sums[0] + pk[u] * rr;
              sums[1] = sums[1] + rr * rr;
            }
            continue;
          }
          double w;
          if (FIXED) {
            w = 0.5 * pk[u];
          } else {
            double d = 0.0;
#pragma unroll
            for (int k = 0; k < S; ++k) {
              const double tt = ua[k] * ub[u][k];
              d = (k == 0) ? tt : d + tt;
            }
            const double rr = d - bk[u];
            const double q = pk[u] + beta * rr;
            w = 0.5 * q;
            if (upper) {
              sums[0] = sums[0] + pk[u] * rr;
              sums[1] = sums[1] + rr * rr;
              sums[2] = sums[2] + q * (rr + bk[u]);
            }
          }
          // skipped terms (w == 0, instances.cpp:47): x + (-0.0) == x exactly
#pragma unroll
          for (int k = 0; k < S; ++k) acc[k] = acc[k] + ((w != 0.0) ? w * ub[u][k] : -0.0);
        }
        st ^= 1;
      }
      if (!GOP && X.mine) {
#pragma unroll
        for (int k = 0; k < S; ++k) epi(X.a, k, acc[k], ua[k]);
      }
      if (!have_next) break;
      if (X.L == 0 && lane == 0 && XN.L > 0) issue(st, XN, 0);  // nothing was prefetched
      sl = sln;
      X = XN;
    }
    __syncwarp();
    if (lane == 0) {
      mbar_inval(bar);
      mbar_inval(bar + 1);
    }
  }
  __syncthreads();
}

// SELL-order copy of a multiplier given its edge-order array (null: none)
__device__ __forceinline__ const double* sell_of(const Params& P, const double* up) {
  if (!P.I.s_col) return nullptr;
  if (up == P.p_up) return P.p_sell;
  if (up == P.q_up) return P.q_sell;
  return nullptr;
}

template <int S, bool FIXED, class UA, class Epi>
__device__ __forceinline__ void row_pass_t(Ctx& c, const Params& P, const UA& U, int s_rt,
                                           const double* __restrict__ Pup,
                                           const double* __restrict__ Plo, double beta,
                                           double alpha, const double* cs, bool zero_init,
                                           double (&sums)[3], Epi& epi) {
  const DevPairs& I = P.I;
  constexpr int SR = S > 0 ? S : kSMax;
  constexpr int kPer = S > 0 ? kTileEntries / kGT : 1;  // entries per thread per batch
  const int s = S > 0 ? S : s_rt;
  const int g = threadIdx.x / kGT;   // tile group
  const int gt = threadIdx.x % kGT;  // thread within the group
  // double-buffered row pointers (tile t and t + kGroups)
  int64_t* const vlo0 = c.vlo + g * 2 * (kTileRows + 1);
  int64_t* const vup0 = c.vup + g * 2 * (kTileRows + 1);
  double* const tw = c.tw + g * kTileEntries;
  int32_t* const tcol = c.tcol + g * kTileEntries;
  double* const tterm = c.tterm + g * 4 * kTileEntries;
  const int nthr = (kGT / s) * s;  // phase-3 threads of the group; column = gt % s
  const int mycol = gt % s;
  publish_rows(c.t, U.base(), c.rl, c.rh, s);  // sharded: gathered rows -> every rank
  if constexpr (S >= 1 && S <= 4) {
    // many rows per CTA: the row-thread engine (same arithmetic, bit-exact)
    const double* Ps = sell_of(P, Pup);
    if constexpr (S == 3) {
      // (team-uniform condition: pad_rows3 synchronises the team)
      {
        if (Ps && P.pad) {  // 256-bit gathers from the padded copy
          pad_rows3(c, P, U);
          const UPad4 Up{P.pad};
          if constexpr (!FIXED) {
            if (I.s_b)
              row_pass_sell_async<S, false, true>(c, P, Up, Ps, beta, alpha, cs, zero_init, sums, epi);
            else
              row_pass_sell_async<S, false, false>(c, P, Up, Ps, beta, alpha, cs, zero_init, sums, epi);
          } else {
            row_pass_sell_async<S, true, false>(c, P, Up, Ps, beta, alpha, cs, zero_init, sums, epi);
          }
          return;
        }
      }
    }
    if (c.rh - c.rl >= kRtMinRows) {
      if (Ps && sell_aligned<S>(U.base())) {
        if constexpr (!FIXED) {
          if (I.s_b)
            row_pass_sell_async<S, false, true>(c, P, U, Ps, beta, alpha, cs, zero_init, sums, epi);
          else
            row_pass_sell_async<S, false, false>(c, P, U, Ps, beta, alpha, cs, zero_init, sums, epi);
        } else {
          row_pass_sell_async<S, true, false>(c, P, U, Ps, beta, alpha, cs, zero_init, sums, epi);
        }
        return;
      }
      // fixed q: cp.async-staged stream (measured 27% faster at H(23,2), s = 1);
      // q formed on the fly: register batches (the staged variant measured slower)
      if constexpr (FIXED)
        row_pass_rt_async<S, FIXED>(c, P, U, Pup, Plo, beta, alpha, cs, zero_init, sums, epi);
      else
        row_pass_rt<S, FIXED>(c, P, U, Pup, Plo, beta, alpha, cs, zero_init, sums, epi);
      return;
    }
  }

  auto vlo = [&](int buf) { return vlo0 + buf * (kTileRows + 1); };
  auto vup = [&](int buf) { return vup0 + buf * (kTileRows + 1); };
  // row pointers of `tile` -> buffer `buf` (visible after the next group_sync)
  auto load_ptrs = [&](int64_t tile, int buf) {
    if (tile < c.th) {
      if (c.cached) {  // shared-memory copies of the static structure
        const int q0 = c.ctr[tile - c.tl], q1 = c.ctr[tile - c.tl + 1];
        if (gt <= q1 - q0) {
          vlo(buf)[gt] = c.clo0 + c.crlo[q0 + gt];
          vup(buf)[gt] = c.cup0 + c.crup[q0 + gt];
        }
        return;
      }
      const int64_t q0 = __ldg(I.tile_row + tile), q1 = __ldg(I.tile_row + tile + 1);
      if (gt <= (int)(q1 - q0)) {
        vlo(buf)[gt] = __ldg(I.lo_ptr + q0 + gt);
        vup(buf)[gt] = __ldg(I.up_ptr + q0 + gt);
      }
    }
  };
  auto tile_nv = [&](int buf, int nr) -> int {
    return (int)((vlo(buf)[nr] - vlo(buf)[0]) + (vup(buf)[nr] - vup(buf)[0]));
  };

  // One batch of a thread's entries: indices -> stream loads -> gathers.
  struct Batch {
    int64_t bcol[kPer];
    double pq[kPer], bb[kPer];
    double ub[kPer][SR];
    int rowr[kPer];
    bool ok[kPer], up[kPer];
  };
  auto issue = [&](Batch& B, int buf, int nr, int nv, int vb0) {
    const int64_t* lo = vlo(buf);
    const int64_t* uq = vup(buf);
    const int64_t lo0 = lo[0], up0 = uq[0];
    int64_t idxs[kPer];
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      const int v = vb0 + gt + e * kGT;
      B.ok[e] = v < nv;
      int l = 0, h = nr - 1;  // last row with vstart(r) <= v
      while (l < h) {
        const int mid = (l + h + 1) >> 1;
        const int64_t vs = (lo[mid] - lo0) + (uq[mid] - up0);
        if (vs <= v) l = mid; else h = mid - 1;
      }
      B.rowr[e] = l;
      const int64_t off = v - ((lo[l] - lo0) + (uq[l] - up0));
      const int64_t nlo_r = lo[l + 1] - lo[l];
      B.up[e] = off >= nlo_r;
      idxs[e] = B.ok[e] ? (B.up[e] ? uq[l] + (off - nlo_r) : lo[l] + off) : 0;
    }
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      const int32_t* cp = (B.up[e] ? I.ej : I.lo_col) + idxs[e];
      const double* pp = (B.up[e] ? Pup : Plo) + idxs[e];
      const double* bp = B.up[e] ? I.b_up : I.b_lo;
      if (c.cached)
        B.bcol[e] = B.ok[e] ? c.ccol[B.up[e] ? c.cnlo + (int)(idxs[e] - c.cup0)
                                             : (int)(idxs[e] - c.clo0)]
                            : 0;
      else
        B.bcol[e] = __ldg(cp);
      B.pq[e] = __ldg(pp);
      B.bb[e] = (!FIXED && bp) ? __ldg(bp + idxs[e]) : 0.0;
    }
#pragma unroll
    for (int e = 0; e < kPer; ++e)
#pragma unroll
      for (int k = 0; k < SR; ++k) B.ub[e][k] = (B.ok[e] && k < s) ? U(B.bcol[e] * s + k) : 0.0;
  };
  // products w_v U(b_v, c) of a batch -> smem (after the previous fold)
  auto finish = [&](Batch& B, int64_t r0, int vb0) {
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      if (!B.ok[e]) continue;
      const int v = vb0 + gt + e * kGT;
      double w;
      if (FIXED) {
        w = 0.5 * B.pq[e];
      } else {
        const int64_t a = r0 + B.rowr[e];
        double d = 0.0;
#pragma unroll
        for (int k = 0; k < SR; ++k)
          if (k < s) {
            const double t = U(a * s + k) * B.ub[e][k];
            d = (k == 0) ? t : d + t;
          }
        const double rr = d - B.bb[e];
        const double q = B.pq[e] + beta * rr;
        w = 0.5 * q;
        if (B.up[e]) {
          sums[0] = sums[0] + B.pq[e] * rr;
          sums[1] = sums[1] + rr * rr;
          sums[2] = sums[2] + q * (rr + B.bb[e]);
        }
      }
      tw[v] = w;
      tcol[v] = (int32_t)B.bcol[e];
      // skipped terms (w == 0, instances.cpp:47) become -0.0: x + (-0.0) == x
      // exactly, so the fold is branch-free and still bit-identical
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < s) tterm[v * 4 + k] = (w != 0.0) ? w * B.ub[e][k] : -0.0;
    }
  };
  // phase 3: fold + epilogue, thread per (row, column)
  auto fold = [&](int buf, int64_t r0, int nr) {
    const int64_t* lo = vlo(buf);
    const int64_t* uq = vup(buf);
    const int64_t lo0 = lo[0], up0 = uq[0];
    if (gt < nthr) {
      for (int idx = gt; idx < nr * s; idx += nthr) {
        const int r = idx / s;
        const int64_t a = r0 + r;
        const double uown = U(a * s + mycol);
        double acc = 0.0;
        if (!zero_init) {
          acc = alpha * uown;
          if (cs) acc = acc - cs[mycol];
        }
        const int vb = (int)((lo[r] - lo0) + (uq[r] - up0));
        const int ve = (int)((lo[r + 1] - lo0) + (uq[r + 1] - up0));
        if (mycol < 4) {
          int v = vb;
          for (; v + 4 <= ve; v += 4) {
            const double t0 = tterm[v * 4 + mycol], t1 = tterm[(v + 1) * 4 + mycol];
            const double t2 = tterm[(v + 2) * 4 + mycol], t3 = tterm[(v + 3) * 4 + mycol];
            acc = acc + t0;
            acc = acc + t1;
            acc = acc + t2;
            acc = acc + t3;
          }
          for (; v < ve; ++v) acc = acc + tterm[v * 4 + mycol];
        } else {
          for (int v = vb; v < ve; ++v) {
            const double w = tw[v];
            if (w != 0.0) acc = acc + w * U((int64_t)tcol[v] * s + mycol);
          }
        }
        epi(a, mycol, acc, uown);
      }
    }
  };
  // a single row longer than a tile: chunked, fold carried in registers
  auto long_row = [&](int buf, int64_t a, int nv) {
    const int64_t* lo = vlo(buf);
    const int64_t* uq = vup(buf);
    const int64_t nlo_r = lo[1] - lo[0];
    double acc = 0.0, uown = 0.0;
    if (gt < s) {
      uown = U(a * s + gt);
      if (!zero_init) {
        acc = alpha * uown;
        if (cs) acc = acc - cs[gt];
      }
    }
    for (int v0 = 0; v0 < nv; v0 += kTileEntries) {
      const int cnt = min(kTileEntries, nv - v0);
      for (int v = gt; v < cnt; v += kGT) {
        const int64_t off = v0 + v;
        const bool upper = off >= nlo_r;
        const int64_t idx = upper ? uq[0] + (off - nlo_r) : lo[0] + off;
        const int64_t b = upper ? I.ej[idx] : I.lo_col[idx];
        const double pq = upper ? Pup[idx] : Plo[idx];
        double w;
        if (FIXED) {
          w = 0.5 * pq;
        } else {
          const double bb = upper ? (I.b_up ? I.b_up[idx] : 0.0) : (I.b_lo ? I.b_lo[idx] : 0.0);
          double d = 0.0;
          for (int k = 0; k < s; ++k) {
            const double t = U(a * s + k) * U(b * s + k);
            d = (k == 0) ? t : d + t;
          }
          const double rr = d - bb;
          const double q = pq + beta * rr;
          w = 0.5 * q;
          if (upper) {
            sums[0] = sums[0] + pq * rr;
            sums[1] = sums[1] + rr * rr;
            sums[2] = sums[2] + q * (rr + bb);
          }
        }
        tw[v] = w;
        tcol[v] = (int32_t)b;
      }
      group_sync(g);
      if (gt < s)
        for (int v = 0; v < cnt; ++v) {
          const double w = tw[v];
          if (w != 0.0) acc = acc + w * U((int64_t)tcol[v] * s + gt);
        }
      group_sync(g);
    }
    if (gt < s && gt < nthr) epi(a, gt, acc, uown);
  };

  // ---- the group's tiles: phase 2 (batched loads/gathers -> smem products,
  //      next tile's row pointers prefetched into the other buffer), then
  //      phase 3 (fold + epilogue).  Four groups per CTA overlap their
  //      latency chains.  (Holding the next tile's batch in registers across
  //      the fold was measured: ~1 KB of spills per thread, slower.)
  int64_t t = c.tl + g;
  int cur = 0;
  load_ptrs(t, cur);
  group_sync(g);
  while (t < c.th) {
    const int64_t r0 = __ldg(I.tile_row + t);
    const int nr = (int)(__ldg(I.tile_row + t + 1) - r0);
    const int nv = tile_nv(cur, nr);
    if (nv > kTileEntries) {
      long_row(cur, r0, nv);
      load_ptrs(t + kGroups, cur ^ 1);
      group_sync(g);
    } else {
      for (int vb0 = 0; vb0 < nv; vb0 += kPer * kGT) {  // one round unless S == 0
        Batch B;
        issue(B, cur, nr, nv, vb0);
        finish(B, r0, vb0);
      }
      load_ptrs(t + kGroups, cur ^ 1);
      group_sync(g);
      fold(cur, r0, nr);
      group_sync(g);
    }
    t += kGroups;
    cur ^= 1;
  }
  __syncthreads();
}

template <int S, bool FIXED, class Epi>
__device__ __forceinline__ void row_pass(Ctx& c, const Params& P, const double* __restrict__ U,
                                         int s_rt, const double* __restrict__ Pup,
                                         const double* __restrict__ Plo, double beta, double alpha,
                                         const double* cs, bool zero_init, double (&sums)[3],
                                         Epi& epi) {
  row_pass_t<S, FIXED>(c, P, UPlain{U}, s_rt, Pup, Plo, beta, alpha, cs, zero_init, sums, epi);
}

// Stage per-thread column partials (in each 128-thread group, thread
// gt < (kGT/s)*s owns column gt % s) into rs.part[w][base + c] as per-warp sums in fixed order, for a
// following team_reduce_smem.  Uses the tile smem as scratch (call after a pass).
__device__ __forceinline__ void stage_colsums(Ctx& c, int s, int base, double val) {
  double* scr = c.tw;
  const int tid = threadIdx.x;
  const int nthr = (kGT / s) * s;
  const int gt = tid % kGT;
  scr[tid] = gt < nthr ? val : 0.0;
  __syncthreads();
  if (c.lane < s) {
    double acc = 0.0;
    for (int l = 0; l < 32; ++l) {
      const int t = c.warp * 32 + l;
      const int tg = t % kGT;
      if (tg < nthr && tg % s == c.lane) acc = acc + scr[t];
    }
    c.rs.part[c.warp * kRedK + base + c.lane] = acc;
  }
  __syncthreads();
}

// GradientOperator build (sdp_instance.cpp:73-83): for every pair constraint
// r_k = U_a.U_b - b_k and q_k = p_k + beta r_k, written in edge order (upper
// entries) and lower order.  Upper entries accumulate p.r and r^2.
template <int S>
__device__ __forceinline__ void gradop_pass(Ctx& c, const Params& P, const double* __restrict__ U, int s_rt,
                            double beta, double (&sums)[2], bool* nonfinite) {
  const DevPairs& I = P.I;
  constexpr int SR = S > 0 ? S : kSMax;
  const int s = S > 0 ? S : s_rt;
  const int lane = c.lane;
  bool bad = false;
  publish_rows(c.t, U, c.rl, c.rh, s);
  for (int64_t a = c.rl + c.warp; a < c.rh; a += kWarps) {
    double ua[SR];
#pragma unroll
    for (int k = 0; k < SR; ++k) ua[k] = (k < s) ? U[a * s + k] : 0.0;
    const int64_t lo0 = I.lo_ptr[a], nlo = I.lo_ptr[a + 1] - lo0;
    const int64_t up0 = I.up_ptr[a], nup = I.up_ptr[a + 1] - up0;
    const int64_t tot = nlo + nup;
    for (int64_t e = lane; e < tot; e += 32) {
      const bool upper = e >= nlo;
      int64_t b, idx;
      double pq, bb = 0.0;
      if (!upper) {
        idx = lo0 + e;
        b = I.lo_col[idx];
        pq = P.p_lo[idx];
        if (I.b_lo) bb = I.b_lo[idx];
      } else {
        idx = up0 + (e - nlo);
        b = I.ej[idx];
        pq = P.p_up[idx];
        if (I.b_up) bb = I.b_up[idx];
      }
      double d = 0.0;
#pragma unroll
      for (int k = 0; k < SR; ++k)
        if (k < s) {
          const double t = ua[k] * U[b * s + k];
          d = (k == 0) ? t : d + t;
        }
      const double r = d - bb;
      const double q = pq + beta * r;
      if (!isfinite(q)) bad = true;
      if (P.q_sell) {
        const int64_t slot = I.s_off[a >> 5] + (a & 31) + 32 * e;
        P.r_sell[slot] = r;
        P.q_sell[slot] = q;
      }
      if (!upper) {
        P.r_lo[idx] = r;
        P.q_lo[idx] = q;
      } else {
        P.r_up[idx] = r;
        P.q_up[idx] = q;
        sums[0] = sums[0] + pq * r;
        sums[1] = sums[1] + r * r;
      }
    }
  }
  *nonfinite = bad;
}

// GradientOperator build on the SELL engine (single GPU, ranks 1..4, large
// instances): q and r in SELL order (the Lanczos / FW passes read q_sell) and
// in edge order; the lower-order copies are not written (the multiplier
// update re-gathers p_lo from p_up, bit-identical).  Returns false when the
// SELL path does not apply (the caller runs gradop_pass).
template <int S>
__device__ __forceinline__ bool gradop_sell(Ctx& c, const Params& P, const double* __restrict__ U,
                                            double beta, double (&sums)[2], bool* nonfinite) {
  if constexpr (S >= 1 && S <= 4) {
    const DevPairs& I = P.I;
    // team-uniform conditions only (pad_rows3 synchronises the team); the
    // SELL engine is correct for any row range
    if (!I.s_col || !P.q_sell || !P.r_sell || !sell_aligned<S>(U)) return false;
    double s3[3] = {0.0, 0.0, 0.0};
    auto none = [](int64_t, int, double, double) {};
    bool done = false;
    if constexpr (S == 3) {
      if (P.pad) {
        pad_rows3(c, P, UPlain{U});
        const UPad4 Up{P.pad};
        if (I.s_b)
          row_pass_sell_async<S, false, true, UPad4, decltype(none), true>(c, P, Up, P.p_sell, beta, 0.0,
                                                                            nullptr, true, s3, none);
        else
          row_pass_sell_async<S, false, false, UPad4, decltype(none), true>(c, P, Up, P.p_sell, beta, 0.0,
                                                                             nullptr, true, s3, none);
        done = true;
      }
    }
    if (!done) {
      if (I.s_b)
        row_pass_sell_async<S, false, true, UPlain, decltype(none), true>(c, P, UPlain{U}, P.p_sell, beta, 0.0,
                                                                           nullptr, true, s3, none);
      else
        row_pass_sell_async<S, false, false, UPlain, decltype(none), true>(c, P, UPlain{U}, P.p_sell, beta,
                                                                            0.0, nullptr, true, s3, none);
    }
    sums[0] = s3[0];
    sums[1] = s3[1];
    *nonfinite = s3[2] != 0.0;
    return true;
  }
  return false;
}

// ------------------------------------------------------------- map pass ---
// Thread per pair constraint k (edge order): d_k = U_{i_k}.U_{j_k} summed over
// columns in order (instances.cpp:27-35).  kUnroll constraints per thread are
// loaded before any is used so each thread keeps several gathers in flight.
enum MapMode : int { kMapPR = 0, kMapRR = 1, kMapOut = 2, kMapFWS = 3, kMapROut = 4 };
constexpr int kUnroll = 4;

// Row values of the gathered factor: either stored (U) or produced on the fly
// from the FISTA step y = (xt - gt/L) [/ nrm] (bit-identical to storing y).
struct RowSrc {
  const double* U = nullptr;
  const double* XT = nullptr;
  const double* GT = nullptr;
  double L = 1.0, nrm = 1.0;
  bool scale = false;
  __device__ __forceinline__ double at(int64_t o) const {
    if (U) return U[o];
    const double z = XT[o] - GT[o] / L;
    return scale ? z / nrm : z;
  }
  // row b (S values), vector loads: same values as at(b * S + k)
  template <int S>
  __device__ __forceinline__ void row(int64_t b, double (&o)[S]) const {
    if (U) {
      sell_row<S>(UPlain{U}, b, o);
      return;
    }
    double x[S], g[S];
    sell_row<S>(UPlain{XT}, b, x);
    sell_row<S>(UPlain{GT}, b, g);
#pragma unroll
    for (int k = 0; k < S; ++k) {
      const double z = x[k] - g[k] / L;
      o[k] = scale ? z / nrm : z;
    }
  }
};

// Map pass on the SELL copy (fast mode, one GPU).  Every pair constraint k is
// the upper entry of row i_k; the slices [0, I.s_up_slices) hold all of them
// (matrix completion: the rows i_k < n1; theta: every slice, entries below
// the slice's smallest lower-entry count are not streamed).  A warp owns one slice
// (global warp index, round robin over every CTA of the team), lane = row a:
// U_a is loaded once per row, the (column, multiplier, right-hand side)
// streams arrive by TMA bulk copies exactly as in row_pass_sell_async, and a
// constraint costs ONE gathered row instead of the edge-order pass's two plus
// its row-index stream.  d_k = sum_c U(i_k,c) U(j_k,c) in column order, so
// d_k and r_k are bit-identical to the edge-order pass (instances.cpp:27-35);
// only the order in which the per-thread partials p.r and r.r are formed
// differs (a fast-mode reduction order).  Ps: multiplier in SELL order, or
// null (r.r only).
template <int S, class UA>
__device__ __forceinline__ void map_pass_sell(Ctx& c, const Params& P, const UA& U,
                                              const double* __restrict__ Ps, double (&sums)[2]) {
  constexpr int B = 6;
  constexpr int kStageInts = B * 32;
  static_assert((1 + 4) * B * kThreads + 2 * kWarps <= kPassScratch, "map stages exceed the pass scratch");
  const DevPairs& I = P.I;
  const int lane = c.lane, warp = c.warp;
  int32_t* const colW = reinterpret_cast<int32_t*>(c.tw) + warp * 2 * kStageInts;
  double* const pW = c.tw + B * kThreads + warp * 2 * kStageInts;
  double* const bW = c.tw + 3 * B * kThreads + warp * 2 * kStageInts;
  unsigned long long* const bar = reinterpret_cast<unsigned long long*>(c.tw + 5 * B * kThreads) + warp * 2;
  const bool hp = Ps != nullptr;
  const bool hb = I.s_b != nullptr;  // theta: b = 0 on the pairs
  const int64_t nsl = I.s_up_slices;
  const int64_t gstride = (int64_t)c.t.size * kWarps;
  struct Sl {
    int64_t a, s_beg;
    int L, nv, nlo, vs;  // vs: first entry any lane needs (warp-uniform)
  };
  auto slice = [&](int64_t sl) {  // warp-collective
    Sl x;
    x.a = (sl << 5) + lane;
    const bool mine = x.a < I.n;
    x.s_beg = __ldg(I.s_off + sl);
    x.L = (int)((__ldg(I.s_off + sl + 1) - x.s_beg) >> 5);
    x.nv = mine ? __ldg(I.s_nv + x.a) : 0;
    x.nlo = mine ? __ldg(I.s_nlo + x.a) : 0;
    // lower entries come first in every row: entries below the smallest nlo
    // of the slice's rows (that have upper entries) are not streamed
    const unsigned cand = x.nv > x.nlo ? (unsigned)x.nlo : 0x7fffffffu;
    const unsigned vs = __reduce_min_sync(0xffffffffu, cand);
    x.vs = vs == 0x7fffffffu ? x.L : (int)vs;
    return x;
  };
  const unsigned long long pol = l2_evict_first();
  auto issue = [&](int st, const Sl& x, int v0) {  // lane 0 only
    const int ne = min(B, x.L - v0) * 32;
    const int64_t g = x.s_beg + (int64_t)v0 * 32;
    mbar_expect_tx(bar + st, (unsigned)ne * (4u + (hp ? 8u : 0u) + (hb ? 8u : 0u)));
    tma_load_1d(colW + st * kStageInts, I.s_col + g, ne * 4, bar + st, pol);
    if (hp) tma_load_1d(pW + st * kStageInts, Ps + g, ne * 8, bar + st, pol);
    if (hb) tma_load_1d(bW + st * kStageInts, I.s_b + g, ne * 8, bar + st, pol);
  };
  int64_t sl = (int64_t)c.t.rank * kWarps + warp;
  if (sl < nsl) {
    if (lane == 0) {
      mbar_init(bar, 1);
      mbar_init(bar + 1, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    Sl X = slice(sl);
    int st = 0;
    unsigned phase = 0;
    if (lane == 0 && X.vs < X.L) issue(0, X, X.vs);
    while (true) {
      double ua[S];
      if (X.nv > X.nlo) {
        sell_row<S>(U, X.a, ua);
      } else {
#pragma unroll
        for (int k = 0; k < S; ++k) ua[k] = 0.0;
      }
      const int64_t sln = sl + gstride;
      const bool have_next = sln < nsl;
      Sl XN{};
      if (have_next) XN = slice(sln);
#pragma unroll 1
      for (int v0 = X.vs; v0 < X.L; v0 += B) {
        if (lane == 0) {
          if (v0 + B < X.L)
            issue(st ^ 1, X, v0 + B);
          else if (have_next && XN.vs < XN.L)
            issue(st ^ 1, XN, XN.vs);
        }
        mbar_wait(bar + st, (phase >> st) & 1u);
        phase ^= 1u << st;
        int32_t bc[B];
        double pk[B], bk[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
          const int v = v0 + u;
          const bool ok = v < X.nv && v >= X.nlo;
          bc[u] = ok ? colW[st * kStageInts + u * 32 + lane] : 0;
          pk[u] = (ok && hp) ? pW[st * kStageInts + u * 32 + lane] : 0.0;
          bk[u] = (ok && hb) ? bW[st * kStageInts + u * 32 + lane] : 0.0;
        }
        __syncwarp();  // stage st is refilled by the next-but-one issue
        double ub[B][S];
#pragma unroll
        for (int u = 0; u < B; ++u) {
          const int v = v0 + u;
          if (v < X.nv && v >= X.nlo) {
            sell_row<S>(U, bc[u], ub[u]);
          } else {
#pragma unroll
            for (int k = 0; k < S; ++k) ub[u][k] = 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
          const int v = v0 + u;
          if (v >= X.nv) break;
          if (v < X.nlo) continue;
          double d = 0.0;
#pragma unroll
          for (int k = 0; k < S; ++k) {
            const double tt = ua[k] * ub[u][k];
            d = (k == 0) ? tt : d + tt;
          }
          const double r = d - bk[u];
          if (hp) sums[0] = sums[0] + pk[u] * r;
          sums[1] = sums[1] + r * r;
        }
        st ^= 1;
      }
      if (!have_next) break;
      if (X.vs >= X.L && lane == 0 && XN.vs < XN.L) issue(st, XN, XN.vs);  // nothing was prefetched
      sl = sln;
      X = XN;
    }
    __syncwarp();
    if (lane == 0) {
      mbar_inval(bar);
      mbar_inval(bar + 1);
    }
  }
  __syncthreads();
}

template <int S>
__device__ __forceinline__ void map_pass_src(Ctx& c, const Params& P, const RowSrc src, int s_rt,
                                          int mode, const double* __restrict__ pup, double* out,
                                          const double* __restrict__ ref, double (&sums)[2]) {
  const DevPairs& I = P.I;
  const int s = S > 0 ? S : s_rt;
  if (src.U) publish_rows(c.t, src.U, c.rl, c.rh, s);
  if constexpr (S == 3) {
    if (I.s_col && P.pad) {  // large single-GPU instance: 256-bit gathers from the padded copy
      if (src.U) {
        pad_rows3(c, P, UPlain{src.U});
      } else {
        pad_rows3(c, P, [&](int64_t o) { return src.at(o); });
      }
    }
  }
  const bool padded = S == 3 && I.s_col && P.pad;
  if constexpr (S >= 1 && S <= 4) {
    // one GPU (matrix completion; theta with little SELL padding): the
    // row-ordered pass over the SELL copy
    if ((mode == kMapPR || mode == kMapRR) && I.s_col && I.s_up_slices > 0) {
      const double* Ps = mode == kMapPR ? sell_of(P, pup) : nullptr;
      if (mode == kMapRR || Ps) {
        if (padded) {
          map_pass_sell<S>(c, P, UPad4{P.pad}, Ps, sums);
          return;
        }
        if (src.U && sell_aligned<S>(src.U)) {
          map_pass_sell<S>(c, P, UPlain{src.U}, Ps, sums);
          return;
        }
      }
    }
  }
  for (int64_t k0 = c.kl + threadIdx.x; k0 < c.kh; k0 += (int64_t)kThreads * kUnroll) {
    int64_t ii[kUnroll], jj[kUnroll];
    double pk[kUnroll], bk[kUnroll], rf[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t k = k0 + (int64_t)u * kThreads;
      const bool ok = k < c.kh;
      ii[u] = ok ? I.ei[k] : 0;
      jj[u] = ok ? I.ej[k] : 0;
      bk[u] = (ok && I.b_up) ? I.b_up[k] : 0.0;
      pk[u] = (ok && mode == kMapPR) ? pup[k] : 0.0;
      rf[u] = (ok && mode == kMapFWS) ? ref[k] : 0.0;
    }
    double d[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      double acc = 0.0;
      if constexpr (S > 0 && S <= 4) {
        // both rows with the widest aligned vector loads (sell_row)
        double ri[S], rj[S];
        if (padded) {
          sell_row<S>(UPad4{P.pad}, ii[u], ri);
          sell_row<S>(UPad4{P.pad}, jj[u], rj);
        } else {
          src.row<S>(ii[u], ri);
          src.row<S>(jj[u], rj);
        }
#pragma unroll
        for (int cc = 0; cc < S; ++cc) {
          const double t = ri[cc] * rj[cc];
          acc = (cc == 0) ? t : acc + t;
        }
      } else if (S > 0) {
#pragma unroll
        for (int cc = 0; cc < (S > 0 ? S : 1); ++cc) {
          const double t = src.at(ii[u] * s + cc) * src.at(jj[u] * s + cc);
          acc = (cc == 0) ? t : acc + t;
        }
      } else {
        for (int cc = 0; cc < s; ++cc) {
          const double t = src.at(ii[u] * s + cc) * src.at(jj[u] * s + cc);
          acc = (cc == 0) ? t : acc + t;
        }
      }
      d[u] = acc;
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t k = k0 + (int64_t)u * kThreads;
      if (k >= c.kh) continue;
      if (mode == kMapOut) {
        out[k] = d[u];
      } else if (mode == kMapROut) {
        out[k] = d[u] - bk[u];  // residual_of (algo: r[k] = map[k] - b[k])
      } else if (mode == kMapFWS) {
        const double t = (rf[u] + bk[u]) - d[u];
        sums[1] = sums[1] + t * t;
      } else {
        const double r = d[u] - bk[u];
        if (mode == kMapPR) sums[0] = sums[0] + pk[u] * r;
        sums[1] = sums[1] + r * r;
      }
    }
  }
}

template <int S>
__device__ __forceinline__ void map_pass(Ctx& c, const Params& P, const double* __restrict__ U,
                                         int s_rt, int mode, const double* __restrict__ pup,
                                         double* out, const double* __restrict__ ref,
                                         double (&sums)[2]) {
  RowSrc src;
  src.U = U;
  map_pass_src<S>(c, P, src, s_rt, mode, pup, out, ref, sums);
}

// -------------------------------------------------------- factor helpers ---
// Per-row loop over this CTA's rows with column statistics.  For S > 0 a
// thread owns whole rows (S column accumulators in registers); for the
// generic rank (S == 0) a warp owns a row and lane c owns column c, so the
// column accumulator is one register per lane.  f(o, k) returns the element
// value at offset o = a*s + k; colsum partials are staged into the reduction
// smem at [base, base + s).
template <int S, class F>
__device__ __forceinline__ void rows_colsum(Ctx& c, int s_rt, int base, F&& f) {
  const int s = S > 0 ? S : s_rt;
  if constexpr (S > 0) {
    double cs[S];
#pragma unroll
    for (int k = 0; k < S; ++k) cs[k] = 0.0;
    for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads) {
#pragma unroll
      for (int k = 0; k < S; ++k) cs[k] = cs[k] + f(a * S + k, k);
    }
#pragma unroll
    for (int k = 0; k < S; ++k) {
      const double x = warp_sum(cs[k]);
      if (c.lane == 0) c.rs.part[c.warp * kRedK + base + k] = x;
    }
  } else {
    double cs = 0.0;
    for (int64_t a = c.rl + c.warp; a < c.rh; a += kWarps)
      if (c.lane < s) cs = cs + f(a * s + c.lane, c.lane);
    if (c.lane < s) c.rs.part[c.warp * kRedK + base + c.lane] = cs;
  }
}

// Stage NV per-thread scalars (warp-summed) at [0, NV) of the reduction smem.
template <int NV>
__device__ __forceinline__ void stage_scalars(Ctx& c, const double (&v)[NV]) {
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const double x = warp_sum(v[k]);
    if (c.lane == 0) c.rs.part[c.warp * kRedK + k] = x;
  }
}

// Statistics of a factor needed before gathering it: theta needs ||U||_F^2
// (trace constraint) and the column sums (C = -ee').  On return (all CTAs):
// *nrm2 and dst_cs[0..s) (dst_cs may be c.cs or another smem array).
template <int S>
__device__ __forceinline__ void factor_stats_to(Ctx& c, const Params& P, const double* __restrict__ U,
                                             int s_rt, double* nrm2, double* dst_cs) {
  const int s = S > 0 ? S : s_rt;
  double sq = 0.0;
  rows_colsum<S>(c, s_rt, 1, [&](int64_t o, int) {
    const double u = U[o];
    sq = sq + u * u;
    return u;
  });
  double v[1] = {sq};
  stage_scalars<1>(c, v);
  team_reduce_smem(c.t, c.rs, 1 + s);
  *nrm2 = c.rs.out[0];
  if (threadIdx.x < (unsigned)s) dst_cs[threadIdx.x] = c.rs.out[1 + threadIdx.x];
  __syncthreads();
}
template <int S>
__device__ __forceinline__ void factor_stats(Ctx& c, const Params& P, const double* __restrict__ U,
                                             int s_rt, double* nrm2) {
  factor_stats_to<S>(c, P, U, s_rt, nrm2, c.cs);
}

// <CU, U> from the statistics: theta -sum_c cs_c^2, MC 0.5||U||^2, PR ||U||^2.
__device__ __forceinline__ double cdot_from_stats(const double* cs, const DevPairs& I, int s,
                                                  double nrm2) {
  if (is_pr(I)) return nrm2;  // C = I (instances.cpp:350)
  if (is_theta(I)) {
    double t = 0.0;
    for (int k = 0; k < s; ++k) t = t + cs[k] * cs[k];
    return -t;
  }
  return 0.5 * nrm2;
}
__device__ __forceinline__ double cdot_from_stats(const Ctx& c, const DevPairs& I, int s,
                                                  double nrm2) {
  return cdot_from_stats(c.cs, I, s, nrm2);
}

__device__ __forceinline__ double theta_alpha_or_half(const DevPairs& I, double qt) {
  return is_theta(I) ? qt : 0.5;
}

template <int S>
__device__ __forceinline__ void copy_rows(Ctx& c, const double* __restrict__ src, double* dst, int s_rt) {
  const int s = S > 0 ? S : s_rt;
  for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads)
    for (int k = 0; k < s; ++k) dst[a * s + k] = src[a * s + k];
}

// al_value (sdp_instance.cpp:50-60) at U: stats pass + map pass.
// Leaves c.cs = colsum(U) (theta).
template <int S>
__device__ __noinline__ bool al_value_dev(Ctx& c, const Params& P, const double* U, int s, const double* pup,
                             double p_trace, double beta, double* val, double* nrm2_out) {
  const DevPairs& I = P.I;
  double nrm2;
  factor_stats<S>(c, P, U, s, &nrm2);
  double sums[2] = {0.0, 0.0};
  if (is_pr(I)) {
    pr_forward(P, c.t.rank, c.t.size, c.X, UPlain{U}, s);
    c.t.sync();
    pr_map_combine(P, c.kl, c.kh, s, [&](int64_t k, double d) {
      const double r = d - I.b_up[k];
      sums[0] = sums[0] + pup[k] * r;
      sums[1] = sums[1] + r * r;
    });
  } else {
    map_pass<S>(c, P, U, s, kMapPR, pup, nullptr, nullptr, sums);
  }
  team_sum<2>(c.t, c.rs, sums);
  double pr = sums[0], rr = sums[1];
  if (is_theta(I)) {
    const double rt = nrm2 - I.b_trace;
    pr = pr + p_trace * rt;
    rr = rr + rt * rt;
  }
  const double cdot = cdot_from_stats(c, I, s, nrm2);
  const double v = cdot + pr + 0.5 * beta * rr;
  if (nrm2_out) *nrm2_out = nrm2;
  if (!isfinite(v)) {
    fail(c, kErrNumerical, kMsgAlValue);
    return false;
  }
  *val = v;
  return true;
}

inline __device__ __noinline__ double team_now(Ctx& c);  // solver.cuh

// ------------------------------------------------------------ ADAP-FISTA ---
struct Roles {
  int rep, yt, wp, best, x, y, xt, gt, yn, v, tmp;
};

struct FistaOut {
  int status;  // 0 success, 1 failure, 2 iter limit
  double L, psi_y, dist0;
  int iters;
};

// a of the curvature line search (adap_fista.cpp:49-50)
__device__ __forceinline__ double fista_a(double tau, double A, double L, double mu) {
  return (tau + sqrt(tau * tau + 4.0 * tau * A * (L - mu))) / (2.0 * (L - mu));
}

// fista_run on psi(u) = lambda L_beta(uu';p) + 0.5||u - W||^2 from x0 = W
// (adap_fista.cpp:14-103, adap_aipp.cpp:20-36).  On success buffers[yn]
// holds y and buffers[v] holds v.
//
// Team passes per iteration (no L-doubling): T2 value+gradient at x~ (row
// pass), T34 y+ and its map (y+ produced on the fly inside the map so no
// separate barrier), T5 gradient at y+ fused with the x update and the NEXT
// iteration's x~ and its statistics.  Three all-reduces per iteration.
template <int S>
__device__ __noinline__ bool fista_dev(Ctx& c, const Params& P, Roles& R, int s, double lambda,
                                       double L0, FistaOut& out) {
  const DevPairs& I = P.I;
  const Cfg& cf = P.cfg;
  const double mu = cf.fista_mu, chi = cf.fista_chi, sigma = cf.fista_sigma;
  const double beta = c.beta;
  const double pt = c.p_trace;
  const bool theta = is_theta(I);
  // y+ recomputed inside the map (saves a barrier) while the instance is
  // latency-bound; beyond ~2^20 factor entries the divisions would dominate
  const bool fuse_y = !is_pr(I) && !c.t.multi() && I.n * (int64_t)s <= (int64_t(1) << 20);
  double A = 0.0, tau = 1.0, L = L0;
  double* csx = c.cs + kSMax;  // column sums of x~ (kept apart from c.cs)
  prof_mark(c, P, kPfAipp);
  {
    const double* W = P.buf[R.wp];
    double* X = P.buf[R.x];
    double* Y = P.buf[R.y];
    for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads)
      for (int k = 0; k < s; ++k) {
        X[a * s + k] = W[a * s + k];
        Y[a * s + k] = W[a * s + k];
      }
    __syncthreads();
  }
  bool pre = false;  // x~ and its statistics already produced by T5
  double dd = 0.0, nt2 = 0.0;
  for (int it = 0;; ++it) {
    if (c.t.xfailed) {
      fail(c, kErrFabric, kMsgFabric);
      return false;
    }
    // time_limit inside long FISTA runs: the reference checks it per outer
    // iteration and per FW step (solver.cpp:141, hlr.cpp:106), which a single
    // HLR call of a large instance can overshoot by minutes; every 512
    // iterations the team reads CTA 0's clock and stops like an iteration limit
    if ((it & 511) == 511 && c.deadline < 1e300 && team_now(c) >= c.deadline) {
      c.timed_out = true;
      out.status = 2;
      out.L = L;
      out.iters = it;
      return true;
    }
    const int cap = cf.fista_max_iters > 0
                        ? cf.fista_max_iters
                        : 50 + (int)(10.0 * sqrt(L / mu) * log2(4.0 + L / L0));
    if (it >= cap) {
      out.status = 2;
      out.L = L;
      out.iters = it;
      return true;
    }
    double a, psi_t, psi_n, dsq, dist0, ny2;
    for (;;) {
      a = fista_a(tau, A, L, mu);
      const double* W = P.buf[R.wp];
      double* XT = P.buf[R.xt];
      if (!pre) {
        // ---- T1: x~ = (A y + a x)/(A + a); ||x~ - W||^2; ||x~||^2, colsum(x~)
        const double* X = P.buf[R.x];
        const double* Y = P.buf[R.y];
        double sc[2] = {0.0, 0.0};
        rows_colsum<S>(c, s, 2, [&](int64_t o, int) {
          const double xt = (A * Y[o] + a * X[o]) / (A + a);
          XT[o] = xt;
          const double dv = xt - W[o];
          sc[0] = sc[0] + dv * dv;
          sc[1] = sc[1] + xt * xt;
          return xt;
        });
        stage_scalars<2>(c, sc);
        team_reduce_smem(c.t, c.rs, 2 + s);
        dd = c.rs.out[0];
        nt2 = c.rs.out[1];
        if (threadIdx.x < (unsigned)s) csx[threadIdx.x] = c.rs.out[2 + threadIdx.x];
        __syncthreads();
        prof_mark(c, P, kPfT1);
      }
      pre = false;
      // ---- T2: value_and_gradient at x~ (sdp_instance.cpp:115-127) fused with
      //          the psi gradient and the projection norm
      double rt = 0.0, qt = 0.0;
      if (theta) {
        rt = nt2 - I.b_trace;
        qt = pt + beta * rt;
      }
      double* GT = P.buf[R.gt];
      double nrmz;
      {
        double hU = 0.0, zz = 0.0;
        auto epi = [&](int64_t row, int cc, double h, double xo) {
          const int64_t o = row * s + cc;
          hU = hU + h * xo;
          const double g = 2.0 * h;
          const double gt = lambda * g + (xo - W[o]);
          GT[o] = gt;
          const double z = xo - gt / L;
          zz = zz + z * z;
        };
        double sums[3] = {0.0, 0.0, 0.0};
        if (is_pr(I)) {
          pr_forward(P, c.t.rank, c.t.size, c.X, UPlain{XT}, s);
          c.t.sync();
          pr_inverse<false>(P, c.t.rank, c.t.size, c.X, s, nullptr, P.p_up, beta, sums);
          c.t.sync();
          pr_combine(P, c.rl, c.rh, UPlain{XT}, s, true, epi);
        } else {
          row_pass<S, false>(c, P, XT, s, P.p_up, P.p_lo, beta, theta_alpha_or_half(I, qt),
                             theta ? csx : nullptr, false, sums, epi);
        }
        double v[5] = {hU, sums[0], sums[1], sums[2], zz};
        team_sum<5>(c.t, c.rs, v);
        prof_mark(c, P, kPfT2);
        double pr = v[1], rr = v[2], qrb = v[3];
        zz = v[4];
        if (theta) {
          pr = pr + pt * rt;
          rr = rr + rt * rt;
          qrb = qrb + qt * (rt + I.b_trace);
        }
        const double cdot = v[0] - qrb;
        const double val = cdot + pr + 0.5 * beta * rr;
        if (!isfinite(val)) {
          fail(c, kErrNumerical, kMsgAlValGrad);
          return false;
        }
        psi_t = lambda * val + 0.5 * dd;
        // project_ball (sdp_instance.cpp:94-99)
        if (!isfinite(zz)) {
          fail(c, kErrInput, kMsgProjectBall);
          return false;
        }
        nrmz = sqrt(zz);
      }
      const bool scale = !(nrmz <= 1.0);
      // ---- T34: y+ (written for the row part, produced on the fly for the
      //           map); ||y-W||^2, ||y-x~||^2, <g~, y-x~>, ||y||^2, colsum(y)
      {
        double* YN = P.buf[R.yn];
        double v3[4] = {0.0, 0.0, 0.0, 0.0};
        rows_colsum<S>(c, s, 6, [&](int64_t o, int) {
          const double xt = XT[o], gt = GT[o];
          const double z = xt - gt / L;
          const double y = scale ? z / nrmz : z;
          YN[o] = y;
          const double d0 = y - W[o];
          const double dx = y - xt;
          v3[0] = v3[0] + d0 * d0;
          v3[1] = v3[1] + dx * dx;
          v3[2] = v3[2] + gt * dx;
          v3[3] = v3[3] + y * y;
          return y;
        });
        RowSrc src;
        if (fuse_y) {
          src.XT = XT;
          src.GT = GT;
          src.L = L;
          src.nrm = nrmz;
          src.scale = scale;
        } else {
          c.t.sync();  // y+ complete before it is gathered
          src.U = YN;
        }
        double ms[2] = {0.0, 0.0};
        if (is_pr(I)) {
          pr_forward(P, c.t.rank, c.t.size, c.X, UPlain{YN}, s);
          c.t.sync();
          pr_map_combine(P, c.kl, c.kh, s, [&](int64_t k, double d) {
            const double r = d - I.b_up[k];
            ms[0] = ms[0] + P.p_up[k] * r;
            ms[1] = ms[1] + r * r;
          });
        } else {
          map_pass_src<S>(c, P, src, s, kMapPR, P.p_up, nullptr, nullptr, ms);
        }
        double v[6] = {v3[0], v3[1], v3[2], v3[3], ms[0], ms[1]};
        stage_scalars<6>(c, v);
        team_reduce_smem(c.t, c.rs, 6 + s);
        prof_mark(c, P, kPfT34);
        dist0 = c.rs.out[0];
        dsq = c.rs.out[1];
        const double lin_s = c.rs.out[2];
        ny2 = c.rs.out[3];
        double pr = c.rs.out[4], rr = c.rs.out[5];
        if (threadIdx.x < (unsigned)s) c.cs[threadIdx.x] = c.rs.out[6 + threadIdx.x];
        __syncthreads();
        if (theta) {
          const double r2 = ny2 - I.b_trace;
          pr = pr + pt * r2;
          rr = rr + r2 * r2;
        }
        const double cdot = cdot_from_stats(c, I, s, ny2);
        const double val = cdot + pr + 0.5 * beta * rr;
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
      return true;
    }
    // ---- T5: gradient at y+ -> v; x update (adap_fista.cpp:68-71, 86-87);
    //          next x~ with the same L and its statistics
    {
      const double* W = P.buf[R.wp];
      double* XT = P.buf[R.xt];
      const double* GT = P.buf[R.gt];
      const double* YN = P.buf[R.yn];
      double* X = P.buf[R.x];
      double* V = P.buf[R.v];
      double qt = 0.0;
      if (theta) qt = pt + beta * (ny2 - I.b_trace);
      const double Lm = L - mu, mua = mu * a, tam = tau - a * mu;
      const double an = fista_a(tau, A_next, L, mu);
      constexpr int CS = (S > 0 && S <= 4) ? S : 1;  // per-column sums of the next x~
      double vv = 0.0, ddn = 0.0, ntn = 0.0, csn[CS];
#pragma unroll
      for (int k = 0; k < CS; ++k) csn[k] = 0.0;
      auto epi = [&](int64_t row, int cc, double h, double yo) {
        {
          const int64_t o = row * s + cc;
          const double g = 2.0 * h;
          const double gy = lambda * g + (yo - W[o]);
          const double xt = XT[o];
          const double vt = gy - GT[o] + L * (xt - yo);
          V[o] = vt;
          vv = vv + vt * vt;
          const double sd = Lm * (xt - yo);
          const double xn = (mua * yo + tam * X[o] - a * sd) / tau;
          X[o] = xn;
          const double xtn = (A_next * yo + an * xn) / (A_next + an);
          XT[o] = xtn;
          const double dv = xtn - W[o];
          ddn = ddn + dv * dv;
          ntn = ntn + xtn * xtn;
          if constexpr (CS > 1) {
#pragma unroll
            for (int k = 0; k < CS; ++k)
              if (k == cc) csn[k] = csn[k] + xtn;
          } else {
            csn[0] = csn[0] + xtn;
          }
        }
      };
      double sums[3] = {0.0, 0.0, 0.0};
      if (is_pr(I)) {
        // spectra of y+ are still cached from T34
        pr_inverse<false>(P, c.t.rank, c.t.size, c.X, s, nullptr, P.p_up, beta, sums);
        c.t.sync();
        pr_combine(P, c.rl, c.rh, UPlain{YN}, s, true, epi);
      } else {
        row_pass<S, false>(c, P, YN, s, P.p_up, P.p_lo, beta, theta_alpha_or_half(I, qt),
                           theta ? c.cs : nullptr, false, sums, epi);
      }
      double v[3] = {vv, ddn, ntn};
      stage_scalars<3>(c, v);
      if constexpr (S > 0 && S <= 4) {
        // any thread may hold any column (engine-independent staging)
#pragma unroll
        for (int k = 0; k < S; ++k) {
          const double x = warp_sum(csn[k]);
          if (c.lane == 0) c.rs.part[c.warp * kRedK + 3 + k] = x;
        }
      } else {
        stage_colsums(c, s, 3, csn[0]);
      }
      team_reduce_smem(c.t, c.rs, 3 + s);
      prof_mark(c, P, kPfT5);
      vv = c.rs.out[0];
      dd = c.rs.out[1];
      nt2 = c.rs.out[2];
      if (threadIdx.x < (unsigned)s) csx[threadIdx.x] = c.rs.out[3 + threadIdx.x];
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
        return true;
      }
    }
    A = A_next;
    const int tmp = R.y;
    R.y = R.yn;
    R.yn = tmp;
    pre = true;
  }
}

// ------------------------------------------------------------- ADAP-AIPP ---
struct AippOut {
  int status;  // 0 converged, 1 iter limit, 2 lambda underflow
  int w_buf;   // buffer holding the returned W
  double R_norm, g_value, lambda;
  int prox_iters, fista_iters;
};

// aipp_run (adap_aipp.cpp:40-116) from buffers[R.yt]; rho given.
template <int S>
__device__ __noinline__ bool aipp_dev(Ctx& c, const Params& P, Roles& R, int s, double rho, AippOut& out) {
  const Cfg& cf = P.cfg;
  double lambda = cf.aipp_lambda0, M_bar = 1.0;
  // W_prev = W_init
  copy_rows<S>(c, P.buf[R.yt], P.buf[R.wp], s);
  __syncthreads();
  double g_prev;
  if (!al_value_dev<S>(c, P, P.buf[R.wp], s, P.p_up, c.p_trace, c.beta, &g_prev, nullptr))
    return false;
  out.w_buf = R.yt;  // out.W = W_init
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
      FistaOut fo;
      if (!fista_dev<S>(c, P, R, s, lambda, fmax(1.0, M_bar / 2.0), fo)) return false;
      out.fista_iters += fo.iters;
      if (c.timed_out) {  // time_limit reached inside FISTA: unwind like an iteration limit
        out.status = 2;
        if (have_best) out.w_buf = R.best;
        return true;
      }
      if (P.cfg.trace >= 2 && P.trace && c.t.rank == 0 && threadIdx.x == 0) {
        // debug (cfg.trace >= 2): one event per fista() call, kind 9 (L0 in
        // eps_inner, status in rank, iterations in outer_iter, final L in gap,
        // psi_y in theta, the prox step lambda in fw_alpha)
        const int i = *P.trace_count;
        if (i < P.trace_cap) {
          TraceEv ev{};
          ev.kind = 9;
          ev.eps_inner = fmax(1.0, M_bar / 2.0);
          ev.rank = fo.status;
          ev.outer_iter = fo.iters;
          ev.gap = fo.L;
          ev.theta = fo.status == 2 ? 0.0 : fo.psi_y;
          ev.fw_alpha = lambda;
          P.trace[i] = ev;
        }
        *P.trace_count = i + 1;
      }
      if (fo.status == 0) {
        const double step_sq = fo.dist0;
        g_W = (fo.psi_y - 0.5 * step_sq) / lambda;
        const double descent = lambda * g_prev - (lambda * g_W + 0.5 * step_sq);
        // vw = <v, W_prev - y>, and ||(v + W_prev - y)/lambda||^2
        const double* V = P.buf[R.v];
        const double* Wp = P.buf[R.wp];
        const double* Yn = P.buf[R.yn];
        double v[2] = {0.0, 0.0};
        for (int64_t a = c.rl + threadIdx.x; a < c.rh; a += kThreads)
          for (int k = 0; k < s; ++k) {
            const int64_t o = a * s + k;
            const double vt = V[o], wp = Wp[o], y = Yn[o];
            v[0] = v[0] + vt * (wp - y);
            const double r = (vt + wp - y) / lambda;
            v[1] = v[1] + r * r;
          }
        team_sum<2>(c.t, c.rs, v);
        prof_mark(c, P, kPfAipp);
        if (descent >= v[0]) {
          L_out = fo.L;
          Rn2 = v[1];
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
      copy_rows<S>(c, P.buf[R.yn], P.buf[R.best], s);
      have_best = true;
      out.w_buf = R.best;
      out.R_norm = R_norm;
      out.g_value = g_W;
      out.lambda = lambda;
    }
    // W_prev = W
    const int tmp = R.wp;
    R.wp = R.yn;
    R.yn = tmp;
    g_prev = g_W;
    __syncthreads();
  }
  out.status = 1;
  return true;
}

}  // namespace hallar
