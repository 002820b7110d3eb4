// Team = every CTA of the persistent launch(es) working on one solve.  On one
// GPU the team is one cooperative launch; a row-sharded solve
// spans `world` launches, one per GPU, that address each other's memory
// through peer pointers (NVLink / NVSwitch).  Provides a grid barrier and a
// deterministic all-reduce: each CTA reduces in a fixed tree, writes one
// partial per value, and after the barrier EVERY CTA sums the partials in the
// same rank order (per GPU, then per rank) — so all CTAs hold bit-identical
// scalars and take the solver's control-flow decisions redundantly without
// any broadcast and without host round-trips.
#pragma once

#include "common.cuh"

namespace hallar {

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long team_clock_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double warp_sum(double v) {
  // xor butterfly: every lane ends with the same (commutative) sum
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

struct Team {
  int rank = 0, size = 1;    // global CTA index / count over all ranks (work splits)
  int lrank = 0, lsize = 1;  // CTA index / count inside this launch
  unsigned long long* bar = nullptr;
  unsigned long long epoch = 0;
  double* slots = nullptr;
  int parity = 0;
  const Fabric* fab = nullptr;
  unsigned long long xepoch = 0;
  bool xfailed = false;  // a rendezvous timed out (same value in every CTA of the rank)

  bool mw = false;  // world > 1 (cached: the fabric lives in parameter space)
  __device__ __forceinline__ bool multi() const { return mw; }

  // barrier over the CTAs of this launch
  __device__ void lsync() {
    __syncthreads();
    if (threadIdx.x == 0) {
      epoch += 1;
      const unsigned long long target = epoch * (unsigned long long)lsize;
      // release-add publishes this CTA's writes (ordered before by bar.sync);
      // system scope when peers on other GPUs read what this CTA wrote
      if (multi())
        asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(bar), "l"(1ULL) : "memory");
      else
        asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(bar), "l"(1ULL) : "memory");
      // acquire poll: each ld.acquire.gpu invalidates this SM's L1 (CCTL.IVALL),
      // so no trailing fence is needed before the CTA reads other CTAs' data
      while (ld_acquire_u64(bar) < target) {
      }
    }
    __syncthreads();
  }

  // rank-level rendezvous, executed by CTA 0 of each launch between two local
  // barriers.  A peer that never arrives (e.g. launches that could not be
  // co-resident) trips the timeout: the error flag is raised and the solve
  // unwinds instead of hanging the device.
  __device__ void xsync() {
    lsync();
    if (lrank == 0 && threadIdx.x == 0) {
      xepoch += 1;
      for (int p = 0; p < fab->world; ++p)
        asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(fab->xbar[p]), "l"(1ULL)
                     : "memory");
      const unsigned long long target = xepoch * (unsigned long long)fab->world;
      const unsigned long long t0 = team_clock_ns();
      if (!*(volatile int*)fab->xerr)
        while (ld_acquire_sys_u64(fab->xbar[fab->me]) < target) {
          if (team_clock_ns() - t0 > fab->timeout_ns) {
            *(volatile int*)fab->xerr = 1;
            break;
          }
        }
    }
    lsync();
    xfailed = *(volatile int*)fab->xerr != 0;
  }

  __device__ void sync() {
    if (multi()) xsync();
    else lsync();
  }

};

// Shared-memory scratch for reductions.
struct RedSmem {
  double* part;  // [kWarps][kRedK]
  double* out;   // [kRedK]
};

// Combine per-warp partials part[w][k] (k < K) across the block and the team;
// result in rs.out[k] (every thread of every CTA sees the same values).
__device__ __forceinline__ void team_reduce_smem(Team& t, RedSmem& rs, int K) {
  __syncthreads();
  double* mine = t.slots + ((size_t)t.parity * t.lsize + t.lrank) * kRedK;
  for (int k = threadIdx.x; k < K; k += kThreads) {
    double s = rs.part[k];
    for (int w = 1; w < kWarps; ++w) s = s + rs.part[w * kRedK + k];
    mine[k] = s;
  }
  t.lsync();
  const double* base = t.slots + (size_t)t.parity * t.lsize * kRedK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = warp; k < K; k += kWarps) {
    // all partial loads issued before the (fixed-order) sum: one L2 round trip
    double v[kMaxTeam / 32];
#pragma unroll
    for (int q = 0; q < kMaxTeam / 32; ++q) {
      const int r = lane + 32 * q;
      v[q] = (r < t.lsize) ? __ldcg(base + (size_t)r * kRedK + k) : 0.0;
    }
    double acc = v[0];
#pragma unroll
    for (int q = 1; q < kMaxTeam / 32; ++q) acc = acc + v[q];
    acc = warp_sum(acc);
    if (lane == 0) rs.out[k] = acc;
  }
  if (t.multi()) {
    // per-rank sums -> every rank's slot table, then a fixed-order sum over ranks
    __syncthreads();
    const Fabric& f = *t.fab;
    if (t.lrank == 0)
      for (int k = threadIdx.x; k < K; k += kThreads)
        for (int p = 0; p < f.world; ++p)
          f.xslots[p][((size_t)t.parity * kMaxWorld + f.me) * kRedK + k] = rs.out[k];
    t.xsync();
    const double* xs = f.xslots[f.me] + (size_t)t.parity * kMaxWorld * kRedK;
    __syncthreads();
    for (int k = threadIdx.x; k < K; k += kThreads) {
      double acc = __ldcv(xs + k);
      for (int p = 1; p < f.world; ++p) acc = acc + __ldcv(xs + (size_t)p * kRedK + k);
      rs.out[k] = acc;
    }
  }
  t.parity ^= 1;
  __syncthreads();
}

// All-reduce of K per-thread values (compile-time K).
template <int K>
__device__ __forceinline__ void team_sum(Team& t, RedSmem& rs, double (&v)[K]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double x = warp_sum(v[k]);
    if (lane == 0) rs.part[warp * kRedK + k] = x;
  }
  team_reduce_smem(t, rs, K);
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = rs.out[k];
}

// All-reduce where lane i of each warp holds the partial of value i (i < K <= 32).
__device__ __forceinline__ void team_sum_lanes(Team& t, RedSmem& rs, double mine, int K) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane < K) rs.part[warp * kRedK + lane] = mine;
  team_reduce_smem(t, rs, K);
}

// Row-sharded solve: push this CTA's rows [rl, rh) of a replicated factor
// buffer (stride s doubles per row) into every peer's copy, then a team
// barrier so the gathers that follow see every row.  Buffers outside the
// replicated arena (read-only inputs uploaded to every rank) need no push.
// One GPU: no-op.
__device__ __forceinline__ void publish_rows(Team& t, const double* buf, int64_t rl, int64_t rh,
                                             int s) {
  if (!t.multi()) return;
  const Fabric& f = *t.fab;
  const double* mine = f.arena[f.me];
  const int64_t off = buf - mine;
  if (off >= 0 && off < f.arena_len) {
    const int64_t lo = rl * s, hi = rh * s;
    for (int p = 0; p < f.world; ++p) {
      if (p == f.me) continue;
      double* dst = f.arena[p] + off;
      for (int64_t o = lo + threadIdx.x; o < hi; o += kThreads) dst[o] = buf[o];
    }
  }
  t.sync();
}

}  // namespace hallar
