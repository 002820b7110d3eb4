// Per-launch setup shared by the persistent kernels (hallar_kernel in
// capi.cu, hallar_parity_kernel in parity_kernel.cu): team identity, the
// dynamic shared-memory carve-up, row / tile / constraint ownership and the
// small-instance structure cache.
#pragma once

#include "device.cuh"

namespace hallar {

__device__ __forceinline__ void setup_ctx(Ctx& c, const Params& P, unsigned char* smem_raw) {
  c.t.rank = P.fab.me * gridDim.x + blockIdx.x;  // global CTA index over all ranks
  c.t.size = P.fab.world * gridDim.x;
  c.t.lrank = blockIdx.x;
  c.t.lsize = gridDim.x;
  c.t.fab = &P.fab;
  c.t.mw = P.fab.world > 1;
  c.t.bar = P.bar;
  c.t.slots = P.slots;
  c.t.epoch = 0;
  c.t.parity = 0;
  c.warp = threadIdx.x >> 5;
  c.lane = threadIdx.x & 31;
  double* sm = reinterpret_cast<double*>(smem_raw);
  c.rs.part = sm;
  sm += kWarps * kRedK;
  c.rs.out = sm;
  sm += kRedK;
  {
    // one pass scratch: tile-engine arrays, or the phase-retrieval transform
    double* base = sm;
    c.X = reinterpret_cast<double2*>(base);
    c.tw = sm;
    sm += kGroups * kTileEntries;
    c.tterm = sm;
    sm += kGroups * 4 * kTileEntries;
    c.vlo = reinterpret_cast<int64_t*>(sm);
    sm += 2 * kGroups * (kTileRows + 1);
    c.vup = reinterpret_cast<int64_t*>(sm);
    sm += 2 * kGroups * (kTileRows + 1);
    c.tcol = reinterpret_cast<int32_t*>(sm);
    sm = base + P.pass_scratch;  // tile arrays (pairs) or one transform (phase retrieval)
  }
  c.cs = sm;
  sm += 2 * kSMax;
  c.H = sm;
  sm += kHLd * kHLd;
  c.JA = sm;
  sm += 32 * 32;
  c.JV = sm;
  sm += 32 * 32;
  c.E = sm;
  sm += 32 * 32;
  c.ev = sm;
  sm += 32;
  c.jcs = sm;
  sm += 32;
  c.hh = sm;
  sm += 32;
  c.hh2 = sm;
  sm += 32;
  c.vsum = sm;
  sm += 64;
  int* ip = reinterpret_cast<int*>(sm);
  c.col = ip;
  ip += 40;
  c.jpq = ip;
  ip += 40;
  c.ccol = ip;
  ip += kCacheEnt;
  c.crlo = ip;
  ip += kCacheRows + 1;
  c.crup = ip;
  ip += kCacheRows + 1;
  c.ctr = ip;
  if (P.I.family == kPhaseret) {
    c.tl = c.th = 0;
    c.rl = P.I.n * c.t.rank / c.t.size;
    c.rh = P.I.n * (c.t.rank + 1) / c.t.size;
  } else {
    if (P.I.split_w >= 0 && P.fab.world == 1) {
      // cost-balanced split: CTA r starts at the first tile whose prefix cost
      // (entries of both CSR halves + split_w per row) reaches r/size of the
      // total.  Equal tile counts leave CTAs of short-row regions with up to 2x
      // the rows and 1.3x the entries of others at matrix completion (tiles cap
      // at 512 entries), and every pass ends at a team barrier.
      const int64_t* tr = P.I.tile_row;
      const int64_t nt = P.I.ntiles, w = P.I.split_w;
      auto cost = [&](int64_t t) {
        const int64_t r = tr[t];
        return P.I.up_ptr[r] + P.I.lo_ptr[r] + w * r;
      };
      const int64_t total = cost(nt);
      auto first_at = [&](int rank) -> int64_t {
        if (rank <= 0) return 0;
        if (rank >= c.t.size) return nt;
        const int64_t target = (int64_t)((__int128)total * rank / c.t.size);
        int64_t lo = 0, hi = nt;  // smallest t with cost(t) >= target
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (cost(mid) < target) lo = mid + 1;
          else hi = mid;
        }
        return lo;
      };
      c.tl = first_at(c.t.rank);
      c.th = first_at(c.t.rank + 1);
    } else {
      c.tl = P.I.ntiles * c.t.rank / c.t.size;
      c.th = P.I.ntiles * (c.t.rank + 1) / c.t.size;
    }
    c.rl = P.I.tile_row[c.tl];
    c.rh = P.I.tile_row[c.th];
  }
  if (P.I.family != kPhaseret) {
    // static structure of the CTA's rows -> shared memory (small instances)
    const int64_t lo0 = P.I.lo_ptr[c.rl], up0 = P.I.up_ptr[c.rl];
    const int64_t nlo = P.I.lo_ptr[c.rh] - lo0, nup = P.I.up_ptr[c.rh] - up0;
    c.cached = c.th - c.tl <= kCacheTiles && c.rh - c.rl <= kCacheRows &&
               nlo + nup <= kCacheEnt;
    if (c.cached) {
      c.clo0 = lo0;
      c.cup0 = up0;
      c.cnlo = (int32_t)nlo;
      for (int64_t r = threadIdx.x; r <= c.rh - c.rl; r += kThreads) {
        c.crlo[r] = (int32_t)(P.I.lo_ptr[c.rl + r] - lo0);
        c.crup[r] = (int32_t)(P.I.up_ptr[c.rl + r] - up0);
      }
      for (int64_t t = threadIdx.x; t <= c.th - c.tl; t += kThreads)
        c.ctr[t] = (int32_t)(P.I.tile_row[c.tl + t] - c.rl);
      for (int64_t e = threadIdx.x; e < nlo; e += kThreads) c.ccol[e] = P.I.lo_col[lo0 + e];
      for (int64_t e = threadIdx.x; e < nup; e += kThreads) c.ccol[nlo + e] = P.I.ej[up0 + e];
    }
    __syncthreads();
  }
  if (P.fab.world > 1) {
    // row-owner sharding: a CTA owns the upper (edge-order) entries of its rows
    c.kl = P.I.up_ptr[c.rl];
    c.kh = P.I.up_ptr[c.rh];
  } else {
    c.kl = P.I.np * c.t.rank / c.t.size;
    c.kh = P.I.np * (c.t.rank + 1) / c.t.size;
  }
}

// dynamic shared memory: fixed solver state + the pass scratch of the family
constexpr size_t smem_bytes(int pass_scratch) {
  return sizeof(double) * (kWarps * kRedK + kRedK + pass_scratch + 2 * kSMax + kHLd * kHLd +
                           3 * 32 * 32 + 4 * 32 + 64) +
         sizeof(int) * (80 + kCacheInts);
}
constexpr size_t kSmemBytes = smem_bytes(kPassScratch);  // the largest (attribute, occupancy)

}  // namespace hallar
