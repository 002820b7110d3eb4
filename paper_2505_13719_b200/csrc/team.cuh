// Team = every CTA of one persistent cooperative launch.  Provides a grid
// barrier and deterministic all-reduce: each CTA reduces in a fixed tree,
// writes one partial per value, and after the barrier EVERY CTA sums the
// partials in the same rank order — so all CTAs hold bit-identical scalars
// and can take the solver's control-flow decisions redundantly without any
// broadcast (and without host round-trips).
#pragma once

#include "common.cuh"

namespace hallar {

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
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
  int rank = 0, size = 1;
  unsigned long long* bar = nullptr;
  unsigned long long epoch = 0;
  double* slots = nullptr;
  int parity = 0;

  __device__ void sync() {
    __syncthreads();
    if (threadIdx.x == 0) {
      epoch += 1;
      const unsigned long long target = epoch * (unsigned long long)size;
      // release-add publishes this CTA's writes (ordered before by bar.sync)
      asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(bar), "l"(1ULL) : "memory");
      // acquire poll: each ld.acquire.gpu invalidates this SM's L1 (CCTL.IVALL),
      // so no trailing fence is needed before the CTA reads other CTAs' data
      while (ld_acquire_u64(bar) < target) {
      }
    }
    __syncthreads();
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
  double* mine = t.slots + ((size_t)t.parity * t.size + t.rank) * kRedK;
  for (int k = threadIdx.x; k < K; k += kThreads) {
    double s = rs.part[k];
    for (int w = 1; w < kWarps; ++w) s = s + rs.part[w * kRedK + k];
    mine[k] = s;
  }
  t.sync();
  const double* base = t.slots + (size_t)t.parity * t.size * kRedK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = warp; k < K; k += kWarps) {
    // all partial loads issued before the (fixed-order) sum: one L2 round trip
    double v[kMaxTeam / 32];
#pragma unroll
    for (int q = 0; q < kMaxTeam / 32; ++q) {
      const int r = lane + 32 * q;
      v[q] = (r < t.size) ? __ldcg(base + (size_t)r * kRedK + k) : 0.0;
    }
    double acc = v[0];
#pragma unroll
    for (int q = 1; q < kMaxTeam / 32; ++q) acc = acc + v[q];
    acc = warp_sum(acc);
    if (lane == 0) rs.out[k] = acc;
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

}  // namespace hallar
