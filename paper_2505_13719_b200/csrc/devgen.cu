// Device-side instance construction: the constraint
// sets of the reference generators, produced on the B200 instead of by a
// sequential host hash set, bit-identical to the reference order.
//
// * Matrix completion, reference rule (instances.cpp:138-175): Omega is the
//   first m DISTINCT keys i*n2 + j of the draw sequence
//   (uniform_below(n1), uniform_below(n2)), (i, j)-sorted.  The draw sequence
//   is one xoshiro256++ stream (rng.cpp:28-52).  Its state update is linear
//   over GF(2), so the state k*C outputs ahead is J^k s with J = T^C (a 256 x
//   256 bit matrix, squared up on the host): every device thread regenerates
//   its own C-output chunk of the stream.  A draw is accepted by
//   uniform_below unless r < 2^64 mod bound (probability < 2^-40 at these
//   bounds); a rejection anywhere shifts the pairing, so the builder reports
//   it and the caller falls back to the sequential host generator.
//   "First m distinct keys in draw order" is computed without a hash set:
//   a stable radix sort of (key, draw index) marks each key's first
//   occurrence, a scan over draw order counts distinct keys, the cutoff draw
//   d* is where the count reaches m, and the survivors (first occurrences
//   with d <= d*) come out of the sort already in key = (i, j) order.
// * Paper rule: the same draws, D of them, deduplicated.
// * b_k = sum_t U(i,t) V(j,t) in column order, multiply then add (no FMA:
//   this TU is compiled with -fmad=false), as instances.cpp:160-175.
// * Hypercube H(d,2) (graph.cpp:135-148): edges (v, v | 2^bit), v without
//   that bit, bits ascending, vertices ascending -- offsets by a scan of
//   d - popcount(v).
// * Pair CSR (both families): row pointers by histogram + scan, the lower
//   (j-side) CSR by a stable radix sort of (j, k), so each row's lower
//   entries stay in increasing k (the reference's adjoint_into order).
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "devgen.hpp"

namespace hallar_dev {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw std::runtime_error(std::string("devgen ") + what + ": " + cudaGetErrorString(e));
}

template <class T>
struct DBuf {
  T* p = nullptr;
  explicit DBuf(size_t n) {
    if (n) ck(cudaMalloc(&p, n * sizeof(T)), "alloc");
  }
  ~DBuf() {
    if (p) cudaFree(p);
  }
  T* release() {
    T* q = p;
    p = nullptr;
    return q;
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
};

struct Temp {
  void* p = nullptr;
  size_t n = 0;
  void* get(size_t want) {
    if (want > n) {
      if (p) cudaFree(p);
      p = nullptr;
      ck(cudaMalloc(&p, want ? want : 1), "temp alloc");
      n = want;
    }
    return p;
  }
  ~Temp() {
    if (p) cudaFree(p);
  }
};

// ------------------------------------------------------- xoshiro256++ ---
struct St {
  uint64_t s[4];
};
__host__ __device__ inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
// one state update (rng.cpp:28-38, without the output)
__host__ __device__ inline void step(uint64_t* s) {
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
}
__device__ inline uint64_t next_out(uint64_t* s) {
  const uint64_t r = rotl64(s[0] + s[3], 23) + s[0];
  step(s);
  return r;
}

// 256 x 256 GF(2) matrix as 256 columns of 4 words: column b = M e_b.
struct BitMat {
  std::vector<uint64_t> c;  // 256 * 4
  BitMat() : c(1024, 0) {}
};
void apply(const BitMat& M, const uint64_t* x, uint64_t* y) {
  uint64_t o[4] = {0, 0, 0, 0};
  for (int w = 0; w < 4; ++w) {
    uint64_t bits = x[w];
    while (bits) {
      const int b = __builtin_ctzll(bits);
      bits &= bits - 1;
      const uint64_t* col = &M.c[size_t(w * 64 + b) * 4];
      o[0] ^= col[0];
      o[1] ^= col[1];
      o[2] ^= col[2];
      o[3] ^= col[3];
    }
  }
  std::memcpy(y, o, sizeof(o));
}
BitMat square(const BitMat& M) {
  BitMat R;
  for (int b = 0; b < 256; ++b) apply(M, &M.c[size_t(b) * 4], &R.c[size_t(b) * 4]);
  return R;
}
// J = T^(2^log2c)
BitMat jump_matrix(int log2c) {
  BitMat T;
  for (int b = 0; b < 256; ++b) {
    uint64_t s[4] = {0, 0, 0, 0};
    s[b / 64] = 1ull << (b % 64);
    step(s);
    std::memcpy(&T.c[size_t(b) * 4], s, sizeof(s));
  }
  for (int i = 0; i < log2c; ++i) T = square(T);
  return T;
}

constexpr int kLog2Chunk = 12;            // raw outputs per thread chunk
constexpr int64_t kChunk = 1 << kLog2Chunk;

// Thread t regenerates raw outputs [t*C, (t+1)*C) and turns consecutive pairs
// into keys: draw d uses outputs 2d, 2d+1.
__global__ void draw_keys(const St* __restrict__ starts, int64_t nthreads, int64_t D, uint64_t n1,
                          uint64_t n2, uint64_t lim1, uint64_t lim2, uint64_t* __restrict__ keys,
                          uint32_t* __restrict__ idx, int* __restrict__ rejected) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nthreads) return;
  uint64_t s[4] = {starts[t].s[0], starts[t].s[1], starts[t].s[2], starts[t].s[3]};
  const int64_t d0 = t * (kChunk / 2);
  int rej = 0;
  for (int64_t q = 0; q < kChunk / 2; ++q) {
    const uint64_t r0 = next_out(s);
    const uint64_t r1 = next_out(s);
    const int64_t d = d0 + q;
    if (d >= D) break;
    rej |= (r0 < lim1) | (r1 < lim2);
    keys[d] = (r0 % n1) * n2 + (r1 % n2);
    idx[d] = uint32_t(d);
  }
  if (rej) atomicOr(rejected, 1);
}

// first occurrence of each key in draw order: after the stable sort a key's
// first sorted position carries its smallest draw index
__global__ void mark_first(const uint64_t* __restrict__ ks, const uint32_t* __restrict__ ds, int64_t D,
                           uint8_t* __restrict__ first_sorted, int32_t* __restrict__ first_draw) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= D) return;
  const int f = (p == 0 || ks[p] != ks[p - 1]) ? 1 : 0;
  first_sorted[p] = uint8_t(f);
  first_draw[ds[p]] = f;
}

// d* = the draw at which the distinct count reaches m
__global__ void find_cutoff(const int32_t* __restrict__ cnt, const int32_t* __restrict__ first_draw,
                            int64_t D, int32_t m, int64_t* __restrict__ cut) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d < D && first_draw[d] && cnt[d] == m) *cut = d;
}

__global__ void keep_flags(const uint8_t* __restrict__ first_sorted, const uint32_t* __restrict__ ds,
                           int64_t D, int64_t cut, uint8_t* __restrict__ keep) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= D) return;
  keep[p] = uint8_t(first_sorted[p] && int64_t(ds[p]) <= cut);
}

// (i, j, b) of the sorted sample keys; U (n1 x r) and V (n2 x r) column-major
__global__ void samples_from_keys(const uint64_t* __restrict__ keys, int64_t m, uint64_t n1, uint64_t n2,
                                  int r, const double* __restrict__ U, const double* __restrict__ V,
                                  int32_t* __restrict__ ei, int32_t* __restrict__ ej,
                                  double* __restrict__ b) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  const uint64_t key = keys[k];
  const int64_t i = int64_t(key / n2), j = int64_t(key % n2);
  ei[k] = int32_t(i);
  ej[k] = int32_t(int64_t(n1) + j);
  double d = U[i] * V[j];
  for (int t = 1; t < r; ++t) d = d + U[i + t * (int64_t)n1] * V[j + t * (int64_t)n2];
  b[k] = d;
}

unsigned blocks(int64_t n, int t = 256) { return unsigned((n + t - 1) / t); }

// ---------------------------------------------------------- hypercube ---
__global__ void cube_degree(int d, int64_t n, int64_t* __restrict__ cnt) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v < n) cnt[v] = d - __popcll((unsigned long long)v);
}
__global__ void cube_edges(int d, int64_t n, const int64_t* __restrict__ off, int32_t* __restrict__ ei,
                           int32_t* __restrict__ ej) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n) return;
  int64_t o = off[v];
  for (int bit = 0; bit < d; ++bit) {
    const int64_t u = v ^ (int64_t(1) << bit);
    if (v < u) {
      ei[o] = int32_t(v);
      ej[o] = int32_t(u);
      ++o;
    }
  }
}

// ---------------------------------------------------------------- CSR ---
__global__ void count_rows(const int32_t* __restrict__ ei, const int32_t* __restrict__ ej, int64_t np,
                           unsigned long long* __restrict__ up, unsigned long long* __restrict__ lo) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= np) return;
  atomicAdd(&up[ei[k]], 1ull);
  atomicAdd(&lo[ej[k]], 1ull);
}
__global__ void iota32(uint32_t* __restrict__ v, int64_t n) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n) v[k] = uint32_t(k);
}
__global__ void lower_cols(const int32_t* __restrict__ ei, const uint32_t* __restrict__ kk, int64_t np,
                           int32_t* __restrict__ lo_col, int64_t* __restrict__ lo_eid) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= np) return;
  const uint32_t k = kk[e];
  lo_col[e] = ei[k];
  lo_eid[e] = int64_t(k);
}
__global__ void scale_b(const double* __restrict__ b, int64_t np, double tau, double* __restrict__ bs) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < np) bs[k] = tau != 1.0 ? b[k] / tau : b[k];
}
__global__ void gather_by(const double* __restrict__ src, const int64_t* __restrict__ eid, int64_t np,
                          double* __restrict__ dst) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < np) dst[e] = src[eid[e]];
}
__global__ void check_pairs(const int64_t* __restrict__ i, const int64_t* __restrict__ j, int64_t m,
                            int64_t n1, int64_t n2, int32_t* __restrict__ ei, int32_t* __restrict__ ej,
                            int* __restrict__ bad) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int64_t a = i[k], c = j[k];
  int err = (a < 0 || a >= n1 || c < 0 || c >= n2) ? 1 : 0;
  if (k > 0 && !err) {
    const int64_t pa = i[k - 1], pc = j[k - 1];
    if (!(pa < a || (pa == a && pc < c))) err = 2;
  }
  if (err) atomicMax(bad, err);
  ei[k] = int32_t(a);
  ej[k] = int32_t(n1 + c);
}

// ---------------------------------------------------------------- SELL ---
__global__ void sell_rowlen(const int64_t* __restrict__ up, const int64_t* __restrict__ lo, int64_t n,
                            int32_t* __restrict__ nlo, int32_t* __restrict__ nv) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= n) return;
  const int64_t l = lo[a + 1] - lo[a], u = up[a + 1] - up[a];
  nlo[a] = int32_t(l);
  nv[a] = int32_t(l + u);
}
// slots of slice t: 32 x (longest row of the slice)
__global__ void sell_slice_len(const int32_t* __restrict__ nv, int64_t n, int64_t nsl,
                               int64_t* __restrict__ len) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nsl) return;
  int mx = 0;
  for (int l = 0; l < 32; ++l) {
    const int64_t a = t * 32 + l;
    if (a < n) mx = max(mx, nv[a]);
  }
  len[t] = int64_t(mx) * 32;
}
__global__ void sell_fill(const int64_t* __restrict__ up, const int64_t* __restrict__ lo,
                          const int32_t* __restrict__ ej, const int32_t* __restrict__ lo_col,
                          const int64_t* __restrict__ lo_eid, const int64_t* __restrict__ off, int64_t n,
                          int32_t* __restrict__ col, uint32_t* __restrict__ eid) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= n) return;
  const int64_t l0 = lo[a], nl = lo[a + 1] - l0, u0 = up[a], nu = up[a + 1] - u0;
  const int64_t base = off[a >> 5] + (a & 31);
  for (int64_t v = 0; v < nl; ++v) {
    col[base + 32 * v] = lo_col[l0 + v];
    eid[base + 32 * v] = uint32_t(lo_eid[l0 + v]);
  }
  for (int64_t v = 0; v < nu; ++v) {
    col[base + 32 * (nl + v)] = ej[u0 + v];
    eid[base + 32 * (nl + v)] = uint32_t(u0 + v);
  }
}
__global__ void sell_gather_k(const double* __restrict__ src, const uint32_t* __restrict__ eid, int64_t slots,
                              double* __restrict__ dst) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= slots) return;
  const uint32_t e = eid[t];
  dst[t] = e != 0xffffffffu ? src[e] : 0.0;
}

// Gaussian measurement vectors: a_ij = (z1 + i z2) / sqrt(2), (z1, z2) by
// Box-Muller from two uniforms of a counter hash of (seed, i, j); stored as the
// m x 2n row-major [Re a_i | Im a_i] (device math: not the host RNG stream)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__global__ void gauss_fill_k(double* __restrict__ A, int64_t m, int64_t n, uint64_t seed) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= m * n) return;
  const int64_t i = t / n, j = t % n;
  const uint64_t h1 = mix64(seed ^ mix64(uint64_t(t)));
  const uint64_t h2 = mix64(h1);
  const double u1 = (double((h1 >> 11) + 1)) * 0x1.0p-53;  // (0, 1]
  const double u2 = double(h2 >> 11) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1)) * 0.70710678118654752440;
  double sn, cs;
  sincospi(2.0 * u2, &sn, &cs);
  A[i * 2 * n + j] = r * cs;
  A[i * 2 * n + n + j] = r * sn;
}

}  // namespace

// ------------------------------------------------------------------ API ---
double* gauss_fill_device(int64_t m, int64_t n, uint64_t seed, cudaStream_t st) {
  double* A = nullptr;
  ck(cudaMalloc(&A, sizeof(double) * 2 * m * n), "gauss alloc");
  gauss_fill_k<<<blocks(m * n), 256, 0, st>>>(A, m, n, seed);
  ck(cudaGetLastError(), "gauss_fill");
  ck(cudaStreamSynchronize(st), "gauss_fill");
  return A;
}
int64_t sell_slots_device(int64_t n, const int64_t* up_ptr, const int64_t* lo_ptr, DevSell* out,
                          cudaStream_t st) {
  const int64_t nsl = (n + 31) / 32;
  DBuf<int32_t> nlo(static_cast<size_t>(n)), nv(static_cast<size_t>(n));
  DBuf<int64_t> len(static_cast<size_t>(nsl + 1)), off(static_cast<size_t>(nsl + 1));
  sell_rowlen<<<blocks(n), 256, 0, st>>>(up_ptr, lo_ptr, n, nlo.p, nv.p);
  ck(cudaGetLastError(), "sell_rowlen");
  ck(cudaMemsetAsync(len.p + nsl, 0, sizeof(int64_t), st), "memset");
  sell_slice_len<<<blocks(nsl), 256, 0, st>>>(nv.p, n, nsl, len.p);
  ck(cudaGetLastError(), "sell_slice_len");
  Temp temp;
  size_t tb = 0;
  ck(cub::DeviceScan::ExclusiveSum(nullptr, tb, len.p, off.p, nsl + 1, st), "scan size");
  ck(cub::DeviceScan::ExclusiveSum(temp.get(tb), tb, len.p, off.p, nsl + 1, st), "scan");
  int64_t slots = 0;
  ck(cudaMemcpyAsync(&slots, off.p + nsl, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "slots");
  ck(cudaStreamSynchronize(st), "sell sizes");
  out->slots = slots;
  out->nslices = nsl;
  out->nlo = nlo.release();
  out->nv = nv.release();
  out->off = off.release();
  return slots;
}

void sell_fill_device(int64_t n, const int64_t* up_ptr, const int64_t* lo_ptr, const int32_t* ej,
                      const int32_t* lo_col, const int64_t* lo_eid, DevSell* out, cudaStream_t st) {
  DBuf<int32_t> col(static_cast<size_t>(out->slots));
  DBuf<uint32_t> eid(static_cast<size_t>(out->slots));
  ck(cudaMemsetAsync(col.p, 0, sizeof(int32_t) * out->slots, st), "memset col");
  ck(cudaMemsetAsync(eid.p, 0xff, sizeof(uint32_t) * out->slots, st), "memset eid");
  sell_fill<<<blocks(n), 256, 0, st>>>(up_ptr, lo_ptr, ej, lo_col, lo_eid, out->off, n, col.p, eid.p);
  ck(cudaGetLastError(), "sell_fill");
  ck(cudaStreamSynchronize(st), "sell fill");
  out->col = col.release();
  out->eid = eid.release();
}

void sell_gather(const double* src_edge_order, const uint32_t* eid, int64_t slots, double* dst,
                 cudaStream_t st) {
  sell_gather_k<<<blocks(slots), 256, 0, st>>>(src_edge_order, eid, slots, dst);
  ck(cudaGetLastError(), "sell_gather");
}
bool gen_matcomp_device(int64_t n1, int64_t n2, int r, const uint64_t state[4], int64_t m_target,
                        int64_t paper_draws, const std::vector<double>& U,
                        const std::vector<double>& V, DevSamples* out, cudaStream_t st) {
  const bool paper = paper_draws > 0;
  const double N = double(n1) * double(n2);
  int64_t D;
  if (paper) {
    D = paper_draws;
  } else {
    // expected draws to see m distinct keys (coupon collector), plus slack
    const double frac = double(m_target) / N;
    const double expect = frac < 1.0 ? -N * std::log1p(-frac) : double(m_target) * 20.0;
    D = int64_t(expect * 1.0005 + 6.0 * std::sqrt(expect) + 4096.0);
    D = std::max<int64_t>(D, m_target);
  }
  if (D >= (int64_t(1) << 32) - 1) throw std::runtime_error("devgen: more than 2^32 draws");
  const uint64_t lim1 = (0 - uint64_t(n1)) % uint64_t(n1), lim2 = (0 - uint64_t(n2)) % uint64_t(n2);
  const BitMat J = jump_matrix(kLog2Chunk);
  Temp temp;
  DBuf<double> dU(U.size()), dV(V.size());
  ck(cudaMemcpyAsync(dU.p, U.data(), U.size() * sizeof(double), cudaMemcpyHostToDevice, st), "U");
  ck(cudaMemcpyAsync(dV.p, V.data(), V.size() * sizeof(double), cudaMemcpyHostToDevice, st), "V");
  int key_bits = 1;
  while (key_bits < 64 && (uint64_t(1) << key_bits) < uint64_t(n1) * uint64_t(n2)) ++key_bits;
  for (int attempt = 0; attempt < 6; ++attempt) {
    const int64_t nthreads = (2 * D + kChunk - 1) / kChunk;
    std::vector<St> starts(static_cast<size_t>(nthreads));
    {
      uint64_t s[4] = {state[0], state[1], state[2], state[3]};
      for (int64_t t = 0; t < nthreads; ++t) {
        std::memcpy(starts[t].s, s, sizeof(s));
        apply(J, s, s);
      }
    }
    DBuf<St> dst(static_cast<size_t>(nthreads));
    DBuf<uint64_t> keys(static_cast<size_t>(D)), keys2(static_cast<size_t>(D));
    DBuf<uint32_t> idx(static_cast<size_t>(D)), idx2(static_cast<size_t>(D));
    DBuf<int> rej(1);
    ck(cudaMemcpyAsync(dst.p, starts.data(), starts.size() * sizeof(St), cudaMemcpyHostToDevice, st),
       "starts");
    ck(cudaMemsetAsync(rej.p, 0, sizeof(int), st), "rej");
    draw_keys<<<blocks(nthreads, 128), 128, 0, st>>>(dst.p, nthreads, D, uint64_t(n1), uint64_t(n2),
                                                     lim1, lim2, keys.p, idx.p, rej.p);
    ck(cudaGetLastError(), "draw_keys");
    int hrej = 0;
    ck(cudaMemcpyAsync(&hrej, rej.p, sizeof(int), cudaMemcpyDeviceToHost, st), "rej D2H");
    ck(cudaStreamSynchronize(st), "draw");
    if (hrej) return false;  // a uniform_below rejection: the host generator handles it
    {
      size_t tb = 0;
      ck(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, keys2.p, idx.p, idx2.p, D, 0, key_bits, st),
         "sort size");
      ck(cub::DeviceRadixSort::SortPairs(temp.get(tb), tb, keys.p, keys2.p, idx.p, idx2.p, D, 0, key_bits,
                                         st),
         "sort");
    }
    // keys2/idx2: sorted.  Reuse keys (D x 8 B) as the flag / count scratch.
    uint8_t* first_sorted = reinterpret_cast<uint8_t*>(keys.p);
    int32_t* first_draw = reinterpret_cast<int32_t*>(idx.p);
    DBuf<int32_t> cnt(static_cast<size_t>(D));
    mark_first<<<blocks(D), 256, 0, st>>>(keys2.p, idx2.p, D, first_sorted, first_draw);
    ck(cudaGetLastError(), "mark_first");
    int64_t cut = D - 1;
    if (!paper) {
      size_t tb = 0;
      ck(cub::DeviceScan::InclusiveSum(nullptr, tb, first_draw, cnt.p, D, st), "scan size");
      ck(cub::DeviceScan::InclusiveSum(temp.get(tb), tb, first_draw, cnt.p, D, st), "scan");
      int32_t total = 0;
      ck(cudaMemcpyAsync(&total, cnt.p + (D - 1), sizeof(int32_t), cudaMemcpyDeviceToHost, st), "total");
      ck(cudaStreamSynchronize(st), "scan");
      if (int64_t(total) < m_target) {
        D = D + (m_target - total) * 2 + (D >> 6) + 4096;  // rare: draw further and redo
        continue;
      }
      DBuf<int64_t> dcut(1);
      find_cutoff<<<blocks(D), 256, 0, st>>>(cnt.p, first_draw, D, int32_t(m_target), dcut.p);
      ck(cudaGetLastError(), "find_cutoff");
      ck(cudaMemcpyAsync(&cut, dcut.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "cut");
      ck(cudaStreamSynchronize(st), "cut");
    }
    uint8_t* keep = reinterpret_cast<uint8_t*>(cnt.p);
    keep_flags<<<blocks(D), 256, 0, st>>>(first_sorted, idx2.p, D, cut, keep);
    ck(cudaGetLastError(), "keep_flags");
    DBuf<int64_t> nsel(1);
    // compact the kept sorted keys into keys (its flag role ended in keep_flags)
    {
      size_t tb = 0;
      ck(cub::DeviceSelect::Flagged(nullptr, tb, keys2.p, keep, keys.p, nsel.p, D, st), "select size");
      ck(cub::DeviceSelect::Flagged(temp.get(tb), tb, keys2.p, keep, keys.p, nsel.p, D, st), "select");
    }
    int64_t m = 0;
    ck(cudaMemcpyAsync(&m, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "nsel");
    ck(cudaStreamSynchronize(st), "select");
    if (!paper && m != m_target) throw std::runtime_error("devgen: distinct-key count mismatch");
    DBuf<int32_t> ei(static_cast<size_t>(m)), ej(static_cast<size_t>(m));
    DBuf<double> b(static_cast<size_t>(m));
    samples_from_keys<<<blocks(m), 256, 0, st>>>(keys.p, m, uint64_t(n1), uint64_t(n2), r, dU.p, dV.p,
                                                 ei.p, ej.p, b.p);
    ck(cudaGetLastError(), "samples_from_keys");
    ck(cudaStreamSynchronize(st), "samples");
    out->m = m;
    out->ei = ei.release();
    out->ej = ej.release();
    out->b = b.release();
    return true;
  }
  throw std::runtime_error("devgen: could not draw enough distinct samples");
}

void gen_hypercube_device(int d, DevSamples* out, cudaStream_t st) {
  const int64_t n = int64_t(1) << d;
  const int64_t np = n * d / 2;
  DBuf<int64_t> cnt(static_cast<size_t>(n)), off(static_cast<size_t>(n));
  cube_degree<<<blocks(n), 256, 0, st>>>(d, n, cnt.p);
  ck(cudaGetLastError(), "cube_degree");
  Temp temp;
  size_t tb = 0;
  ck(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, off.p, n, st), "scan size");
  ck(cub::DeviceScan::ExclusiveSum(temp.get(tb), tb, cnt.p, off.p, n, st), "scan");
  DBuf<int32_t> ei(static_cast<size_t>(np)), ej(static_cast<size_t>(np));
  cube_edges<<<blocks(n), 256, 0, st>>>(d, n, off.p, ei.p, ej.p);
  ck(cudaGetLastError(), "cube_edges");
  ck(cudaStreamSynchronize(st), "hypercube");
  out->m = np;
  out->ei = ei.release();
  out->ej = ej.release();
  out->b = nullptr;
}

void pairs_from_host(int64_t n1, int64_t n2, int64_t m, const int64_t* i, const int64_t* j,
                     DevSamples* out, cudaStream_t st) {
  DBuf<int64_t> di(static_cast<size_t>(m)), dj(static_cast<size_t>(m));
  ck(cudaMemcpyAsync(di.p, i, size_t(m) * sizeof(int64_t), cudaMemcpyHostToDevice, st), "i H2D");
  ck(cudaMemcpyAsync(dj.p, j, size_t(m) * sizeof(int64_t), cudaMemcpyHostToDevice, st), "j H2D");
  DBuf<int32_t> ei(static_cast<size_t>(m)), ej(static_cast<size_t>(m));
  DBuf<int> bad(1);
  ck(cudaMemsetAsync(bad.p, 0, sizeof(int), st), "bad");
  check_pairs<<<blocks(m), 256, 0, st>>>(di.p, dj.p, m, n1, n2, ei.p, ej.p, bad.p);
  ck(cudaGetLastError(), "check_pairs");
  int hb = 0;
  ck(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st), "bad D2H");
  ck(cudaStreamSynchronize(st), "pairs");
  if (hb == 1) throw std::invalid_argument("matcomp samples: index out of range");
  if (hb == 2) throw std::invalid_argument("matcomp samples: (i, j) must be strictly increasing");
  out->m = m;
  out->ei = ei.release();
  out->ej = ej.release();
  out->b = nullptr;
}

void build_csr_device(int64_t n, int64_t np, const int32_t* ei, const int32_t* ej, DevCsr* out,
                      cudaStream_t st) {
  if (np >= (int64_t(1) << 32)) throw std::runtime_error("devgen: more than 2^32 pair constraints");
  Temp temp;
  {
    DBuf<unsigned long long> cu(static_cast<size_t>(n + 1)), cl(static_cast<size_t>(n + 1));
    ck(cudaMemsetAsync(cu.p, 0, sizeof(unsigned long long) * (n + 1), st), "memset");
    ck(cudaMemsetAsync(cl.p, 0, sizeof(unsigned long long) * (n + 1), st), "memset");
    count_rows<<<blocks(np), 256, 0, st>>>(ei, ej, np, cu.p, cl.p);
    ck(cudaGetLastError(), "count_rows");
    DBuf<int64_t> up(static_cast<size_t>(n + 1)), lo(static_cast<size_t>(n + 1));
    size_t tb = 0;
    auto* cu64 = reinterpret_cast<int64_t*>(cu.p);
    auto* cl64 = reinterpret_cast<int64_t*>(cl.p);
    ck(cub::DeviceScan::ExclusiveSum(nullptr, tb, cu64, up.p, n + 1, st), "scan size");
    ck(cub::DeviceScan::ExclusiveSum(temp.get(tb), tb, cu64, up.p, n + 1, st), "scan");
    ck(cub::DeviceScan::ExclusiveSum(temp.get(tb), tb, cl64, lo.p, n + 1, st), "scan");
    out->up_ptr = up.release();
    out->lo_ptr = lo.release();
  }
  {
    DBuf<uint32_t> key2(static_cast<size_t>(np)), kk(static_cast<size_t>(np)), kk2(static_cast<size_t>(np));
    iota32<<<blocks(np), 256, 0, st>>>(kk.p, np);
    ck(cudaGetLastError(), "iota");
    int bits = 1;
    while (bits < 32 && (int64_t(1) << bits) < n) ++bits;
    const auto* keys = reinterpret_cast<const uint32_t*>(ej);
    size_t tb = 0;
    ck(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, key2.p, kk.p, kk2.p, np, 0, bits, st), "sort size");
    ck(cub::DeviceRadixSort::SortPairs(temp.get(tb), tb, keys, key2.p, kk.p, kk2.p, np, 0, bits, st), "sort");
    DBuf<int32_t> lo_col(static_cast<size_t>(np));
    DBuf<int64_t> lo_eid(static_cast<size_t>(np));
    lower_cols<<<blocks(np), 256, 0, st>>>(ei, kk2.p, np, lo_col.p, lo_eid.p);
    ck(cudaGetLastError(), "lower_cols");
    ck(cudaStreamSynchronize(st), "csr");
    out->lo_col = lo_col.release();
    out->lo_eid = lo_eid.release();
  }
}

void scale_and_lower(const double* b, int64_t np, double tau, const int64_t* lo_eid, double* b_up,
                     double* b_lo, cudaStream_t st) {
  scale_b<<<blocks(np), 256, 0, st>>>(b, np, tau, b_up);
  ck(cudaGetLastError(), "scale_b");
  gather_by<<<blocks(np), 256, 0, st>>>(b_up, lo_eid, np, b_lo);
  ck(cudaGetLastError(), "gather_by");
}

}  // namespace hallar_dev
