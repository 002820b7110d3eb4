// Device-side instance construction (devgen.cu): matrix-completion samples
// and hypercube edges generated on the GPU, bit-identical to the reference
// generators, and the pair CSR built on the GPU.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace hallar_dev {

// Device arrays of pair constraints (sorted by (ei, ej)); ownership passes
// to the caller (cudaFree).
struct DevSamples {
  int64_t m = 0;
  int32_t* ei = nullptr;
  int32_t* ej = nullptr;  // matrix completion: n1 + j
  double* b = nullptr;    // unscaled right-hand side (matrix completion)
};

struct DevCsr {
  int64_t* up_ptr = nullptr;  // n + 1
  int64_t* lo_ptr = nullptr;  // n + 1
  int32_t* lo_col = nullptr;  // np
  int64_t* lo_eid = nullptr;  // np
};

// Omega and b of gen_matrix_completion (instances.cpp:131-175) from the RNG
// state after the hidden factors were drawn.  m_target > 0: the reference rule
// (first m distinct draws); paper_draws > 0: that many draws, deduplicated.
// U (n1 x r) and V (n2 x r) column-major.  Returns false when a uniform_below
// rejection occurs in the stream (the caller then generates on the host).
bool gen_matcomp_device(int64_t n1, int64_t n2, int r, const uint64_t state[4], int64_t m_target,
                        int64_t paper_draws, const std::vector<double>& U,
                        const std::vector<double>& V, DevSamples* out, cudaStream_t st);

// make_hypercube(d) edges (graph.cpp:135-148) on the device.
void gen_hypercube_device(int d, DevSamples* out, cudaStream_t st);

// Host sample lists (int64, (i, j) strictly increasing, i < n1, j < n2) -> device
// pairs (j offset by n1); throws std::invalid_argument on bad input.
void pairs_from_host(int64_t n1, int64_t n2, int64_t m, const int64_t* i, const int64_t* j,
                     DevSamples* out, cudaStream_t st);

// Row pointers of both halves and the lower (j-side) CSR, stable in k.
void build_csr_device(int64_t n, int64_t np, const int32_t* ei, const int32_t* ej, DevCsr* out,
                      cudaStream_t st);

// b_up = b / tau (edge order), b_lo = b_up[lo_eid] (lower order).
void scale_and_lower(const double* b, int64_t np, double tau, const int64_t* lo_eid, double* b_up,
                     double* b_lo, cudaStream_t st);

// SELL-32 copy of the merged row streams (common.cuh DevPairs::s_*).
struct DevSell {
  int64_t slots = 0, nslices = 0;
  int64_t* off = nullptr;   // [nslices + 1]
  int32_t* nlo = nullptr;   // [n]
  int32_t* nv = nullptr;    // [n]
  int32_t* col = nullptr;   // [slots]
  uint32_t* eid = nullptr;  // [slots]
};
// sizes (off, nlo, nv) -> returns the slot count; then the slot arrays
int64_t sell_slots_device(int64_t n, const int64_t* up_ptr, const int64_t* lo_ptr, DevSell* out,
                          cudaStream_t st);
void sell_fill_device(int64_t n, const int64_t* up_ptr, const int64_t* lo_ptr, const int32_t* ej,
                      const int32_t* lo_col, const int64_t* lo_eid, DevSell* out, cudaStream_t st);
// dst[slot] = src[eid[slot]] (0 on padding): an edge-order vector -> SELL order
void sell_gather(const double* src_edge_order, const uint32_t* eid, int64_t slots, double* dst,
                 cudaStream_t st);

// Gaussian phase retrieval: the m x 2n row-major [Re a_i | Im a_i] (caller frees)
double* gauss_fill_device(int64_t m, int64_t n, uint64_t seed, cudaStream_t st);

}  // namespace hallar_dev
