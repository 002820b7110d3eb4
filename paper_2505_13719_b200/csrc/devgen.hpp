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

}  // namespace hallar_dev
