// C-ABI of libcuhallar.so (include/cuhallar.h): instance upload, persistent
// kernel launch, host <-> device layout conversion.  Host orchestration only;
// all solver arithmetic runs in hallar_kernel (solve.cuh).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <functional>
#include <atomic>
#include <thread>
#include <string>
#include <vector>

#include "../../include/cuhallar.h"
#include "devgen.hpp"
#include "host_instances.hpp"
#include "kernel_setup.cuh"
#include "solve.cuh"

using namespace hallar;
namespace hh = hallar_host;
namespace hd = hallar_dev;

// ----------------------------------------------------------------- kernel ---
namespace hallar {
__global__ void __launch_bounds__(kThreads, 1)
    hallar_kernel(const __grid_constant__ Params P, SolveOut* so) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Ctx c;
  setup_ctx(c, P, smem_raw);
  if (P.op == kOpSolve) {
    solve_dev(c, P, so);
  } else {
    HALLAR_DISPATCH_S(P.s_in, op_dispatch<S_>(c, P, so));
  }
}

// column-major (ld) <-> row-major (stride s) factor conversion
__global__ void to_rowmajor(const double* __restrict__ src, int64_t ld, int s, int64_t n,
                            double* __restrict__ dst) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * s) return;
  const int64_t a = t / s, k = t % s;
  dst[t] = src[a + k * ld];
}
__global__ void to_colmajor(const double* __restrict__ src, int s, int64_t n, double* dst,
                            int64_t ld) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * s) return;
  const int64_t a = t % n, k = t / n;
  dst[a + k * ld] = src[a * s + k];
}
// lower-order copy of an edge-order vector: dst[e] = src[eid[e]]
__global__ void gather_lower(const double* __restrict__ src, const int64_t* __restrict__ eid,
                             int64_t cnt, double* __restrict__ dst) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < cnt) dst[e] = src[eid[e]];
}
}  // namespace hallar

namespace hallar {
// parity_kernel.cu
const void* hallar_parity_kernel_fn();
int hallar_parity_prepare();  // sets the smem attribute; returns resident CTAs per SM
}  // namespace hallar

namespace {

thread_local std::string g_err;


struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
T* dalloc(size_t count, int64_t* acct) {
  if (count == 0) count = 1;
  void* p = nullptr;
  ck(cudaMalloc(&p, count * sizeof(T)), "cudaMalloc");
  if (acct) *acct += int64_t(count * sizeof(T));
  return static_cast<T*>(p);
}
template <class T>
T* dupload(const std::vector<T>& v, int64_t* acct) {
  T* p = dalloc<T>(v.size(), acct);
  if (!v.empty()) ck(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "H2D");
  return p;
}

int grid_size(int requested) {
  static int cache[64];
  static bool init = false;
  if (!init) {
    for (auto& x : cache) x = -1;
    init = true;
  }
  int cur = 0;
  ck(cudaGetDevice(&cur), "device");
  int& cached = cache[cur & 63];
  if (cached < 0) {
    ck(cudaFuncSetAttribute(hallar_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(kSmemBytes)),
       "smem attr");
    int dev = 0, sms = 0, per = 0;
    ck(cudaGetDevice(&dev), "device");
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sm count");
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, hallar_kernel, kThreads, kSmemBytes),
       "occupancy");
    if (per < 1) throw CudaError("hallar_kernel cannot be resident");
    const int pp = hallar_parity_prepare();  // same team size for both persistent kernels
    if (pp < 1) throw CudaError("hallar_parity_kernel cannot be resident");
    per = std::min(per, pp);
    cached = std::min(sms * per, kMaxTeam);
  }
  if (requested > 0) return std::min(requested, cached);
  return cached;
}

}  // namespace

// ---------------------------------------------------------------- instance ---
struct cuhallar_instance {
  hh::HostInst h;
  DevPairs I{};
  int64_t bytes = 0;
  int64_t h2d = 0;
  // device arrays
  int32_t *ei = nullptr, *ej = nullptr, *lo_col = nullptr;
  int64_t *up_ptr = nullptr, *lo_ptr = nullptr, *lo_eid = nullptr, *tile_row = nullptr;
  double *b_up = nullptr, *b_lo = nullptr;      // scaled b/tau (solve)
  double *ub_up = nullptr, *ub_lo = nullptr;    // unscaled b (operator ABI), lazy
  double2 *masks = nullptr, *twid = nullptr, *prF = nullptr, *prG = nullptr;  // phase retrieval
  double* gA = nullptr;  // Gaussian phase retrieval: m x 2n measurement matrix
  // workspace
  int ws_grid = 0;
  unsigned long long* bar = nullptr;
  double* slots = nullptr;
  double* buf[kNBuf] = {};
  double* vslot = nullptr;
  int nslot = 0;
  double* arena = nullptr;  // buf[0..kNBuf) and the Lanczos slots: the replicated factor arena
  int64_t arena_len = 0;
  int device = 0;
  std::vector<int64_t> tile_row_host, up_ptr_host;
  // sharded-solve rendezvous state (this rank's side)
  unsigned long long* xbar = nullptr;
  double* xslots = nullptr;
  int* xerr = nullptr;
  double *p_up = nullptr, *p_lo = nullptr, *q_up = nullptr, *q_lo = nullptr, *r_up = nullptr,
         *r_lo = nullptr;
  double* lz_rand = nullptr;
  // Lanczos refills beyond the pre-drawn ones (RefillService)
  std::unique_ptr<hh::Xoshiro> lz_gen;           // positioned after the pre-drawn normals
  std::vector<std::vector<double>> lz_extra;     // refills n_refill + 1, ... drawn so far
  int *svc_req_h = nullptr, *svc_ready_h = nullptr, *svc_err_d = nullptr;
  double* svc_buf_h = nullptr;
  hd::DevSell sell;  // SELL-32 row-stream copy (single-GPU row passes), optional
  double *s_b = nullptr, *s_ub = nullptr, *p_sell = nullptr, *q_sell = nullptr, *r_sell = nullptr;
  double* pad = nullptr;  // n x 4 padded rank-3 factor rows (SELL passes)
  int n_refill = 0;
  uint64_t lz_seed = ~0ull;
  double* dscal = nullptr;
  int* discal = nullptr;
  SolveOut* dso = nullptr;
  unsigned long long* dprof = nullptr;
  std::vector<unsigned long long> last_prof;
  TraceEv* trace_host = nullptr;
  int* trace_count_host = nullptr;
  int trace_cap = 65536;
  std::mutex mu;

  ~cuhallar_instance() {
    auto f = [](void* p) {
      if (p) cudaFree(p);
    };
    f(ei); f(ej); f(lo_col); f(up_ptr); f(lo_ptr); f(lo_eid); f(tile_row); f(b_up); f(b_lo); f(ub_up); f(ub_lo);
    f(masks); f(twid); f(prF); f(prG); f(gA);
    f(bar); f(slots); f(arena); f(xbar); f(xslots); f(xerr);
    f(p_up); f(p_lo); f(q_up); f(q_lo); f(r_up); f(r_lo); f(lz_rand); f(dscal); f(discal); f(dso); f(dprof);
    f(sell.off); f(sell.nlo); f(sell.nv); f(sell.col); f(sell.eid); f(s_b); f(s_ub); f(pad); f(p_sell); f(q_sell); f(r_sell);
    if (trace_host) cudaFreeHost(trace_host);
    if (svc_req_h) cudaFreeHost(svc_req_h);
    if (svc_ready_h) cudaFreeHost(svc_ready_h);
    if (svc_buf_h) cudaFreeHost(svc_buf_h);
    f(svc_err_d);
    if (trace_count_host) cudaFreeHost(trace_count_host);
  }
};

struct cuhallar_solution {
  int64_t n = 0, m = 0;
  int rank = 0;
  std::vector<double> U;  // column-major
  std::vector<double> p;  // host copy (sharded solves), empty when p_dev holds it
  // single-GPU solves: a device copy of the pair multipliers (D2D at solve end)
  // and the trace multiplier; cuhallar_solution_get_p copies straight into the
  // caller's buffer (one D2H, no zero-filled 1 GB staging vector at C4)
  double* p_dev = nullptr;
  int64_t np = 0;
  bool has_trace = false;
  double p_trace = 0.0;
  int device = 0;
  ~cuhallar_solution() {
    if (p_dev) {
      int cur = 0;
      cudaGetDevice(&cur);
      cudaSetDevice(device);
      cudaFree(p_dev);
      cudaSetDevice(cur);
    }
  }
};

namespace {

// SELL-32 copy of the row streams (common.cuh DevPairs::s_*) for the
// single-GPU row passes of large instances (>= kRtMinRows rows per CTA), when
// HBM allows it next to the factor arena; CUHALLAR_NO_SELL=1 disables it.
int grid_size(int requested);
void build_sell(cuhallar_instance* in) {
  const auto& h = in->h;
  const char* e = std::getenv("CUHALLAR_NO_SELL");
  if (e && *e && *e != '0') return;
  int team = 148;
  try {
    team = grid_size(0);
  } catch (...) {
  }
  if (h.n < int64_t(team) * kRtMinRows) return;
  hd::DevSell sl;
  const int64_t slots = hd::sell_slots_device(h.n, in->up_ptr, in->lo_ptr, &sl, 0);
  const int64_t per_slot = 4 + 4 + 24 + (h.has_trace ? 0 : 8);
  const int64_t arena = h.n * (int64_t(kNBuf) * kSMax + kLanczosMax + kLanczosMax / 3 + 8) * 8;
  size_t fr = 0, tot = 0;
  ck(cudaMemGetInfo(&fr, &tot), "mem info");
  if (int64_t(fr) < slots * per_slot + arena + (int64_t(4) << 30)) {  // no room: the row-thread engine
    cudaFree(sl.off); cudaFree(sl.nlo); cudaFree(sl.nv);
    return;
  }
  hd::sell_fill_device(h.n, in->up_ptr, in->lo_ptr, in->ej, in->lo_col, in->lo_eid, &sl, 0);
  in->sell = sl;
  in->bytes += slots * 8 + (sl.nslices + 1) * 8 + h.n * 8;
  in->pad = dalloc<double>(size_t(h.n) * 4, &in->bytes);
  in->p_sell = dalloc<double>(size_t(slots), &in->bytes);
  in->q_sell = dalloc<double>(size_t(slots), &in->bytes);
  in->r_sell = dalloc<double>(size_t(slots), &in->bytes);
  ck(cudaMemset(in->p_sell, 0, slots * sizeof(double)), "p_sell");
  if (!h.has_trace) {
    in->s_b = dalloc<double>(size_t(slots), &in->bytes);
    hd::sell_gather(in->b_up, sl.eid, slots, in->s_b, 0);
  }
  ck(cudaDeviceSynchronize(), "sell");
  DevPairs& I = in->I;
  I.s_off = sl.off;
  I.s_col = sl.col;
  I.s_nlo = sl.nlo;
  I.s_nv = sl.nv;
  I.s_b = in->s_b;
  I.s_eid = sl.eid;
  I.s_slots = slots;
  // matrix completion: rows <= max i_k = ei[np-1] (edges sorted by (i, j)) hold
  // every upper entry -> the row-ordered map pass (device.cuh map_pass_sell);
  // CUHALLAR_NO_SELL_MAP=1 keeps the edge-order map (A/B runs)
  // cost-balanced CTA row split (kernel_setup.cuh); CUHALLAR_EVEN_TILES=1
  // keeps equal tile counts (A/B runs).  32 entries per row: the C4 solve
  // measured 3.27 / 3.26 / 3.41 / 3.43 s at 16 / 32 / 64 / 128 per row and
  // 3.77 s with equal tile counts (profiles/r02/ab_s4)
  const char* et = std::getenv("CUHALLAR_EVEN_TILES");
  if (!(et && *et && *et != '0')) I.split_w = 32;
  if (const char* ew = std::getenv("CUHALLAR_SPLIT_W")) I.split_w = std::max(0, std::atoi(ew));  // sweeps
  const char* em = std::getenv("CUHALLAR_NO_SELL_MAP");
  if (h.family == kMatcomp && !h.has_trace && h.np > 0 && in->s_b && !(em && *em && *em != '0')) {
    int32_t last = 0;
    ck(cudaMemcpy(&last, in->ei + (h.np - 1), sizeof(int32_t), cudaMemcpyDeviceToHost), "ei tail");
    I.s_up_slices = (int64_t(last) + 32) / 32;
  }
  // theta: upper entries in every slice; worth it while the SELL padding is
  // small (uniform degrees, e.g. hypercubes: s_slots == 2 np)
  if (h.has_trace && h.np > 0 && slots <= 2 * h.np + h.np / 2 && !(em && *em && *em != '0'))
    I.s_up_slices = sl.nslices;
}

// Device structure of a pair instance (devgen.cu builds it on the GPU):
// ei / ej (device, sorted by (i, j); the instance takes ownership), the row
// pointers of both halves, the lower CSR stable by edge id, row tiles, and
// the scaled right-hand side in both orders.  b_dev: unscaled device b
// (matrix completion, owned from here on) or null (b from h.b / theta).
void build_pairs(cuhallar_instance* in, int32_t* d_ei, int32_t* d_ej, double* b_dev,
                 const double* b_host = nullptr) {
  auto& h = in->h;
  const int64_t n = h.n, np = h.np;
  in->ei = d_ei;
  in->ej = d_ej;
  in->bytes += int64_t(2 * np * sizeof(int32_t));
  hd::DevCsr csr;
  hd::build_csr_device(n, np, d_ei, d_ej, &csr, 0);
  in->up_ptr = csr.up_ptr;
  in->lo_ptr = csr.lo_ptr;
  in->lo_col = csr.lo_col;
  in->lo_eid = csr.lo_eid;
  in->bytes += int64_t(2 * (n + 1) * sizeof(int64_t) + np * (sizeof(int32_t) + sizeof(int64_t)));
  std::vector<int64_t> up(n + 1), lo(n + 1);
  ck(cudaMemcpy(up.data(), csr.up_ptr, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost), "up_ptr");
  ck(cudaMemcpy(lo.data(), csr.lo_ptr, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost), "lo_ptr");
  {
    // Row tiles for the tile engine: consecutive rows, <= kTileRows rows and
    // <= target entries, target chosen so that every CTA gets tiles.
    int team = 148;
    try {
      team = grid_size(0);
    } catch (...) {
    }
    const int64_t total = 2 * np;
    const int64_t target =
        std::max<int64_t>(32, std::min<int64_t>(kTileEntries, (total + team * kGroups - 1) / (team * kGroups)));
    std::vector<int64_t> tr{0};
    int64_t r0 = 0;
    while (r0 < n) {
      int64_t r1 = r0, ent = 0;
      while (r1 < n && r1 - r0 < kTileRows) {
        const int64_t d = (up[r1 + 1] - up[r1]) + (lo[r1 + 1] - lo[r1]);
        if (r1 > r0 && ent + d > target) break;
        ent += d;
        ++r1;
        if (ent > kTileEntries) break;  // a single long row becomes its own tile
      }
      tr.push_back(r1);
      r0 = r1;
    }
    in->tile_row = dupload(tr, &in->bytes);
    in->h2d += int64_t(tr.size() * sizeof(int64_t));
    in->tile_row_host = tr;
    in->up_ptr_host = up;
    in->I.tile_row = in->tile_row;
    in->I.ntiles = int64_t(tr.size()) - 1;
  }
  DevPairs& I = in->I;
  I.family = h.family;
  I.has_trace = h.has_trace ? 1 : 0;
  I.n = n;
  I.np = np;
  I.m = h.m;
  I.ei = in->ei;
  I.ej = in->ej;
  I.up_ptr = in->up_ptr;
  I.lo_ptr = in->lo_ptr;
  I.lo_col = in->lo_col;
  I.lo_eid = in->lo_eid;
  I.norm_C1 = h.norm_C1;
  if (h.has_trace) {
    // theta: b = e_{m-1}, tau = 1 (instances.cpp:80-87)
    I.b_trace = h.b.empty() ? 1.0 : h.b[h.m - 1];
    I.norm_b1 = h.norm_b1;
    I.nb2 = std::fabs(I.b_trace);
    for (int64_t k = 0; k + 1 < int64_t(h.b.size()); ++k)
      if (h.b[k] != 0.0) throw hh::InputError("theta: nonzero edge right-hand side");
    build_sell(in);
    return;
  }
  // matrix completion: unscaled b on the device (edge order); the Eigen-order
  // norms on the host from b_host, else from h.b (copied back if the device
  // generated b); scale_instance (solver.cpp:31-42): b <- b / tau
  if (!b_host && !h.b.empty()) b_host = h.b.data();
  if (!b_dev) {
    if (!b_host) throw hh::InputError("matcomp: no right-hand side");
    b_dev = dalloc<double>(size_t(np), nullptr);
    ck(cudaMemcpy(b_dev, b_host, np * sizeof(double), cudaMemcpyHostToDevice), "b");
    in->h2d += int64_t(np * sizeof(double));
  } else if (!b_host) {
    h.b.resize(size_t(np));
    ck(cudaMemcpy(h.b.data(), b_dev, np * sizeof(double), cudaMemcpyDeviceToHost), "b D2H");
    b_host = h.b.data();
  }
  in->ub_up = b_dev;
  in->bytes += int64_t(np * sizeof(double));
  in->b_up = dalloc<double>(size_t(np), &in->bytes);
  in->b_lo = dalloc<double>(size_t(np), &in->bytes);
  hd::scale_and_lower(b_dev, np, h.tau, in->lo_eid, in->b_up, in->b_lo, 0);
  // host reductions overlap the device scaling
  if (h.norm_b1 == 0.0) h.norm_b1 = hh::eigen_order_sum_abs(b_host, np);
  I.norm_b1 = h.tau != 1.0 ? h.norm_b1 / h.tau : h.norm_b1;
  I.nb2 = std::sqrt(hh::eigen_order_sum_sq_scaled(b_host, np, h.tau));
  ck(cudaDeviceSynchronize(), "b scale");
  I.b_up = in->b_up;
  I.b_lo = in->b_lo;
  build_sell(in);
}

// host-built pair instance -> device
void upload_pairs(cuhallar_instance* in) {
  auto& h = in->h;
  int32_t* dei = dalloc<int32_t>(size_t(h.np), nullptr);
  int32_t* dej = dalloc<int32_t>(size_t(h.np), nullptr);
  ck(cudaMemcpy(dei, h.ei.data(), h.np * sizeof(int32_t), cudaMemcpyHostToDevice), "ei");
  ck(cudaMemcpy(dej, h.ej.data(), h.np * sizeof(int32_t), cudaMemcpyHostToDevice), "ej");
  in->h2d += int64_t(2 * h.np * sizeof(int32_t));
  std::vector<int32_t>().swap(h.ei);
  std::vector<int32_t>().swap(h.ej);
  build_pairs(in, dei, dej, nullptr);
}

void ensure_workspace(cuhallar_instance* in, int grid, uint64_t seed, int block_restart) {
  const int64_t n = in->h.n, np = in->h.np;
  if (!in->bar) {
    in->bar = dalloc<unsigned long long>(1, &in->bytes);
    // factor pool + Lanczos slots in one allocation, identical layout on every
    // rank of a sharded solve (peer address = peer arena + same offset)
    in->nslot = kLanczosMax + kLanczosMax / 3 + 8;
    in->arena_len = int64_t(n) * (int64_t(kNBuf) * kSMax + in->nslot);
    in->arena = dalloc<double>(size_t(in->arena_len), &in->bytes);
    for (int i = 0; i < kNBuf; ++i) in->buf[i] = in->arena + size_t(i) * n * kSMax;
    in->vslot = in->arena + size_t(kNBuf) * n * kSMax;
    in->p_up = dalloc<double>(np, &in->bytes);
    in->p_lo = dalloc<double>(np, &in->bytes);
    in->q_up = dalloc<double>(np, &in->bytes);
    in->q_lo = dalloc<double>(np, &in->bytes);
    in->r_up = dalloc<double>(np, &in->bytes);
    in->r_lo = dalloc<double>(np, &in->bytes);
    in->dscal = dalloc<double>(8, &in->bytes);
    in->discal = dalloc<int>(8, &in->bytes);
    in->dso = dalloc<SolveOut>(1, &in->bytes);

  }
  if (grid > in->ws_grid) {
    if (in->slots) cudaFree(in->slots);
    in->slots = dalloc<double>(size_t(2) * grid * kRedK, &in->bytes);
    in->ws_grid = grid;
  }
  (void)block_restart;  // slots sized for the device cap (kLanczosMax) at allocation
  if (seed != in->lz_seed) {
    // Lanczos start vector + breakdown refills: the stream of
    // gaussian_vector(n, Rng(seed ^ 0x9b97f4a7c15)) calls (lanczos.cpp:46-50, 128-129)
    // (a refill is drawn only when a Krylov basis breaks down before reaching n:
    // rare, so a few per call suffice beyond tiny instances)
    // more are drawn on demand by the launch's RefillService
    int refill = int(std::max<int64_t>(4, std::min<int64_t>(64, (int64_t(1) << 16) / n)));
    if (const char* e = std::getenv("CUHALLAR_LZ_PREDRAW")) refill = std::max(0, std::atoi(e));  // tests
    in->lz_gen = std::make_unique<hh::Xoshiro>(seed ^ 0x9b97f4a7c15ULL);
    in->lz_extra.clear();
    std::vector<double> v(size_t(n) * (1 + refill));
    for (auto& x : v) x = in->lz_gen->normal();
    if (in->lz_rand) cudaFree(in->lz_rand);
    in->lz_rand = dupload(v, &in->bytes);
    in->h2d += int64_t(v.size() * sizeof(double));
    in->n_refill = refill;
    in->lz_seed = seed;
    if (!in->svc_buf_h) {
      ck(cudaHostAlloc(&in->svc_req_h, sizeof(int), cudaHostAllocMapped), "svc req");
      ck(cudaHostAlloc(&in->svc_ready_h, sizeof(int), cudaHostAllocMapped), "svc ready");
      ck(cudaHostAlloc(&in->svc_buf_h, sizeof(double) * n, cudaHostAllocMapped), "svc buf");
      in->svc_err_d = dalloc<int>(1, &in->bytes);
    }
  }
}

Params base_params(cuhallar_instance* in, const cuhallar_config* cfg);
int launch(cuhallar_instance* in, Params& P, int grid, cudaStream_t st, SolveOut* so,
           float* ms = nullptr, const std::function<void()>& poll = nullptr);

void upload_pr(cuhallar_instance* in);
// Gaussian phase retrieval: A' generated on the device, the spectrum cache F
// (kSMax x m) and the adjoint partials G (kSMax x parts x n), then b = the
// device map of the hidden signal, as upload_pr does for coded diffraction.
void upload_gpr(cuhallar_instance* in, uint64_t seed) {
  auto& h = in->h;
  const int64_t n = h.nc, m = h.m;
  h.np = m;
  in->gA = hd::gauss_fill_device(m, n, seed ^ 0x5eed9a55ULL, 0);
  in->bytes += int64_t(2 * m * n * sizeof(double));
  in->prF = dalloc<double2>(size_t(kSMax) * m, &in->bytes);
  in->prG = dalloc<double2>(size_t(kSMax) * h.L * n, &in->bytes);
  DevPairs& I = in->I;
  I.family = kPhaseret;
  I.has_trace = 0;
  I.n = h.n;
  I.np = m;
  I.m = m;
  I.nc = n;
  I.L = h.L;
  I.lognc = 0;
  I.gA = in->gA;
  I.F = in->prF;
  I.G = in->prG;
  I.norm_C1 = h.norm_C1;
  {
    const int grid = grid_size(0);
    ensure_workspace(in, grid, 0, 30);
    std::vector<double> x(size_t(h.n));
    for (int64_t j = 0; j < n; ++j) {
      x[j] = h.hidden_x[j].real();
      x[n + j] = h.hidden_x[j].imag();
    }
    ck(cudaMemcpy(in->buf[0], x.data(), x.size() * sizeof(double), cudaMemcpyHostToDevice), "x");
    in->h2d += int64_t(x.size() * sizeof(double));
    double* bd = in->r_up;
    Params P = base_params(in, nullptr);
    P.op = kOpMap;
    P.s_in = 1;
    P.out_vec = bd;
    SolveOut so{};
    if (launch(in, P, grid, 0, &so, nullptr) != kOk) throw CudaError("gauss_pr: b map failed");
    h.b.resize(m);
    ck(cudaMemcpy(h.b.data(), bd, m * sizeof(double), cudaMemcpyDeviceToHost), "b");
  }
  h.norm_b1 = hh::eigen_order_sum_abs(h.b.data(), m);
  std::vector<double> bs(m);
  for (int64_t k = 0; k < m; ++k) bs[k] = h.tau != 1.0 ? h.b[k] / h.tau : h.b[k];
  I.norm_b1 = h.tau != 1.0 ? h.norm_b1 / h.tau : h.norm_b1;
  I.nb2 = std::sqrt(hh::eigen_order_sum_sq(bs.data(), m));
  in->b_up = dupload(bs, &in->bytes);
  in->h2d += int64_t(m * sizeof(double));
  I.b_up = in->b_up;
  I.b_lo = nullptr;
}

void upload_pr(cuhallar_instance* in) {
  auto& h = in->h;
  const int64_t nc = h.nc, m = h.m;
  h.np = m;  // constraint-order vectors (p, q, r, b) use the edge-order slots
  int lg = 0;
  while ((int64_t(1) << lg) < nc) ++lg;
  {
    std::vector<double2> mk(h.masks.size()), tw(std::max<size_t>(1, h.twiddle.size()));
    for (size_t i = 0; i < mk.size(); ++i) mk[i] = make_double2(h.masks[i].real(), h.masks[i].imag());
    for (size_t i = 0; i < h.twiddle.size(); ++i)
      tw[i] = make_double2(h.twiddle[i].real(), h.twiddle[i].imag());
    in->masks = dupload(mk, &in->bytes);
    in->twid = dupload(tw, &in->bytes);
  }
  in->prF = dalloc<double2>(size_t(kSMax) * m, &in->bytes);
  in->prG = dalloc<double2>(size_t(kSMax) * m, &in->bytes);
  in->h2d += in->bytes;
  DevPairs& I = in->I;
  I.family = kPhaseret;
  I.has_trace = 0;
  I.n = h.n;
  I.np = m;
  I.m = m;
  I.nc = nc;
  I.L = h.L;
  I.lognc = lg;
  I.masks = in->masks;
  I.twid = in->twid;
  I.F = in->prF;
  I.G = in->prG;
  I.norm_C1 = h.norm_C1;
  // b = A(x x*) of the hidden signal through the device map (s = 1)
  {
    const int grid = grid_size(0);
    ensure_workspace(in, grid, 0, 30);
    std::vector<double> x(size_t(h.n));
    for (int64_t j = 0; j < nc; ++j) {
      x[j] = h.hidden_x[j].real();
      x[nc + j] = h.hidden_x[j].imag();
    }
    ck(cudaMemcpy(in->buf[0], x.data(), x.size() * sizeof(double), cudaMemcpyHostToDevice), "x");
    double* bd = in->r_up;  // scratch
    Params P = base_params(in, nullptr);
    P.op = kOpMap;
    P.s_in = 1;
    P.out_vec = bd;
    SolveOut so{};
    if (launch(in, P, grid, 0, &so, nullptr) != kOk) throw CudaError("phaseret: b map failed");
    h.b.resize(m);
    ck(cudaMemcpy(h.b.data(), bd, m * sizeof(double), cudaMemcpyDeviceToHost), "b");
  }
  h.norm_b1 = hh::eigen_order_sum_abs(h.b.data(), m);
  // scale_instance (solver.cpp:31-42)
  std::vector<double> bs(m);
  for (int64_t k = 0; k < m; ++k) bs[k] = h.tau != 1.0 ? h.b[k] / h.tau : h.b[k];
  I.norm_b1 = h.tau != 1.0 ? h.norm_b1 / h.tau : h.norm_b1;
  I.nb2 = std::sqrt(hh::eigen_order_sum_sq(bs.data(), m));
  in->b_up = dupload(bs, &in->bytes);
  in->h2d += int64_t(m * sizeof(double));
  I.b_up = in->b_up;
  I.b_lo = nullptr;
}

Cfg to_dev_cfg(const cuhallar_config& c) {
  Cfg d{};
  d.eps = c.eps;
  d.beta0 = c.beta0;
  d.beta_growth = c.beta_growth;
  d.eps0 = c.eps0;
  d.eps_decay = c.eps_decay;
  d.eps_floor = c.eps_floor;
  d.max_outer = c.max_outer;
  d.time_limit = c.time_limit;
  d.eig_tol = c.eig_tol;
  d.eig_max_iters = c.eig_max_iters;
  d.eig_block_restart = c.eig_block_restart;
  d.aipp_lambda0 = c.aipp_lambda0;
  d.aipp_rho = c.aipp_rho;
  d.aipp_max_outer = c.aipp_max_outer;
  d.aipp_lambda_underflow = c.aipp_lambda_underflow;
  d.fista_sigma = c.fista_sigma;
  d.fista_chi = c.fista_chi;
  d.fista_mu = c.fista_mu;
  d.fista_L0 = c.fista_L0;
  d.fista_max_iters = c.fista_max_iters;
  d.max_fw_steps = c.max_fw_steps;
  d.trace = c.trace;
  d.parity = c.parity;
  return d;
}

void validate_cfg(const cuhallar_config& c) {
  auto need = [](bool ok, const char* w) {
    if (!ok) throw hh::InputError(w);
  };
  need(c.eps > 0, "config: eps must be positive");
  need(c.beta_growth >= 1.0, "config: beta_growth must be >= 1");
  need(c.eps_decay > 0 && c.eps_decay <= 1.0, "config: eps_decay in (0,1]");
  need(c.max_outer >= 1, "config: max_outer must be >= 1");
  need(c.time_limit > 0, "config: time_limit must be positive");
  need(c.max_fw_steps >= 1, "config: max_fw_steps must be >= 1");
  need(c.eig_tol > 0, "eig: tol must be positive");
  need(c.eig_block_restart >= 2, "eig: block_restart must be >= 2");
  need(c.eig_block_restart <= kLanczosMax, "eig: block_restart above the device cap (32)");
  need(c.eig_max_iters >= c.eig_block_restart, "eig: max_iters < block_restart");
  need(c.aipp_lambda0 > 0, "aipp: lambda0 must be positive");
  need(c.aipp_max_outer >= 1, "aipp: max_outer must be >= 1");
  need(c.fista_sigma > 0 && c.fista_sigma < 0.5, "fista: sigma must lie in (0, 1/2)");
  need(c.fista_chi > 0 && c.fista_chi < 1, "fista: chi must lie in (0, 1)");
  need(c.fista_mu > 0, "fista: mu must be positive");
}

const char* msg_text(int id) {
  switch (id) {
    case kMsgFistaDiverged: return "fista: curvature estimate diverged";
    case kMsgAlValue: return "al_value: non-finite result";
    case kMsgAlValGrad: return "AlFunction::value_and_gradient: non-finite result";
    case kMsgAlGrad: return "al_gradient: non-finite result";
    case kMsgGradOp: return "gradient_operator: non-finite multiplier";
    case kMsgProjectBall: return "project_ball: non-finite input";
    case kMsgNonFinite: return "non-finite iterate";
    case kMsgRankCap: return "factor rank exceeds the device cap (32)";
    case kMsgRefillCap: return "lanczos: breakdown refill / slot capacity exceeded";
    case kMsgRank32: return "factor rank above 32 is not supported";
    case kMsgFabric: return "sharded solve: a peer rank did not reach the rendezvous (timeout)";
    default: return "";
  }
}

Params base_params(cuhallar_instance* in, const cuhallar_config* cfg) {
  Params P;
  P.I = in->I;
  P.pass_scratch = in->gA ? kGprLd * kGprChunk  // staged DMMA right-hand side
                  : in->h.family == kPhaseret
                      ? int(std::max<int64_t>(2 * in->h.nc, 1024))
                      : (in->sell.col ? kPassScratch  // SELL stages (row_pass_sell_async)
                                      : std::max(kTileDoubles, kRtTheta));  // fixed-q staging has no rhs
  cuhallar_config dc;
  cuhallar_config_default(&dc);
  P.cfg = to_dev_cfg(cfg ? *cfg : dc);
  P.bar = in->bar;
  P.slots = in->slots;
  for (int i = 0; i < kNBuf; ++i) P.buf[i] = in->buf[i];
  P.vslot = in->vslot;
  P.nslot = in->nslot;
  P.lz_rand = in->lz_rand;
  P.n_refill = in->n_refill;
  if (in->svc_buf_h) {
    int* dreq = nullptr;
    int* drdy = nullptr;
    double* dbuf = nullptr;
    cudaHostGetDevicePointer(&dreq, in->svc_req_h, 0);
    cudaHostGetDevicePointer(&drdy, in->svc_ready_h, 0);
    cudaHostGetDevicePointer(&dbuf, in->svc_buf_h, 0);
    P.svc_req = dreq;
    P.svc_ready = drdy;
    P.svc_buf = dbuf;
    P.svc_err = in->svc_err_d;
  }
  P.p_up = in->p_up;
  P.p_lo = in->p_lo;
  P.q_up = in->q_up;
  P.q_lo = in->q_lo;
  P.r_up = in->r_up;
  P.r_lo = in->r_lo;
  P.p_sell = in->p_sell;
  P.q_sell = in->q_sell;
  P.r_sell = in->r_sell;
  P.pad = in->pad;
  P.scalars = in->dscal;
  P.iscalars = in->discal;
  P.trace = nullptr;
  if (in->trace_host) {
    TraceEv* dptr = nullptr;
    int* cptr = nullptr;
    cudaHostGetDevicePointer(&dptr, in->trace_host, 0);
    cudaHostGetDevicePointer(&cptr, in->trace_count_host, 0);
    P.trace = dptr;
    P.trace_count = cptr;
    P.trace_cap = in->trace_cap;
  }
  return P;
}

// Operator calls act on the instance as built (unscaled b), like the
// reference's al_value(inst, ...) / GradientOperator(inst, ...); only the
// solve works on the scaled instance b / tau (solver.cpp:31-42).
void use_unscaled_b(cuhallar_instance* in, Params& P) {
  if (in->h.has_trace || in->h.tau == 1.0) return;
  if (!in->ub_up) {
    std::vector<double> up(in->h.b.begin(), in->h.b.begin() + in->h.np);
    in->ub_up = dupload(up, &in->bytes);
  }
  if (!in->ub_lo && in->h.family != kPhaseret) {
    in->ub_lo = dalloc<double>(size_t(in->h.np), &in->bytes);
    gather_lower<<<unsigned((in->h.np + 255) / 256), 256>>>(in->ub_up, in->lo_eid, in->h.np, in->ub_lo);
    ck(cudaGetLastError(), "gather_lower");
  }
  P.I.b_up = in->ub_up;
  P.I.b_lo = in->ub_lo;
  if (in->sell.col) {
    if (!in->s_ub) {
      in->s_ub = dalloc<double>(size_t(in->sell.slots), &in->bytes);
      hd::sell_gather(in->ub_up, in->sell.eid, in->sell.slots, in->s_ub, 0);
    }
    P.I.s_b = in->s_ub;
  }
}

// Host side of the Lanczos refill protocol (solver.cuh lz_refill): while a
// launch runs, serve refill j = the j-th gaussian_vector after the start
// vector of Rng(seed ^ 0x9b97f4a7c15) (lanczos.cpp:46-50, 127-130; the
// Box-Muller spare carries over, rng.cpp:54-67), drawn once and cached.
struct RefillService {
  cuhallar_instance* in;
  std::atomic<bool> stop{false};
  std::thread th;
  explicit RefillService(cuhallar_instance* in_) : in(in_) {
    *(volatile int*)in->svc_req_h = 0;
    *(volatile int*)in->svc_ready_h = 0;
    th = std::thread([this] { run(); });
  }
  void run() {
    const int64_t n = in->h.n;
    int served = 0;
    while (!stop.load(std::memory_order_acquire)) {
      const int j = *(volatile int*)in->svc_req_h;
      if (j > in->n_refill && j != served) {
        const size_t k = size_t(j - in->n_refill - 1);
        while (in->lz_extra.size() <= k) {
          std::vector<double> v(static_cast<size_t>(n));
          for (auto& x : v) x = in->lz_gen->normal();
          in->lz_extra.push_back(std::move(v));
        }
        std::memcpy(in->svc_buf_h, in->lz_extra[k].data(), sizeof(double) * n);
        std::atomic_thread_fence(std::memory_order_seq_cst);
        *(volatile int*)in->svc_ready_h = j;
        served = j;
      } else {
        std::this_thread::sleep_for(std::chrono::microseconds(20));
      }
    }
  }
  ~RefillService() {
    stop.store(true, std::memory_order_release);
    th.join();
  }
};

// Launch the persistent kernel; returns the solver status and fills *so.
int launch(cuhallar_instance* in, Params& P, int grid, cudaStream_t st, SolveOut* so,
           float* ms, const std::function<void()>& poll) {
  ck(cudaMemsetAsync(in->bar, 0, sizeof(unsigned long long), st), "memset bar");
  ck(cudaMemsetAsync(in->dso, 0, sizeof(SolveOut), st), "memset out");
  if (in->trace_count_host) *in->trace_count_host = 0;
  SolveOut* dso = in->dso;
  void* args[] = {&P, &dso};
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ms) {
    ck(cudaEventCreate(&e0), "event");
    ck(cudaEventCreate(&e1), "event");
    ck(cudaEventRecord(e0, st), "event");
  }
  // parity mode (parity.cuh) runs in its own persistent kernel (parity_kernel.cu)
  const bool par = P.cfg.parity && (P.op == kOpSolve || P.op == kOpMinEigG || P.op == kOpAipp);
  if (par || P.fab.world > 1) {  // the SELL engine serves single-GPU fast-mode passes only
    P.I.s_col = nullptr;
    P.p_sell = P.q_sell = P.r_sell = nullptr;
    P.pad = nullptr;
    P.I.split_w = -1;  // the parity / sharded kernels keep equal tile counts
  }
  std::unique_ptr<RefillService> svc;
  if (P.svc_req && P.fab.world == 1 && (P.op == kOpSolve || P.op == kOpMinEigG || P.op == kOpAipp))
    svc = std::make_unique<RefillService>(in);
  else
    P.svc_req = nullptr;
  ck(cudaLaunchCooperativeKernel(par ? hallar_parity_kernel_fn() : (const void*)hallar_kernel,
                                 dim3(grid), dim3(kThreads), args, smem_bytes(P.pass_scratch), st),
     "cooperative launch");
  if (ms) ck(cudaEventRecord(e1, st), "event");
  if (poll) {  // e.g. trace events delivered while the solve runs (before any blocking copy)
    cudaError_t q;
    while ((q = cudaStreamQuery(st)) == cudaErrorNotReady) {
      poll();
      std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
    if (q != cudaSuccess) ck(q, "hallar_kernel");
  }
  ck(cudaMemcpyAsync(so, in->dso, sizeof(SolveOut), cudaMemcpyDeviceToHost, st), "D2H out");
  ck(cudaStreamSynchronize(st), "hallar_kernel");
  svc.reset();
  if (ms) {
    cudaEventElapsedTime(ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  return so->status;
}

int status_to_rc(int st, int msg) {
  if (st == kOk) return 0;
  g_err = msg_text(msg);
  if (st == kErrNumerical) return CUHALLAR_ERR_NUMERICAL;
  if (st == kErrInput) return CUHALLAR_ERR_INPUT;
  if (st == kErrCapacity) return CUHALLAR_ERR_CAPACITY;
  return CUHALLAR_ERR_CUDA;
}

struct DevGuard {  // run an entry point on the instance's device
  int prev = 0;
  explicit DevGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DevGuard() { cudaSetDevice(prev); }
};

template <class F>
int guard(F&& f) {
  try {
    return f();
  } catch (const hh::InputError& e) {
    g_err = e.what();
    return CUHALLAR_ERR_INPUT;
  } catch (const std::ios_base::failure& e) {
    g_err = e.what();
    return CUHALLAR_ERR_IO;
  } catch (const CudaError& e) {
    g_err = e.what();
    return CUHALLAR_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CUHALLAR_ERR_CUDA;
  }
}

cuhallar_instance* finish_pairs(hh::HostInst&& h) {
  auto in = std::make_unique<cuhallar_instance>();
  ck(cudaGetDevice(&in->device), "device");
  in->h = std::move(h);
  upload_pairs(in.get());
  return in.release();
}

// pair instance whose constraint arrays are already on the device
cuhallar_instance* finish_pairs_dev(hh::HostInst&& h, const hd::DevSamples& ds,
                                    const double* b_host = nullptr) {
  auto in = std::make_unique<cuhallar_instance>();
  ck(cudaGetDevice(&in->device), "device");
  in->h = std::move(h);
  in->h.np = ds.m;
  in->h.m = ds.m + (in->h.has_trace ? 1 : 0);
  build_pairs(in.get(), ds.ei, ds.ej, ds.b, b_host);
  return in.release();
}

hh::HostInst theta_meta(int64_t n) {
  hh::HostInst h;
  h.family = kTheta;
  h.n = n;
  h.has_trace = true;
  h.tau = 1.0;
  h.norm_b1 = 1.0;
  h.norm_C1 = double(n) * double(n);
  return h;
}

bool host_gen_forced() {
  const char* e = std::getenv("CUHALLAR_HOST_GEN");
  return e && *e && *e != '0';
}

// gen_matrix_completion (instances.cpp:131-234): hidden factors on the host,
// the sample draws on the device (devgen.cu), the host generator when the
// stream hits a uniform_below rejection or CUHALLAR_HOST_GEN=1
cuhallar_instance* gen_matcomp(int64_t n1, int64_t n2, int r, uint64_t seed, bool offset,
                               double tau_safety, int64_t paper_draws) {
  if (!host_gen_forced()) {
    auto pre = hh::matcomp_prefix(n1, n2, r, seed, offset, tau_safety, paper_draws);
    hd::DevSamples ds;
    if (hd::gen_matcomp_device(n1, n2, r, pre.state, pre.m_target, paper_draws, pre.U, pre.V, &ds, 0)) {
      hh::HostInst h;
      h.family = kMatcomp;
      h.n = n1 + n2;
      h.n1 = n1;
      h.nuclear = pre.nuclear;
      h.tau = pre.tau;
      h.norm_C1 = 0.5 * double(h.n);
      return finish_pairs_dev(std::move(h), ds);
    }
  }
  return finish_pairs(hh::make_matcomp(n1, n2, r, seed, offset, tau_safety, paper_draws));
}

// gen_phase_retrieval (instances.cpp:298-389): masks, twiddles and the
// spectrum / adjoint scratch go to HBM; b = map of the hidden signal is
// computed by the device operator itself (instances.cpp:323-328).
void upload_pr(cuhallar_instance* in);
cuhallar_instance* finish_pr(hh::HostInst&& h) {
  auto in = std::make_unique<cuhallar_instance>();
  ck(cudaGetDevice(&in->device), "device");
  in->h = std::move(h);
  upload_pr(in.get());
  return in.release();
}

// column-major (host or device) U -> buffer 0 (row-major)
void load_factor_dev(cuhallar_instance* in, const double* U_dev, int64_t ld, int s,
                     cudaStream_t st) {
  const int64_t n = in->h.n;
  const int64_t tot = n * s;
  to_rowmajor<<<unsigned((tot + 255) / 256), 256, 0, st>>>(U_dev, ld, s, n, in->buf[0]);
  ck(cudaGetLastError(), "to_rowmajor");
}
void store_factor_dev(cuhallar_instance* in, const double* src_rowmajor, int s, double* dst,
                      int64_t ld, cudaStream_t st) {
  const int64_t n = in->h.n;
  const int64_t tot = n * s;
  to_colmajor<<<unsigned((tot + 255) / 256), 256, 0, st>>>(src_rowmajor, s, n, dst, ld);
  ck(cudaGetLastError(), "to_colmajor");
}
// multiplier (length m, device) -> p_up / p_lo (+ trace scalar)
double load_multiplier_dev(cuhallar_instance* in, const double* p_dev, double* up, double* lo,
                           double* sell, cudaStream_t st) {
  const int64_t np = in->h.np;
  ck(cudaMemcpyAsync(up, p_dev, sizeof(double) * np, cudaMemcpyDeviceToDevice, st), "D2D p");
  if (in->h.family != kPhaseret) {
    gather_lower<<<unsigned((np + 255) / 256), 256, 0, st>>>(p_dev, in->lo_eid, np, lo);
    ck(cudaGetLastError(), "gather_lower");
  }
  if (sell && in->sell.col) hd::sell_gather(p_dev, in->sell.eid, in->sell.slots, sell, st);
  double pt = 0.0;
  if (in->h.has_trace)
    ck(cudaMemcpyAsync(&pt, p_dev + np, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H pt");
  ck(cudaStreamSynchronize(st), "multiplier");
  return pt;
}

}  // namespace

// ==================================================================== ABI ===
extern "C" {

const char* cuhallar_last_error(void) { return g_err.c_str(); }
const char* cuhallar_version(void) { return "cuhallar-b200 0.1.0 (sm_100a)"; }

void cuhallar_config_default(cuhallar_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->eps = 1e-5;
  c->beta_growth = 2.0;
  c->eps_decay = 0.5;
  c->max_outer = 500;
  c->time_limit = 3600.0;
  c->seed = 0;
  c->eig_tol = 1e-8;
  c->eig_max_iters = 5000;
  c->eig_block_restart = 30;
  c->aipp_lambda0 = 10.0;
  c->aipp_rho = 1e-4;
  c->aipp_max_outer = 2000;
  c->aipp_lambda_underflow = 1e-12;
  c->fista_sigma = 0.3;
  c->fista_chi = 0.5;
  c->fista_mu = 0.5;
  c->fista_L0 = 1.0;
  c->fista_max_iters = 0;
  c->max_fw_steps = 500;
}

int cuhallar_theta_hypercube(int d, cuhallar_instance** out) {
  return guard([&] {
    if (d < 1 || d >= 31) throw hh::InputError("hypercube dimension out of range");
    if (host_gen_forced()) {
      *out = finish_pairs(hh::make_theta(int64_t(1) << d, hh::edges_hypercube(d)));
    } else {
      hd::DevSamples ds;
      hd::gen_hypercube_device(d, &ds, 0);
      *out = finish_pairs_dev(theta_meta(int64_t(1) << d), ds);
    }
    return 0;
  });
}
int cuhallar_theta_cycle(int n, cuhallar_instance** out) {
  return guard([&] {
    *out = finish_pairs(hh::make_theta(n, hh::edges_cycle(n)));
    return 0;
  });
}
int cuhallar_theta_petersen(cuhallar_instance** out) {
  return guard([&] {
    *out = finish_pairs(hh::make_theta(10, hh::edges_petersen()));
    return 0;
  });
}
int cuhallar_theta_edges(int64_t n_vertices, int64_t n_pairs, const int64_t* u, const int64_t* v,
                         cuhallar_instance** out) {
  return guard([&] {
    hh::Edges raw(static_cast<size_t>(n_pairs));
    for (int64_t k = 0; k < n_pairs; ++k) raw[k] = {u[k], v[k]};
    int64_t n = 0;
    const auto e = hh::normalise_edges(n_vertices, raw, &n);
    *out = finish_pairs(hh::make_theta(n, e));
    return 0;
  });
}
int cuhallar_theta_file(const char* path, int fmt, cuhallar_instance** out) {
  return guard([&] {
    int64_t n = 0;
    const auto e = hh::edges_from_file(path, fmt, &n);
    *out = finish_pairs(hh::make_theta(n, e));
    return 0;
  });
}
int cuhallar_gen_matrix_completion(int64_t n1, int64_t n2, int r, uint64_t seed, int offset,
                                   double tau_safety, cuhallar_instance** out) {
  return guard([&] {
    *out = gen_matcomp(n1, n2, r, seed, offset != 0, tau_safety, 0);
    return 0;
  });
}
int cuhallar_gen_matrix_completion_paper(int64_t n1, int64_t n2, int r, uint64_t seed,
                                         int64_t draws, double tau_safety,
                                         cuhallar_instance** out) {
  return guard([&] {
    if (draws < 1) throw hh::InputError("matcomp: draws must be >= 1");
    *out = gen_matcomp(n1, n2, r, seed, false, tau_safety, draws);
    return 0;
  });
}
int cuhallar_matcomp_from_samples(int64_t n1, int64_t n2, int64_t m, const int64_t* i,
                                  const int64_t* j, const double* b, double tau,
                                  cuhallar_instance** out) {
  return guard([&] {
    if (!(n1 >= 1 && n2 >= 1 && n1 + n2 < (int64_t(1) << 31)))
      throw hh::InputError("matcomp samples: bad dimensions");
    if (m < 1 || m > n1 * n2) throw hh::InputError("matcomp samples: bad sample count");
    if (!(tau > 0.0 && std::isfinite(tau))) throw hh::InputError("matcomp samples: tau must be positive");
    if (!i || !j || !b) throw hh::InputError("matcomp samples: null array");
    hd::DevSamples ds;
    try {
      hd::pairs_from_host(n1, n2, m, i, j, &ds, 0);
    } catch (const std::invalid_argument& e) {
      throw hh::InputError(e.what());
    }
    hh::HostInst h;
    h.family = kMatcomp;
    h.n = n1 + n2;
    h.n1 = n1;
    h.tau = tau;
    h.norm_C1 = 0.5 * double(h.n);
    *out = finish_pairs_dev(std::move(h), ds, b);
    return 0;
  });
}
int64_t cuhallar_matcomp_constraint_count(int64_t n1, int64_t n2, int r, int offset) {
  return hh::matcomp_count(n1, n2, r, offset != 0);
}
int cuhallar_gen_phase_retrieval(int64_t n, int L, uint64_t seed, double tau_slack,
                                 cuhallar_instance** out) {
  return guard([&] {
    if (n > kPrMaxNc)
      throw hh::InputError("phaseret: n above the device transform length cap (8192)");
    *out = finish_pr(hh::make_phaseret(n, L, seed, tau_slack));
    return 0;
  });
}
int cuhallar_gen_gauss_phase_retrieval(int64_t n, int64_t m, uint64_t seed, double tau_slack,
                                       cuhallar_instance** out) {
  return guard([&] {
    if (n < 1 || m < 1 || 2 * n * m > (int64_t(1) << 36))
      throw hh::InputError("gauss_pr: n, m out of range");
    const int parts = int(std::max<int64_t>(1, std::min<int64_t>(16, m / 4096)));
    auto in = std::make_unique<cuhallar_instance>();
    ck(cudaGetDevice(&in->device), "device");
    in->h = hh::make_gauss_pr(n, m, parts, seed, tau_slack);
    upload_gpr(in.get(), seed);
    *out = in.release();
    return 0;
  });
}
int cuhallar_instance_get_gauss(const cuhallar_instance* in, double* A_re, double* A_im) {
  return guard([&] {
    if (!in->gA) throw hh::InputError("get_gauss: not a Gaussian phase-retrieval instance");
    DevGuard dg(in->device);
    const int64_t n = in->h.nc, m = in->h.m;
    std::vector<double> row(size_t(2 * n));
    for (int64_t i = 0; i < m; ++i) {
      ck(cudaMemcpy(row.data(), in->gA + i * 2 * n, 2 * n * sizeof(double), cudaMemcpyDeviceToHost), "A D2H");
      std::memcpy(A_re + i * n, row.data(), n * sizeof(double));
      std::memcpy(A_im + i * n, row.data() + n, n * sizeof(double));
    }
    return 0;
  });
}
void cuhallar_instance_destroy(cuhallar_instance* inst) { delete inst; }

int cuhallar_instance_get_info(const cuhallar_instance* in, cuhallar_instance_info* o) {
  o->n = in->h.n;
  o->m = in->h.m;
  o->identity_constraint = in->h.has_trace ? in->h.m - 1 : -1;
  o->field_kind = in->h.family == kPhaseret ? CUHALLAR_FIELD_COMPLEX_EMBEDDED : CUHALLAR_FIELD_REAL;
  o->family = in->h.family;
  o->tau = in->h.tau;
  o->norm_b1 = in->h.norm_b1;
  o->norm_C1 = in->h.norm_C1;
  o->nuclear_norm = in->h.nuclear;
  o->device_bytes = in->bytes;
  o->h2d_bytes = in->h2d;
  o->team_ctas = 0;
  try {
    o->team_ctas = grid_size(0);
  } catch (...) {
  }
  return 0;
}
int cuhallar_instance_get_b(const cuhallar_instance* in, double* b) {
  return guard([&] {
    const auto& h = in->h;
    if (int64_t(h.b.size()) == h.m) {
      std::memcpy(b, h.b.data(), sizeof(double) * h.b.size());
    } else if (h.has_trace) {  // theta: e_{m-1}
      std::memset(b, 0, sizeof(double) * h.m);
      b[h.m - 1] = 1.0;
    } else {
      DevGuard dg(in->device);
      ck(cudaMemcpy(b, in->ub_up, sizeof(double) * h.m, cudaMemcpyDeviceToHost), "b D2H");
    }
    return 0;
  });
}
int cuhallar_instance_get_pairs(const cuhallar_instance* in, int64_t* i, int64_t* j) {
  return guard([&] {
    if (in->h.family == kPhaseret) throw hh::InputError("get_pairs: not a pair instance");
    DevGuard dg(in->device);
    const int64_t np = in->h.np;
    std::vector<int32_t> a(static_cast<size_t>(np)), c(static_cast<size_t>(np));
    ck(cudaMemcpy(a.data(), in->ei, np * sizeof(int32_t), cudaMemcpyDeviceToHost), "ei D2H");
    ck(cudaMemcpy(c.data(), in->ej, np * sizeof(int32_t), cudaMemcpyDeviceToHost), "ej D2H");
    const int64_t off = in->h.family == kMatcomp ? in->h.n1 : 0;  // omega_j = j - n1
    for (int64_t k = 0; k < np; ++k) {
      i[k] = a[k];
      j[k] = c[k] - off;
    }
    return 0;
  });
}
int cuhallar_instance_get_phaseret(const cuhallar_instance* in, double* x, double* masks) {
  if (x) std::memcpy(x, in->h.hidden_x.data(), sizeof(double) * 2 * in->h.hidden_x.size());
  if (masks && !in->h.masks.empty())
    std::memcpy(masks, in->h.masks.data(), sizeof(double) * 2 * in->h.masks.size());
  return 0;
}

// --------------------------------------------------------------- operators ---
static int run_op(cuhallar_instance* in, int op, const double* U_dev, int64_t ldu, int s,
                  const double* vec_dev, double beta, double* out_vec, double* out_mat,
                  int64_t ldo, double* val_host, cudaStream_t st) {
  return guard([&] {
    DevGuard dg(in->device);
    if (s < 1 || s > kSMax) throw hh::InputError("factor rank must be in [1, 32]");
    if (ldu < in->h.n) throw hh::InputError("leading dimension < n");
    std::lock_guard<std::mutex> lk(in->mu);
    const int grid = grid_size(0);
    ensure_workspace(in, grid, 0, 30);
    Params P = base_params(in, nullptr);
    P.op = op;
    P.s_in = s;
    P.beta_in = beta;
    use_unscaled_b(in, P);
    load_factor_dev(in, U_dev, ldu, s, st);
    if (op == kOpCPlusAdj || op == kOpAdj) {
      P.q_trace_in = load_multiplier_dev(in, vec_dev, in->q_up, in->q_lo, in->q_sell, st);
    } else if (op == kOpAlValue || op == kOpAlValGrad || op == kOpAlGrad) {
      P.p_trace = load_multiplier_dev(in, vec_dev, in->p_up, in->p_lo, in->p_sell, st);
    }
    if (op == kOpMap) P.out_vec = out_vec;
    double* rm = nullptr;
    if (out_mat) {
      rm = in->buf[11];
      P.out_mat = rm;
    }
    SolveOut so{};
    const int stt = launch(in, P, grid, st, &so);
    if (stt != kOk) return status_to_rc(stt, so.msg);
    if (out_mat) {
      store_factor_dev(in, rm, s, out_mat, ldo, st);
      ck(cudaStreamSynchronize(st), "store");
    }
    if (val_host) ck(cudaMemcpy(val_host, in->dscal, sizeof(double), cudaMemcpyDeviceToHost), "val");
    return 0;
  });
}

int cuhallar_apply_map(cuhallar_instance* in, const double* U, int64_t ldu, int s, double* out,
                       cuhallar_stream st) {
  return run_op(in, kOpMap, U, ldu, s, nullptr, 0.0, out, nullptr, 0, nullptr, (cudaStream_t)st);
}
int cuhallar_apply_C(cuhallar_instance* in, const double* U, int64_t ldu, int s, double* out,
                     int64_t ldo, cuhallar_stream st) {
  return run_op(in, kOpApplyC, U, ldu, s, nullptr, 0.0, nullptr, out, ldo, nullptr,
                (cudaStream_t)st);
}
int cuhallar_apply_adjoint(cuhallar_instance* in, const double* p, const double* U, int64_t ldu,
                           int s, double* out, int64_t ldo, cuhallar_stream st) {
  return run_op(in, kOpAdj, U, ldu, s, p, 0.0, nullptr, out, ldo, nullptr, (cudaStream_t)st);
}
int cuhallar_c_plus_adjoint(cuhallar_instance* in, const double* q, const double* U, int64_t ldu,
                            int s, double* out, int64_t ldo, cuhallar_stream st) {
  return run_op(in, kOpCPlusAdj, U, ldu, s, q, 0.0, nullptr, out, ldo, nullptr, (cudaStream_t)st);
}
int cuhallar_al_value(cuhallar_instance* in, const double* U, int64_t ldu, int s, const double* p,
                      double beta, double* val, cuhallar_stream st) {
  if (!(beta > 0)) {
    g_err = "al_value: beta must be positive";
    return CUHALLAR_ERR_INPUT;
  }
  return run_op(in, kOpAlValue, U, ldu, s, p, beta, nullptr, nullptr, 0, val, (cudaStream_t)st);
}
int cuhallar_al_gradient(cuhallar_instance* in, const double* U, int64_t ldu, int s,
                         const double* p, double beta, double* grad, int64_t ldg,
                         cuhallar_stream st) {
  if (!(beta > 0)) {
    g_err = "al_gradient: beta must be positive";
    return CUHALLAR_ERR_INPUT;
  }
  return run_op(in, kOpAlGrad, U, ldu, s, p, beta, nullptr, grad, ldg, nullptr, (cudaStream_t)st);
}
int cuhallar_al_value_and_gradient(cuhallar_instance* in, const double* U, int64_t ldu, int s,
                                   const double* p, double beta, double* val, double* grad,
                                   int64_t ldg, cuhallar_stream st) {
  return run_op(in, kOpAlValGrad, U, ldu, s, p, beta, nullptr, grad, ldg, val, (cudaStream_t)st);
}

// ------------------------------------------------------------------ solve ---
static void host_factor_to_buf0(cuhallar_instance* in, const double* U_host, int s) {
  const int64_t n = in->h.n;
  std::vector<double> rm(size_t(n) * s);
  for (int64_t a = 0; a < n; ++a)
    for (int k = 0; k < s; ++k) rm[a * s + k] = U_host[a + k * n];
  ck(cudaMemcpy(in->buf[0], rm.data(), rm.size() * sizeof(double), cudaMemcpyHostToDevice), "U0");
  in->h2d += int64_t(rm.size() * sizeof(double));
}
static double host_multiplier_to_dev(cuhallar_instance* in, const double* p_host) {
  const int64_t np = in->h.np;
  if (!p_host) {  // cold start p0 = 0 (solver.cpp:126-134): no host staging
    ck(cudaMemset(in->p_up, 0, np * sizeof(double)), "p_up");
    ck(cudaMemset(in->p_lo, 0, np * sizeof(double)), "p_lo");
    if (in->p_sell) ck(cudaMemset(in->p_sell, 0, in->sell.slots * sizeof(double)), "p_sell");
    return 0.0;
  }
  ck(cudaMemcpy(in->p_up, p_host, np * sizeof(double), cudaMemcpyHostToDevice), "p_up");
  if (in->h.family != kPhaseret) {
    gather_lower<<<unsigned((np + 255) / 256), 256>>>(in->p_up, in->lo_eid, np, in->p_lo);
    ck(cudaGetLastError(), "gather_lower");
    if (in->p_sell) hd::sell_gather(in->p_up, in->sell.eid, in->sell.slots, in->p_sell, 0);
  }
  in->h2d += int64_t(np * sizeof(double));
  return (in->h.has_trace && p_host) ? p_host[np] : 0.0;
}

static int fill_report(cuhallar_instance* in, const SolveOut& so, float ms, double wall,
                       cuhallar_report* rep, cuhallar_solution** sol,
                       const std::vector<cuhallar_instance*>& ranks);

// Start point into buffer 0: warm-start factor, or u0 = gaussian_vector(n,
// Rng(seed)) / |u0| (solver.cpp:126-134).  Returns its rank.
static int upload_start(cuhallar_instance* in, const cuhallar_config* cfg, const double* U0_host,
                        int s0) {
  const int64_t n = in->h.n;
  if (U0_host) {
    if (s0 < 1 || s0 > kSMax) throw hh::InputError("solve: warm-start rank must be in [1, 32]");
    std::vector<double> tmp(U0_host, U0_host + n * s0);
    const double nrm = std::sqrt(hh::eigen_order_sum_sq(tmp.data(), n * s0));
    if (!(nrm <= 1.0 + 1e-12)) throw hh::InputError("solve: warm-start factor outside unit ball");
    host_factor_to_buf0(in, U0_host, s0);
    return s0;
  }
  std::vector<double> u0 = hh::gaussian_stream(cfg->seed, n);
  const double nu = std::sqrt(hh::eigen_order_sum_sq(u0.data(), n));
  for (auto& x : u0) x = x / nu;
  ck(cudaMemcpy(in->buf[0], u0.data(), n * sizeof(double), cudaMemcpyHostToDevice), "U0");
  in->h2d += int64_t(n * sizeof(double));
  return 1;
}

int cuhallar_solve(cuhallar_instance* in, const cuhallar_config* cfg, const double* U0_host,
                   int s0, const double* p0_host, cuhallar_report* rep, cuhallar_solution** sol,
                   cuhallar_trace_fn fn, void* user) {
  return guard([&] {
    DevGuard dg(in->device);
    validate_cfg(*cfg);
    if (cfg->parity && in->h.family == kPhaseret)
      throw hh::InputError("parity mode: pair families only (theta, matrix completion)");
    std::lock_guard<std::mutex> lk(in->mu);
    const auto t_start = std::chrono::steady_clock::now();
    const int64_t n = in->h.n;
    const int grid = grid_size(cfg->team_ctas);
    ensure_workspace(in, grid, cfg->seed, cfg->eig_block_restart);
    const int s = upload_start(in, cfg, U0_host, s0);
    if (cfg->trace && !in->trace_host) {  // TraceEvent ring, mapped host memory (lazy)
      ck(cudaHostAlloc(&in->trace_host, sizeof(TraceEv) * in->trace_cap, cudaHostAllocMapped),
         "trace ring");
      ck(cudaHostAlloc(&in->trace_count_host, sizeof(int), cudaHostAllocMapped), "trace count");
    }
    Params P = base_params(in, cfg);
    P.op = kOpSolve;
    P.s_in = s;
    P.p_trace = host_multiplier_to_dev(in, p0_host);
    if (cfg->profile) {
      if (!in->dprof) in->dprof = dalloc<unsigned long long>(2 * kProfCats, &in->bytes);
      ck(cudaMemset(in->dprof, 0, sizeof(unsigned long long) * 2 * kProfCats), "prof");
      P.prof = in->dprof;
    }
    SolveOut so{};
    float ms = 0.f;
    // trace.hpp sinks see the events while the solve runs (the ring is mapped
    // host memory; an event is complete once the count has moved past it)
    int delivered = 0;
    auto deliver = [&](bool all) {
      if (!fn || !cfg->trace) return;
      int cnt = std::min(static_cast<int>(*(volatile int*)in->trace_count_host), in->trace_cap);
      if (!all) cnt = std::max(delivered, cnt - 1);
      for (; delivered < cnt; ++delivered) {
        const TraceEv& e = in->trace_host[delivered];
        cuhallar_trace_event ev{e.kind, e.outer_iter, e.beta, e.eps_inner, e.gap, e.theta,
                                e.rank, e.al_value, e.fw_alpha, e.rel_pfeas, e.rel_gap,
                                e.rel_dfeas};
        fn(&ev, user);
      }
    };
    const int stt = launch(in, P, grid, 0, &so, &ms, [&] { deliver(false); });
    if (cfg->profile) {
      in->last_prof.assign(2 * kProfCats, 0);
      ck(cudaMemcpy(in->last_prof.data(), in->dprof, sizeof(unsigned long long) * 2 * kProfCats,
                    cudaMemcpyDeviceToHost),
         "prof D2H");
    }
    const double wall =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    deliver(true);
    (void)stt;
    (void)n;
    return fill_report(in, so, ms, wall, rep, sol, {in});
  });
}

// The SolveOut of a finished solve -> SolveReport (tau rescaling as finish(),
// solver.cpp:175-202) and, on request, the solution.  For a sharded solve,
// ranks[r] holds the multiplier entries of its rows; U is complete on rank 0.
static int fill_report(cuhallar_instance* in, const SolveOut& so, float ms, double wall,
                       cuhallar_report* rep, cuhallar_solution** sol,
                       const std::vector<cuhallar_instance*>& ranks) {
  {
    const int stt = so.status;
    const int64_t n = in->h.n;
    if (stt != 0 && stt != 1 && stt != 2 && stt != 3) return status_to_rc(stt, so.msg);
    if (so.status == kErrInput || so.status == kErrCapacity) return status_to_rc(so.status, so.msg);
    const double tau = in->h.tau;
    std::memset(rep, 0, sizeof(*rep));
    rep->status = so.status;
    rep->pval = tau * so.pval;
    rep->dval = tau * so.dval;
    rep->dval_no_theta = tau * so.dval_no_theta;
    rep->rel_pfeas = so.rel_pfeas;
    rep->rel_gap = so.rel_gap;
    rep->rel_dfeas = so.rel_dfeas;
    rep->rank = so.rank;
    rep->outer_iters = so.outer_iters;
    rep->fw_steps = so.fw_steps;
    rep->aipp_iters = so.aipp_iters;
    rep->fista_iters = so.fista_iters;
    rep->eig_products = so.eig_products;
    rep->wall_seconds = wall;
    rep->device_seconds = ms * 1e-3;
    rep->tau = tau;
    rep->theta = so.theta;
    rep->trace_dropped = in->trace_count_host ? std::max(0, *in->trace_count_host - in->trace_cap) : 0;
    std::snprintf(rep->message, sizeof(rep->message), "%s", msg_text(so.msg));
    if (sol) {
      auto S = std::make_unique<cuhallar_solution>();
      S->n = n;
      S->m = in->h.m;
      S->rank = so.rank;
      std::vector<double> rm(size_t(n) * so.rank);
      ck(cudaMemcpy(rm.data(), in->buf[so.out_buf], rm.size() * sizeof(double),
                    cudaMemcpyDeviceToHost),
         "U out");
      S->U.resize(rm.size());
      for (int64_t a = 0; a < n; ++a)
        for (int k = 0; k < so.rank; ++k) S->U[a + k * n] = rm[a * so.rank + k];
      const int world = int(ranks.size());
      if (world == 1) {
        S->np = in->h.np;
        S->has_trace = in->h.has_trace != 0;
        S->p_trace = so.p_trace;
        S->device = in->device;
        ck(cudaMalloc(&S->p_dev, std::max<int64_t>(1, in->h.np) * sizeof(double)), "p out");
        ck(cudaMemcpy(S->p_dev, in->p_up, in->h.np * sizeof(double), cudaMemcpyDeviceToDevice), "p out");
      } else {
        S->p.resize(in->h.m);
        const int64_t nt = int64_t(in->tile_row_host.size()) - 1;
        for (int r = 0; r < world; ++r) {
          const int64_t rl = in->tile_row_host[nt * r / world];
          const int64_t rh = in->tile_row_host[nt * (r + 1) / world];
          const int64_t k0 = in->up_ptr_host[rl], k1 = in->up_ptr_host[rh];
          DevGuard dg(ranks[r]->device);
          if (k1 > k0)
            ck(cudaMemcpy(S->p.data() + k0, ranks[r]->p_up + k0, (k1 - k0) * sizeof(double),
                          cudaMemcpyDeviceToHost),
               "p out");
        }
      }
      if (in->h.has_trace && world > 1) S->p[in->h.np] = so.p_trace;
      *sol = S.release();
    }
    return 0;
  }
}

int cuhallar_solve_sharded(cuhallar_instance* const* insts, int world, const cuhallar_config* cfg,
                           const double* U0_host, int s0, const double* p0_host,
                           cuhallar_report* rep, cuhallar_solution** sol) {
  return guard([&] {
    if (world < 1 || world > kMaxWorld) throw hh::InputError("sharded solve: world must lie in [1, 8]");
    validate_cfg(*cfg);
    if (cfg->parity) throw hh::InputError("parity mode: single-GPU solve only");
    std::vector<cuhallar_instance*> R(insts, insts + world);
    for (int r = 0; r < world; ++r) {
      if (!R[r]) throw hh::InputError("sharded solve: null instance");
      if (R[r]->h.family == kPhaseret)
        throw hh::InputError("sharded solve: phase retrieval does not shard (replicas only)");
      if (R[r]->h.n != R[0]->h.n || R[r]->h.m != R[0]->h.m || R[r]->h.np != R[0]->h.np ||
          R[r]->tile_row_host != R[0]->tile_row_host)
        throw hh::InputError("sharded solve: ranks hold different instances");
      for (int q = 0; q < r; ++q)
        if (R[q] == R[r]) throw hh::InputError("sharded solve: one instance per rank");
    }
    std::vector<std::unique_lock<std::mutex>> locks;
    for (auto* in : R) locks.emplace_back(in->mu);
    int prev = 0;
    ck(cudaGetDevice(&prev), "device");
    struct Restore {
      int d;
      ~Restore() { cudaSetDevice(d); }
    } restore{prev};
    const auto t_start = std::chrono::steady_clock::now();
    // peer access between distinct devices (NVLink / NVSwitch)
    std::vector<int> share(world, 0);
    for (int r = 0; r < world; ++r)
      for (int q = 0; q < world; ++q) {
        if (R[q]->device == R[r]->device) {
          ++share[r];
          continue;
        }
        int ok = 0;
        ck(cudaDeviceCanAccessPeer(&ok, R[r]->device, R[q]->device), "peer query");
        if (!ok) throw CudaError("sharded solve: devices without peer access");
        ck(cudaSetDevice(R[r]->device), "device");
        const cudaError_t e = cudaDeviceEnablePeerAccess(R[q]->device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else ck(e, "peer enable");
      }
    // equal team per rank; ranks sharing a device split its SMs (co-resident launches)
    int G = kMaxTeam;
    for (int r = 0; r < world; ++r) {
      ck(cudaSetDevice(R[r]->device), "device");
      G = std::min(G, grid_size(0) / share[r]);
    }
    if (cfg->team_ctas > 0) G = std::min(G, cfg->team_ctas);
    if (G < 1) throw CudaError("sharded solve: not enough SMs for the ranks");
    int s = 1;
    for (int r = 0; r < world; ++r) {  // every rank's state exists before any Params is built
      cuhallar_instance* in = R[r];
      ck(cudaSetDevice(in->device), "device");
      ensure_workspace(in, G, cfg->seed, cfg->eig_block_restart);
      if (!in->xbar) {
        in->xbar = dalloc<unsigned long long>(1, &in->bytes);
        in->xslots = dalloc<double>(size_t(2) * kMaxWorld * kRedK, &in->bytes);
        in->xerr = dalloc<int>(1, &in->bytes);
      }
      ck(cudaMemset(in->xbar, 0, sizeof(unsigned long long)), "xbar");
      ck(cudaMemset(in->xerr, 0, sizeof(int)), "xerr");
    }
    std::vector<Params> Ps(world);
    for (int r = 0; r < world; ++r) {
      cuhallar_instance* in = R[r];
      ck(cudaSetDevice(in->device), "device");
      s = upload_start(in, cfg, U0_host, s0);
      Params& P = Ps[r];
      P = base_params(in, cfg);
      P.op = kOpSolve;
      P.s_in = s;
      P.p_trace = host_multiplier_to_dev(in, p0_host);
      P.fab.world = world;
      P.fab.me = r;
      P.I.s_col = nullptr;  // row-owner sharding keeps the CSR engines
      P.I.split_w = -1;
      P.p_sell = P.q_sell = P.r_sell = nullptr;
      P.svc_req = nullptr;  // refills: the pre-drawn ones only
      P.fab.arena_len = in->arena_len;
      P.fab.xerr = in->xerr;
      for (int q = 0; q < world; ++q) {
        P.fab.xbar[q] = R[q]->xbar;
        P.fab.xslots[q] = R[q]->xslots;
        P.fab.arena[q] = R[q]->arena;
      }
    }
    // all ranks in flight before any wait: the team needs every launch resident
    std::vector<cudaStream_t> st(world);
    std::vector<cudaEvent_t> e0(world), e1(world);
    for (int r = 0; r < world; ++r) {
      cuhallar_instance* in = R[r];
      ck(cudaSetDevice(in->device), "device");
      ck(cudaStreamCreateWithFlags(&st[r], cudaStreamNonBlocking), "stream");
      ck(cudaEventCreate(&e0[r]), "event");
      ck(cudaEventCreate(&e1[r]), "event");
      ck(cudaMemsetAsync(in->bar, 0, sizeof(unsigned long long), st[r]), "bar");
      ck(cudaMemsetAsync(in->dso, 0, sizeof(SolveOut), st[r]), "dso");
      if (in->trace_count_host) *in->trace_count_host = 0;
      ck(cudaEventRecord(e0[r], st[r]), "event");
      SolveOut* dso = in->dso;
      void* args[] = {&Ps[r], &dso};
      ck(cudaLaunchCooperativeKernel((void*)hallar_kernel, dim3(G), dim3(kThreads), args,
                                     smem_bytes(Ps[r].pass_scratch), st[r]),
         "cooperative launch (sharded)");
      ck(cudaEventRecord(e1[r], st[r]), "event");
    }
    float ms = 0.f;
    int xerr = 0;
    for (int r = 0; r < world; ++r) {
      ck(cudaSetDevice(R[r]->device), "device");
      ck(cudaStreamSynchronize(st[r]), "hallar_kernel (sharded)");
      float t = 0.f;
      ck(cudaEventElapsedTime(&t, e0[r], e1[r]), "event");
      ms = std::max(ms, t);  // device time of the solve = max over ranks
      int e = 0;
      ck(cudaMemcpy(&e, R[r]->xerr, sizeof(int), cudaMemcpyDeviceToHost), "xerr");
      xerr |= e;
      cudaEventDestroy(e0[r]);
      cudaEventDestroy(e1[r]);
      cudaStreamDestroy(st[r]);
    }
    ck(cudaSetDevice(R[0]->device), "device");
    SolveOut so{};
    ck(cudaMemcpy(&so, R[0]->dso, sizeof(SolveOut), cudaMemcpyDeviceToHost), "D2H out");
    if (xerr && so.status == kOk) {
      so.status = kErrFabric;
      so.msg = kMsgFabric;
    }
    const double wall =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    return fill_report(R[0], so, ms, wall, rep, sol, R);
  });
}

// ---- one process per GPU (torchrun): the same row-owner sharded solve with
// the peers' rendezvous counters, partial slots and factor arenas mapped
// through CUDA IPC handles instead of one process's peer pointers.
int cuhallar_shard_export(cuhallar_instance* in, int team_ctas, cuhallar_shard_handle* out) {
  return guard([&] {
    DevGuard dg(in->device);
    if (in->h.family == kPhaseret)
      throw hh::InputError("sharded solve: phase retrieval does not shard (replicas only)");
    std::lock_guard<std::mutex> lk(in->mu);
    const int G = grid_size(team_ctas);
    ensure_workspace(in, G, in->lz_seed == ~0ull ? 0 : in->lz_seed, 30);
    if (!in->xbar) {
      in->xbar = dalloc<unsigned long long>(1, &in->bytes);
      in->xslots = dalloc<double>(size_t(2) * kMaxWorld * kRedK, &in->bytes);
      in->xerr = dalloc<int>(1, &in->bytes);
    }
    std::memset(out, 0, sizeof(*out));
    cudaIpcMemHandle_t h[3];
    ck(cudaIpcGetMemHandle(&h[0], in->xbar), "ipc xbar");
    ck(cudaIpcGetMemHandle(&h[1], in->xslots), "ipc xslots");
    ck(cudaIpcGetMemHandle(&h[2], in->arena), "ipc arena");
    static_assert(3 * sizeof(cudaIpcMemHandle_t) + 32 <= sizeof(out->bytes), "handle blob");
    std::memcpy(out->bytes, h, sizeof(h));
    int64_t meta[4] = {in->h.n, in->h.np, in->arena_len, G};
    std::memcpy(out->bytes + sizeof(h), meta, sizeof(meta));
    return 0;
  });
}

int cuhallar_solve_rank(cuhallar_instance* in, int world, int rank, const cuhallar_shard_handle* peers,
                        const cuhallar_config* cfg, const double* U0_host, int s0,
                        const double* p0_host, cuhallar_report* rep, cuhallar_solution** sol) {
  return guard([&] {
    if (world < 1 || world > kMaxWorld) throw hh::InputError("sharded solve: world must lie in [1, 8]");
    if (rank < 0 || rank >= world) throw hh::InputError("sharded solve: rank out of range");
    validate_cfg(*cfg);
    if (cfg->parity) throw hh::InputError("parity mode: single-GPU solve only");
    DevGuard dg(in->device);
    std::lock_guard<std::mutex> lk(in->mu);
    if (!in->xbar) throw hh::InputError("sharded solve: cuhallar_shard_export first");
    int64_t meta0[4];
    std::memcpy(meta0, peers[0].bytes + 3 * sizeof(cudaIpcMemHandle_t), sizeof(meta0));
    const int G = int(meta0[3]);
    for (int q = 0; q < world; ++q) {
      int64_t mq[4];
      std::memcpy(mq, peers[q].bytes + 3 * sizeof(cudaIpcMemHandle_t), sizeof(mq));
      if (mq[0] != in->h.n || mq[1] != in->h.np || mq[2] != in->arena_len || mq[3] != G)
        throw hh::InputError("sharded solve: ranks hold different instances or team sizes");
    }
    ensure_workspace(in, G, cfg->seed, cfg->eig_block_restart);
    std::vector<void*> opened;
    struct Close {
      std::vector<void*>& v;
      ~Close() {
        for (void* p : v) cudaIpcCloseMemHandle(p);
      }
    } closer{opened};
    Params P = base_params(in, cfg);
    P.op = kOpSolve;
    P.s_in = upload_start(in, cfg, U0_host, s0);
    P.p_trace = host_multiplier_to_dev(in, p0_host);
    P.fab.world = world;
    P.fab.me = rank;
    P.fab.arena_len = in->arena_len;
    P.fab.xerr = in->xerr;
    P.I.s_col = nullptr;  // row-owner sharding keeps the CSR engines
      P.I.split_w = -1;
    P.p_sell = P.q_sell = P.r_sell = nullptr;
    P.svc_req = nullptr;
    for (int q = 0; q < world; ++q) {
      if (q == rank) {
        P.fab.xbar[q] = in->xbar;
        P.fab.xslots[q] = in->xslots;
        P.fab.arena[q] = in->arena;
        continue;
      }
      cudaIpcMemHandle_t h[3];
      std::memcpy(h, peers[q].bytes, sizeof(h));
      void* ptr[3];
      for (int t = 0; t < 3; ++t) {
        ck(cudaIpcOpenMemHandle(&ptr[t], h[t], cudaIpcMemLazyEnablePeerAccess), "ipc open");
        opened.push_back(ptr[t]);
      }
      P.fab.xbar[q] = static_cast<unsigned long long*>(ptr[0]);
      P.fab.xslots[q] = static_cast<double*>(ptr[1]);
      P.fab.arena[q] = static_cast<double*>(ptr[2]);
    }
    ck(cudaMemset(in->xerr, 0, sizeof(int)), "xerr");
    const auto t_start = std::chrono::steady_clock::now();
    float ms = 0.f;
    SolveOut so{};
    launch(in, P, G, 0, &so, &ms);
    int xe = 0;
    ck(cudaMemcpy(&xe, in->xerr, sizeof(int), cudaMemcpyDeviceToHost), "xerr");
    if (xe && so.status == kOk) {
      so.status = kErrFabric;
      so.msg = kMsgFabric;
    }
    const double wall =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    std::vector<cuhallar_instance*> me{in};
    return fill_report(in, so, ms, wall, rep, sol, me);
  });
}

int cuhallar_last_trace(const cuhallar_instance* in, cuhallar_trace_event* out, int cap) {
  if (!in->trace_host || !in->trace_count_host) return 0;
  const int cnt = std::min(std::min(*in->trace_count_host, in->trace_cap), cap);
  for (int i = 0; i < cnt; ++i) {
    const TraceEv& e = in->trace_host[i];
    out[i] = cuhallar_trace_event{e.kind, e.outer_iter, e.beta, e.eps_inner, e.gap, e.theta,
                                  e.rank, e.al_value, e.fw_alpha, e.rel_pfeas, e.rel_gap,
                                  e.rel_dfeas};
  }
  return cnt;
}

int cuhallar_last_profile(const cuhallar_instance* in, double* ns, int64_t* counts, int cap) {
  if (in->last_prof.empty()) return 0;
  const int k = std::min<int>(cap, kProfCats);
  for (int i = 0; i < k; ++i) {
    ns[i] = double(in->last_prof[i]);
    counts[i] = int64_t(in->last_prof[kProfCats + i]);
  }
  return k;
}

int cuhallar_solution_get_U(const cuhallar_solution* s, double* U) {
  std::memcpy(U, s->U.data(), s->U.size() * sizeof(double));
  return 0;
}
int cuhallar_solution_get_p(const cuhallar_solution* s, double* p) {
  return guard([&] {
    if (s->p_dev) {
      DevGuard dg(s->device);
      ck(cudaMemcpy(p, s->p_dev, s->np * sizeof(double), cudaMemcpyDeviceToHost), "p out");
      if (s->has_trace) p[s->np] = s->p_trace;
    } else {
      std::memcpy(p, s->p.data(), s->p.size() * sizeof(double));
    }
    return 0;
  });
}
void cuhallar_solution_destroy(cuhallar_solution* s) { delete s; }

static int min_eig_impl(cuhallar_instance* in, const double* U_host, int s, const double* p_host,
                        double beta, double tol, int max_iters, int block_restart, uint64_t seed,
                        int parity, double* lambda, double* v_host, double* residual,
                        int* matvecs, int* converged) {
  return guard([&] {
    if (parity && in->h.family == kPhaseret)
      throw hh::InputError("parity mode: pair families only (theta, matrix completion)");
    DevGuard dg(in->device);
    if (s < 1 || s > kSMax) throw hh::InputError("factor rank must be in [1, 32]");
    if (block_restart < 2 || block_restart > kLanczosMax)
      throw hh::InputError("eig: block_restart must lie in [2, 32]");
    std::lock_guard<std::mutex> lk(in->mu);
    const int grid = grid_size(0);
    ensure_workspace(in, grid, seed, block_restart);
    cuhallar_config cfg;
    cuhallar_config_default(&cfg);
    cfg.eig_max_iters = max_iters;
    cfg.eig_block_restart = block_restart;
    cfg.parity = parity;
    Params P = base_params(in, &cfg);
    P.op = kOpMinEigG;
    use_unscaled_b(in, P);
    P.s_in = s;
    P.beta_in = beta;
    P.rho_in = tol;
    host_factor_to_buf0(in, U_host, s);
    P.p_trace = host_multiplier_to_dev(in, p_host);
    double* vout = in->buf[11];
    P.out_vec = vout;
    SolveOut so{};
    const int stt = launch(in, P, grid, 0, &so);
    if (stt != kOk) return status_to_rc(stt, so.msg);
    double sc[2];
    int isc[2];
    ck(cudaMemcpy(sc, in->dscal, sizeof(sc), cudaMemcpyDeviceToHost), "scalars");
    ck(cudaMemcpy(isc, in->discal, sizeof(isc), cudaMemcpyDeviceToHost), "iscalars");
    *lambda = sc[0];
    *residual = sc[1];
    *matvecs = isc[0];
    *converged = isc[1];
    if (v_host) ck(cudaMemcpy(v_host, vout, in->h.n * sizeof(double), cudaMemcpyDeviceToHost), "v");
    return 0;
  });
}

int cuhallar_min_eig_gradient(cuhallar_instance* in, const double* U_host, int s,
                              const double* p_host, double beta, double tol, int max_iters,
                              int block_restart, uint64_t seed, double* lambda, double* v_host,
                              double* residual, int* matvecs, int* converged) {
  return min_eig_impl(in, U_host, s, p_host, beta, tol, max_iters, block_restart, seed, 0, lambda,
                      v_host, residual, matvecs, converged);
}

int cuhallar_min_eig_gradient_cfg(cuhallar_instance* in, const double* U_host, int s,
                                  const double* p_host, double beta, double tol,
                                  const cuhallar_config* cfg, double* lambda, double* v_host,
                                  double* residual, int* matvecs, int* converged) {
  return min_eig_impl(in, U_host, s, p_host, beta, tol, cfg->eig_max_iters, cfg->eig_block_restart,
                      cfg->seed, cfg->parity, lambda, v_host, residual, matvecs, converged);
}

int cuhallar_aipp(cuhallar_instance* in, const double* p_host, double beta, const double* W_host,
                  int s, double rho, const cuhallar_config* cfg, double* W_out, int* status,
                  int* prox_iters, int* fista_iters, double* R_norm, double* g_value,
                  double* lambda) {
  return guard([&] {
    DevGuard dg(in->device);
    if (s < 1 || s > kSMax) throw hh::InputError("factor rank must be in [1, 32]");
    if (cfg && cfg->parity && in->h.family == kPhaseret)
      throw hh::InputError("parity mode: pair families only (theta, matrix completion)");
    std::lock_guard<std::mutex> lk(in->mu);
    const int grid = grid_size(cfg ? cfg->team_ctas : 0);
    ensure_workspace(in, grid, 0, 30);
    if (cfg && cfg->trace && !in->trace_host) {
      ck(cudaHostAlloc(&in->trace_host, sizeof(TraceEv) * in->trace_cap, cudaHostAllocMapped),
         "trace ring");
      ck(cudaHostAlloc(&in->trace_count_host, sizeof(int), cudaHostAllocMapped), "trace count");
    }
    Params P = base_params(in, cfg);
    P.op = kOpAipp;
    use_unscaled_b(in, P);
    P.s_in = s;
    P.beta_in = beta;
    P.rho_in = rho;
    host_factor_to_buf0(in, W_host, s);
    P.p_trace = host_multiplier_to_dev(in, p_host);
    double* wout = in->buf[11];
    P.out_mat = wout;
    SolveOut so{};
    const int stt = launch(in, P, grid, 0, &so);
    if (stt != kOk) return status_to_rc(stt, so.msg);
    double sc[3];
    int isc[3];
    ck(cudaMemcpy(sc, in->dscal, sizeof(sc), cudaMemcpyDeviceToHost), "scalars");
    ck(cudaMemcpy(isc, in->discal, sizeof(isc), cudaMemcpyDeviceToHost), "iscalars");
    *R_norm = sc[0];
    *g_value = sc[1];
    *lambda = sc[2];
    *status = isc[0];
    *prox_iters = isc[1];
    *fista_iters = isc[2];
    std::vector<double> rm(size_t(in->h.n) * s);
    ck(cudaMemcpy(rm.data(), wout, rm.size() * sizeof(double), cudaMemcpyDeviceToHost), "W");
    for (int64_t a = 0; a < in->h.n; ++a)
      for (int k = 0; k < s; ++k) W_out[a + k * in->h.n] = rm[a * s + k];
    return 0;
  });
}

int cuhallar_bench_pass(cuhallar_instance* in, int kind, const double* U_host, int s,
                        const double* p_host, double beta, int iters, int team_ctas,
                        double* ns_per_pass) {
  return guard([&] {
    DevGuard dg(in->device);
    if (s < 1 || s > kSMax) throw hh::InputError("factor rank must be in [1, 32]");
    std::lock_guard<std::mutex> lk(in->mu);
    const int grid = grid_size(team_ctas);
    ensure_workspace(in, grid, 0, 30);
    Params P = base_params(in, nullptr);
    P.op = kOpBench;
    P.bench_kind = kind;
    P.bench_iters = iters;
    P.s_in = s;
    P.beta_in = beta;
    host_factor_to_buf0(in, U_host, s);
    P.p_trace = host_multiplier_to_dev(in, p_host);
    P.out_mat = in->buf[11];
    SolveOut so{};
    const int stt = launch(in, P, grid, 0, &so);
    if (stt != kOk) return status_to_rc(stt, so.msg);
    ck(cudaMemcpy(ns_per_pass, in->dscal, sizeof(double), cudaMemcpyDeviceToHost), "ns");
    return 0;
  });
}

}  // extern "C"
