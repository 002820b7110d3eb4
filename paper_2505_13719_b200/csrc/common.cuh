// Shared host/device definitions for the B200 HALLaR solver.
#pragma once

#include <cstdint>

namespace hallar {

constexpr int kThreads = 512;            // threads per persistent CTA
constexpr int kWarps = kThreads / 32;
constexpr int kSMax = 32;                // max factor rank (one lane per column)
constexpr int kLanczosMax = 32;          // max Lanczos basis (block_restart cap)
constexpr int kRedK = 40;                // max values per team reduction
constexpr int kNBuf = 12;                // n x kSMax factor buffers in the pool
constexpr int kTile = 8;                 // columns per fold chunk
constexpr int kMaxTeam = 320;            // max persistent CTAs (team reduction width)
constexpr int kGroups = 4;               // independent 128-thread tile groups per CTA
constexpr int kGT = kThreads / kGroups;  // threads per tile group
constexpr int kTileEntries = 512;        // entries per row tile (per group)
constexpr int kTileRows = 32;            // rows per row tile
constexpr int kPrMaxNc = 8192;           // phase retrieval: transform length held in smem
// shared scratch of one pass: the tile engine's arrays or one complex transform
constexpr int kTileDoubles = kGroups * (5 * kTileEntries + 4 * (kTileRows + 1) + kTileEntries / 2);
constexpr int kPassScratch0 = kTileDoubles > 2 * kPrMaxNc ? kTileDoubles : 2 * kPrMaxNc;
constexpr int kPassScratch = kPassScratch0;
constexpr int kRtMinRows = 2 * kThreads; // rows per CTA from which the row-thread engine runs
// Small instances: a CTA's static structure (row pointers, tile starts and the
// column index of every entry it folds) is cached in shared memory for the
// whole launch, removing two dependent global round trips from every row pass.
constexpr int kCacheEnt = 3072;          // entries (int32 columns)
constexpr int kCacheRows = 1024;         // rows (+1 pointers, lower and upper)
constexpr int kCacheTiles = 32;          // tiles (+1 starts)
constexpr int kCacheInts = kCacheEnt + 2 * (kCacheRows + 1) + (kCacheTiles + 1) + 1;
// fixed-q row-thread staging: col [2][8][threads] int32 + q [2][8][threads] f64
constexpr int kRtTheta = 2 * 8 * kThreads / 2 + 2 * 8 * kThreads;

enum Family : int { kTheta = 0, kMatcomp = 1, kPhaseret = 2 };

// Row-sharded solve across GPUs: one persistent launch per
// rank; the ranks address each other's memory through peer pointers.
constexpr int kMaxWorld = 8;
struct Fabric {
  int world = 1, me = 0;
  unsigned long long* xbar[kMaxWorld] = {};  // rank-rendezvous counter on each rank
  double* xslots[kMaxWorld] = {};            // [2][kMaxWorld][kRedK] per-rank partials on each rank
  double* arena[kMaxWorld] = {};             // replicated factor arena on each rank
  int64_t arena_len = 0;                     // doubles
  int* xerr = nullptr;                       // this rank's error flag (rendezvous timeout)
  unsigned long long timeout_ns = 20000000000ull;
};

// Optional in-solve phase profile (CTA 0's %globaltimer between phase ends).
enum ProfCat : int {
  kPfT1 = 0, kPfT2, kPfT34, kPfT5, kPfAipp, kPfLzApply, kPfLzCgs, kPfJacobi, kPfLzMeasure,
  kPfLzRestart, kPfGradop, kPfGap, kPfFwStep, kPfOuter, kPfOther, kProfCats
};

enum Status : int {
  kOk = 0,
  kErrInput = 64,
  kErrNumerical = 3,
  kErrCapacity = 65,  // rank or Lanczos refill capacity exceeded
  kErrFabric = 71,    // sharded team: a peer rank did not arrive
};

// Pair-constraint instance as resident in HBM (theta / graph / matcomp).
// Constraints k < np are X_{ei[k], ej[k]} with ei < ej, sorted by (ei, ej);
// theta adds the trace constraint k = np (= m-1).  Rows are vertices.
//   upper CSR: row a owns edges k in [up_ptr[a], up_ptr[a+1]) (ei[k] == a)
//   lower CSR: row a owns lo entries e in [lo_ptr[a], lo_ptr[a+1]) with
//              lo_col[e] = ei[k], lo_eid[e] = k, ej[k] == a, sorted by k.
// Every lower k of row a precedes every upper k of row a, so folding lower
// then upper entries reproduces the reference's increasing-k accumulation
// order (instances.cpp:45-52).
struct DevPairs {
  int family = kTheta;
  int has_trace = 0;
  int64_t n = 0, np = 0, m = 0;
  const int32_t* ei = nullptr;
  const int32_t* ej = nullptr;
  const int64_t* up_ptr = nullptr;
  const int64_t* lo_ptr = nullptr;
  const int32_t* lo_col = nullptr;
  const int64_t* lo_eid = nullptr;
  const double* b_up = nullptr;  // scaled b (edge order), null = all zero
  const double* b_lo = nullptr;  // scaled b (lower order)
  double b_trace = 0.0;          // scaled b[m-1] (theta)
  const int64_t* tile_row = nullptr;  // [ntiles+1] first row of each row tile
  int64_t ntiles = 0;
  double norm_b1 = 0.0, nb2 = 0.0, norm_C1 = 0.0;  // scaled instance norms
  // SELL-32 copy of the merged row streams for the single-GPU row passes:
  // slice t = rows [32t, 32t + 32); entry v of row a (its lower entries, then
  // its upper entries, increasing k) sits at slot s_off[a / 32] + 32 v + a % 32,
  // so a warp reading entry v of its 32 rows touches 32 consecutive slots.
  const int64_t* s_off = nullptr;   // [nslices + 1]
  const int32_t* s_col = nullptr;   // slot -> gathered row (null: no SELL copy)
  const int32_t* s_nlo = nullptr;   // [n] lower entries of each row
  const int32_t* s_nv = nullptr;    // [n] entries of each row
  const double* s_b = nullptr;      // slot -> scaled b (matrix completion)
  const uint32_t* s_eid = nullptr;  // slot -> edge id (padding 0xffffffff)
  int64_t s_slots = 0;
  // matrix completion: slices [0, s_up_slices) hold every upper entry (rows
  // i_k < n1), later slices none (the row-ordered map pass); 0 = not used
  int64_t s_up_slices = 0;
  // CTA row split (one GPU, SELL instances): < 0 = equal tile counts; >= 0 =
  // equal cost, cost(rows [0, r)) = entries + split_w * r (kernel_setup.cuh)
  int split_w = -1;
  // phase retrieval (family kPhaseret): np = m, b_up = b (constraint order)
  int64_t nc = 0;                 // complex dimension (n = 2 nc)
  int L = 0, lognc = 0;           // masks, log2(nc)
  const double2* masks = nullptr; // nc x L column-major
  const double2* twid = nullptr;  // FftPlan forward twiddles (nc - 1)
  double2* F = nullptr;           // spectrum cache [kSMax][m]
  double2* G = nullptr;           // adjoint partials [kSMax][L][nc]
  // Gaussian-measurement phase retrieval: the measurement
  // vectors as an m x 2n row-major real matrix [Re a_i | Im a_i]; L is then the
  // number of split-K parts of the adjoint (summed by pr_combine), nc = n
  const double* gA = nullptr;
};

// Solver configuration (mirrors cuhallar_config / SolverConfig).
struct Cfg {
  double eps, beta0, beta_growth, eps0, eps_decay, eps_floor;
  int max_outer;
  double time_limit;
  double eig_tol;
  int eig_max_iters, eig_block_restart;
  double aipp_lambda0, aipp_rho;
  int aipp_max_outer;
  double aipp_lambda_underflow;
  double fista_sigma, fista_chi, fista_mu, fista_L0;
  int fista_max_iters, max_fw_steps;
  int trace;
  int parity;  // reductions in the checker's order (parity.cuh)
};

struct TraceEv {
  int kind, outer_iter;
  double beta, eps_inner, gap, theta;
  int64_t rank;
  double al_value, fw_alpha, rel_pfeas, rel_gap, rel_dfeas;
};

// Operation selector for the persistent kernel.
enum Op : int {
  kOpSolve = 0,
  kOpMap = 1,          // out_vec = A(UU') (edge order, trace at m-1)
  kOpCPlusAdj = 2,     // out = CU + (A* q)U, q given (edge + lower order)
  kOpAdj = 3,          // out = (A* q)U
  kOpApplyC = 4,       // out = CU
  kOpAlValue = 5,      // scalars[0] = L_beta(UU'; p)
  kOpAlValGrad = 6,    // scalars[0] = value, out = gradient
  kOpAlGrad = 7,       // out = gradient
  kOpMinEigG = 8,      // Lanczos on G(U,p,beta)
  kOpAipp = 9,         // aipp on L_beta(.;p) from U
  kOpBench = 10,       // repeat one pass bench_iters times, scalars[0] = ns / pass
};

// Everything the persistent kernel touches; lives in device memory.
struct Params {
  int op = kOpSolve;
  DevPairs I;
  Cfg cfg;
  int pass_scratch = 0;  // doubles of per-pass shared scratch in this launch
  // team
  Fabric fab;
  unsigned long long* bar = nullptr;
  double* slots = nullptr;  // [2][G][kRedK]
  // factor pool, row-major n x s (stride s) inside capacity n x kSMax
  double* buf[kNBuf] = {};
  // Lanczos column slots (n each), plus w
  double* vslot = nullptr;
  int nslot = 0;
  double* lw = nullptr;
  const double* lz_rand = nullptr;  // n * (1 + n_refill) host-generated N(0,1)
  int n_refill = 0;
  // refills beyond n_refill: requested from the host service thread of the
  // launch (capi.cu RefillService) through host-mapped memory; null: none
  int* svc_req = nullptr;          // mapped: refill index wanted
  const int* svc_ready = nullptr;  // mapped: refill index staged in svc_buf
  const double* svc_buf = nullptr; // mapped: n normals of that refill
  int* svc_err = nullptr;          // device: service timeout flag
  // multipliers / gradient operator (edge + lower order)
  double* p_up = nullptr;
  double* p_lo = nullptr;
  double* q_up = nullptr;
  double* q_lo = nullptr;
  double* r_up = nullptr;
  double* r_lo = nullptr;
  double* pad = nullptr;     // n x 4: rank-3 factor rows padded to 32 B for 256-bit gathers (SELL)
  double* p_sell = nullptr;  // the same multipliers in SELL slot order (null: no SELL copy)
  double* q_sell = nullptr;
  double* r_sell = nullptr;
  double p_trace = 0.0;      // p[m-1] input (theta)
  // op inputs
  int s_in = 1;              // rank of buf[0] input
  double beta_in = 0.0;
  double q_trace_in = 0.0;   // kOpCPlusAdj / kOpAdj: q[m-1]
  double rho_in = 0.0;
  int bench_kind = 0;
  unsigned long long* prof = nullptr;  // [2 * kProfCats]: ns, count
  int bench_iters = 0;
  double* out_vec = nullptr; // kOpMap
  double* out_mat = nullptr; // row-major n x s
  // outputs
  double* scalars = nullptr; // device scalars out
  int* iscalars = nullptr;
  // trace ring (host mapped)
  TraceEv* trace = nullptr;
  int trace_cap = 0;
  int* trace_count = nullptr;
  // start vector (solve): buf[0] holds U0 (s_in columns)
};

// Solve outputs written by CTA 0 (device memory, copied back by the host).
struct SolveOut {
  int status;
  int outer_iters, fw_steps;
  int out_buf;     // index of the buffer holding the final U
  int rank;
  long long aipp_iters, fista_iters, eig_products;
  double pval, dval, dval_no_theta, rel_pfeas, rel_gap, rel_dfeas;
  double theta, p_trace;
  int msg;         // message id
};

}  // namespace hallar
