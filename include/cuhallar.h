/* cuhallar.h — C-ABI of the B200-native HALLaR solver (libcuhallar.so).
 *
 * Drop-in boundary for the reference lrsdp solve path
 * (/root/reference/proj).  Every entry point cites the reference interface it
 * replaces.  Plain pointers and sizes only: no C++ or torch types cross this
 * boundary, nothing throws across it, every function returns a status code:
 *   0 ok, 64 input error (lrsdp::InputError, types.hpp:14-17),
 *   3 numerical failure (lrsdp::NumericalError, types.hpp:20-23),
 *   66 I/O error (std::ios_base::failure), 70 CUDA/internal error.
 * cuhallar_last_error() returns a thread-local message for the last failure.
 *
 * Layout at the boundary: factors U are n x s COLUMN-MAJOR (the reference's
 * Eigen::MatrixXd, types.hpp:9) with leading dimension ld >= n; constraint
 * vectors (b, p, q, A(UU')) are length-m in the reference's constraint order.
 * "_dev" pointers are CUDA device pointers, "_host" pointers host memory.
 */
#ifndef CUHALLAR_H
#define CUHALLAR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cuhallar_instance cuhallar_instance;
typedef void* cuhallar_stream; /* cudaStream_t; NULL = legacy default stream */

enum {
  CUHALLAR_OK = 0,
  CUHALLAR_ERR_INPUT = 64,
  CUHALLAR_ERR_NUMERICAL = 3,
  CUHALLAR_ERR_IO = 66,
  CUHALLAR_ERR_CUDA = 70,
  /* a device capacity was exceeded (factor rank above 32, Lanczos slots, an
   * unanswered refill request): not a CUDA fault; the message names the cap */
  CUHALLAR_ERR_CAPACITY = 71
};

/* SdpInstance::field_kind (sdp_instance.hpp:11) */
enum { CUHALLAR_FIELD_REAL = 0, CUHALLAR_FIELD_COMPLEX_EMBEDDED = 1 };
/* instance families */
enum { CUHALLAR_THETA = 0, CUHALLAR_MATCOMP = 1, CUHALLAR_PHASERET = 2 };
/* SolveStatus (solver.hpp:31-36) */
enum {
  CUHALLAR_OPTIMAL = 0,
  CUHALLAR_ITERATION_LIMIT = 1,
  CUHALLAR_TIME_LIMIT = 2,
  CUHALLAR_NUMERICAL_FAILURE = 3
};

const char* cuhallar_last_error(void);
const char* cuhallar_version(void);

/* ------------------------------------------------------------ instances --- */
/* build_theta_instance(make_hypercube(d))  instances.cpp:63-112, graph.cpp:135-148 */
int cuhallar_theta_hypercube(int d, cuhallar_instance** out);
/* build_theta_instance(make_cycle(n)) / make_petersen()  graph.cpp:111-133 */
int cuhallar_theta_cycle(int n, cuhallar_instance** out);
int cuhallar_theta_petersen(cuhallar_instance** out);
/* build_theta_instance(Graph{n, edges}) from raw 0-based pairs; self-loops are
 * dropped and duplicates collapsed as load_graph does (graph.cpp:41-51). */
int cuhallar_theta_edges(int64_t n_vertices, int64_t n_pairs, const int64_t* u_host,
                         const int64_t* v_host, cuhallar_instance** out);
/* build_theta_instance(load_graph(path, fmt)); fmt 0 edge-list, 1 matrix-market,
 * 2 gset (graph.cpp:56-109) */
int cuhallar_theta_file(const char* path, int fmt, cuhallar_instance** out);
/* gen_matrix_completion(McSpec)  instances.cpp:117-234 */
int cuhallar_gen_matrix_completion(int64_t n1, int64_t n2, int r, uint64_t seed,
                                   int offset_sample_count, double tau_safety,
                                   cuhallar_instance** out);
/* Matrix completion with the paper's sampling rule (
 * no reference counterpart — the reference draws m = matcomp_constraint_count
 * distinct entries, instances.cpp:123-159): `draws` (i, j) draws with replacement
 * from the same Rng stream after the hidden factors, deduplicated and sorted.
 * The paper's tables use draws = 40 (n1 + n2). */
int cuhallar_gen_matrix_completion_paper(int64_t n1, int64_t n2, int r, uint64_t seed,
                                         int64_t draws, double tau_safety,
                                         cuhallar_instance** out);
/* A matrix-completion instance from a caller's sample list, host buffers:
 * Omega = {(i_k, j_k)} strictly increasing in (i, j) with 0 <= i < n1,
 * 0 <= j < n2 (the order gen_matrix_completion produces, instances.cpp:160-175),
 * b_k = M(i_k, j_k), and the trace bound tau (the reference derives it as
 * 2 * tau_safety * ||M||_*, instances.cpp:212).  The SdpInstance the reference's
 * McSpec path builds (instances.cpp:190-234) for data the caller already holds;
 * validation on the device (CUHALLAR_ERR_INPUT on unsorted / out-of-range pairs). */
int cuhallar_matcomp_from_samples(int64_t n1, int64_t n2, int64_t m, const int64_t* i,
                                  const int64_t* j, const double* b, double tau,
                                  cuhallar_instance** out);
/* matcomp_constraint_count  instances.cpp:123-129 */
int64_t cuhallar_matcomp_constraint_count(int64_t n1, int64_t n2, int r, int offset);
/* gen_phase_retrieval(PrSpec)  instances.cpp:239-389 */
int cuhallar_gen_phase_retrieval(int64_t n, int L, uint64_t seed, double tau_slack,
                                 cuhallar_instance** out);
/* Gaussian-measurement phase retrieval (BASELINE configs[2];
 * NOT in the reference): b_i = |a_i^* x|^2, i < m, a_i in C^n with i.i.d. CN(0,1)
 * entries generated on the device from `seed`, x drawn like gen_phase_retrieval's
 * hidden signal (instances.cpp:298-306), C = I, tau = tau_slack ||x||^2.  The map
 * and adjoint are FP64 tensor-core (DMMA) contractions over the stored m x 2n
 * measurement matrix.  Same operator / solve entry points as the other families. */
int cuhallar_gen_gauss_phase_retrieval(int64_t n, int64_t m, uint64_t seed, double tau_slack,
                                       cuhallar_instance** out);
/* the measurement vectors of a Gaussian phase-retrieval instance (m x n row-major) */
int cuhallar_instance_get_gauss(const cuhallar_instance* inst, double* A_re, double* A_im);
void cuhallar_instance_destroy(cuhallar_instance* inst);

typedef struct {
  int64_t n, m;
  int64_t identity_constraint; /* -1 = none (std::optional empty) */
  int field_kind, family;
  double tau, norm_b1, norm_C1;
  double nuclear_norm; /* matcomp only */
  int64_t device_bytes; /* HBM held by the instance */
  int64_t h2d_bytes;    /* host->device bytes copied so far (upload + solves) */
  int team_ctas;        /* persistent CTAs per launch on this device */
} cuhallar_instance_info;
/* SdpInstance public fields  sdp_instance.hpp:22-35 */
int cuhallar_instance_get_info(const cuhallar_instance* inst, cuhallar_instance_info* out);
/* SdpInstance::b (unscaled) */
int cuhallar_instance_get_b(const cuhallar_instance* inst, double* b_host);
/* theta: graph edges (i<j); matcomp: McInstance::omega_i / omega_j (j in [0,n2)) */
int cuhallar_instance_get_pairs(const cuhallar_instance* inst, int64_t* i_host, int64_t* j_host);
/* phaseret: PrInstance::hidden_x (nc complex) and masks (nc x L, column-major),
 * complex values as interleaved (re, im) doubles */
int cuhallar_instance_get_phaseret(const cuhallar_instance* inst, double* x_host,
                                   double* masks_host);

/* --------------------------------------------------- operator kernels ---- */
/* SdpInstance::apply_map  U -> A(UU')  (sdp_instance.hpp:39) */
int cuhallar_apply_map(cuhallar_instance* inst, const double* U_dev, int64_t ldu, int s,
                       double* out_dev, cuhallar_stream stream);
/* SdpInstance::apply_C  U -> CU  (sdp_instance.hpp:37) */
int cuhallar_apply_C(cuhallar_instance* inst, const double* U_dev, int64_t ldu, int s,
                     double* out_dev, int64_t ldo, cuhallar_stream stream);
/* SdpInstance::apply_adjoint  (p,U) -> (A*p)U  (sdp_instance.hpp:38) */
int cuhallar_apply_adjoint(cuhallar_instance* inst, const double* p_dev, const double* U_dev,
                           int64_t ldu, int s, double* out_dev, int64_t ldo,
                           cuhallar_stream stream);
/* SdpInstance::C_plus_adjoint  (q,U) -> CU + (A*q)U  (sdp_instance.hpp:43-46) */
int cuhallar_c_plus_adjoint(cuhallar_instance* inst, const double* q_dev, const double* U_dev,
                            int64_t ldu, int s, double* out_dev, int64_t ldo,
                            cuhallar_stream stream);
/* al_value (sdp_instance.hpp:67-68): value to *val_host */
int cuhallar_al_value(cuhallar_instance* inst, const double* U_dev, int64_t ldu, int s,
                      const double* p_dev, double beta, double* val_host,
                      cuhallar_stream stream);
/* al_gradient (sdp_instance.hpp:73-74) */
int cuhallar_al_gradient(cuhallar_instance* inst, const double* U_dev, int64_t ldu, int s,
                         const double* p_dev, double beta, double* grad_dev, int64_t ldg,
                         cuhallar_stream stream);
/* AlFunction::value_and_gradient (sdp_instance.hpp:115-127) */
int cuhallar_al_value_and_gradient(cuhallar_instance* inst, const double* U_dev, int64_t ldu,
                                   int s, const double* p_dev, double beta, double* val_host,
                                   double* grad_dev, int64_t ldg, cuhallar_stream stream);

/* ------------------------------------------------------------- solver ---- */
/* SolverConfig (solver.hpp:12-29) incl. EigSettings (lanczos.hpp:12-19),
 * AippParams (adap_aipp.hpp:8-16), FistaParams (adap_fista.hpp:24-32). */
typedef struct {
  double eps, beta0, beta_growth, eps0, eps_decay, eps_floor;
  int max_outer;
  double time_limit;
  uint64_t seed;
  double eig_tol;
  int eig_max_iters, eig_block_restart;
  double aipp_lambda0, aipp_rho;
  int aipp_max_outer;
  double aipp_lambda_underflow;
  double fista_sigma, fista_chi, fista_mu, fista_L0;
  int fista_max_iters, max_fw_steps;
  int threads;   /* record-only, as in the reference (README.md:108-111) */
  int trace;     /* deliver TraceEvents to the callback (costs one extra map per rank step) */
  int team_ctas; /* 0 = one persistent CTA per SM slot (auto) */
  int profile;   /* record per-phase device time (cuhallar_last_profile) */
  int parity;    /* 1 = parity mode: every reduction in the reference binary's order
                    (Eigen LinearVectorized redux, ordered CGS2 dots),
                    so counters match the CPU oracle; pair families, one GPU, slower */
} cuhallar_config;
/* Fills the reference defaults. */
void cuhallar_config_default(cuhallar_config* cfg);

/* TraceEvent (trace.hpp:12-28) */
typedef struct {
  int kind; /* 0 inner stationary, 1 inner rank step, 2 outer */
  int outer_iter;
  double beta, eps_inner, gap, theta;
  int64_t rank;
  double al_value, fw_alpha, rel_pfeas, rel_gap, rel_dfeas;
} cuhallar_trace_event;
typedef void (*cuhallar_trace_fn)(const cuhallar_trace_event* ev, void* user);

/* SolveReport (solver.hpp:40-61) */
typedef struct {
  int status;
  double pval, dval, dval_no_theta, rel_pfeas, rel_gap, rel_dfeas;
  int64_t rank;
  int outer_iters, fw_steps;
  int64_t aipp_iters, fista_iters, eig_products;
  double wall_seconds; /* host clock around the device solve, like solver.cpp:139 */
  double device_seconds; /* CUDA-event time of the persistent solve kernel */
  double tau, theta;
  int64_t trace_dropped;
  char message[256];
} cuhallar_report;

typedef struct cuhallar_solution cuhallar_solution;

/* solve(inst, cfg, sink) and the warm-start overload (solver.hpp:95-101).
 * U0_host (n x s0 column-major, scaled-ball factor) and p0_host (length m) may
 * be NULL for the cold start (u0 = gaussian_vector(n, Rng(seed))/|u0|).
 * The solution (U, p, theta) stays on the device in *sol until fetched. */
int cuhallar_solve(cuhallar_instance* inst, const cuhallar_config* cfg, const double* U0_host,
                   int s0, const double* p0_host, cuhallar_report* rep,
                   cuhallar_solution** sol, cuhallar_trace_fn fn, void* user);
/* Row-sharded solve over `world` ranks (no reference
 * counterpart — the reference is single-process, solver.hpp:95-101 is the
 * interface it extends).  insts[r] is the same instance built on rank r's
 * device (e.g. one per B200); each rank's persistent launch owns a contiguous
 * block of rows and the upper constraints of those rows, pushes the rows of
 * every gathered factor into its peers' replicas over peer memory
 * (NVLink/NVSwitch), and joins the per-rank partial sums of every reduction
 * in rank order.  Ranks may share a device (co-resident launches, used by the
 * single-GPU tests).  Pair families only (theta, matrix completion); the
 * report's device_seconds is the max over ranks. */
int cuhallar_solve_sharded(cuhallar_instance* const* insts, int world, const cuhallar_config* cfg,
                           const double* U0_host, int s0, const double* p0_host,
                           cuhallar_report* rep, cuhallar_solution** sol);

/* The same row-sharded solve with one process per GPU (torchrun): every rank
 * builds the instance on its own device, exports its rendezvous / partial-sum /
 * factor-arena allocations as CUDA IPC handles, the ranks exchange the handles
 * (any host-side collective) and call cuhallar_solve_rank concurrently.  Rows
 * and constraints are owned by rank as in cuhallar_solve_sharded; reductions
 * join per-rank partials in rank order, so every rank reports the same
 * scalars.  The solution's U is complete on every rank (replicated factor
 * arena); its p holds this rank's constraints (first index in its rows). */
typedef struct { unsigned char bytes[512]; } cuhallar_shard_handle;
int cuhallar_shard_export(cuhallar_instance* inst, int team_ctas, cuhallar_shard_handle* out);
int cuhallar_solve_rank(cuhallar_instance* inst, int world, int rank, const cuhallar_shard_handle* peers,
                        const cuhallar_config* cfg, const double* U0_or_null, int s0,
                        const double* p0_or_null, cuhallar_report* rep, cuhallar_solution** sol);
/* SolveReport::U (n x rank, column-major) and SolveReport::dual.p (length m) */
int cuhallar_solution_get_U(const cuhallar_solution* sol, double* U_host);
int cuhallar_solution_get_p(const cuhallar_solution* sol, double* p_host);
void cuhallar_solution_destroy(cuhallar_solution* sol);

/* ---------------------------------------- sub-solvers (parity testing) --- */
/* min_eigenpair of the HLR gradient operator G = C + A*(p + beta(A(UU')-b))
 * (hlr.cpp:12-29 over lanczos.cpp:32-141).  v_host may be NULL. */
int cuhallar_min_eig_gradient(cuhallar_instance* inst, const double* U_host, int s,
                              const double* p_host, double beta, double tol, int max_iters,
                              int block_restart, uint64_t seed, double* lambda,
                              double* v_host, double* residual, int* matvecs, int* converged);
/* As cuhallar_min_eig_gradient with EigSettings taken from cfg (eig_max_iters,
 * eig_block_restart, seed) and cfg->parity selecting the checker-order mode. */
int cuhallar_min_eig_gradient_cfg(cuhallar_instance* inst, const double* U_host, int s,
                                  const double* p_host, double beta, double tol,
                                  const cuhallar_config* cfg, double* lambda, double* v_host,
                                  double* residual, int* matvecs, int* converged);
/* aipp_run on g = L_beta(.;p) from W_host (adap_aipp.cpp:40-116) */
int cuhallar_aipp(cuhallar_instance* inst, const double* p_host, double beta,
                  const double* W_host, int s, double rho, const cuhallar_config* cfg,
                  double* W_out_host, int* status, int* prox_iters, int* fista_iters,
                  double* R_norm, double* g_value, double* lambda);

/* ------------------------------------------------------ measurement ------ */
/* In-kernel timing of one solver pass repeated `iters` times inside a single
 * persistent launch: kind 0 team barrier, 1 team all-reduce (5 values),
 * 2 fused value+gradient row pass (C + A*(p + beta(A(UU')-b)))U + reductions,
 * 3 constraint map pass A(UU') + reductions, 4 Lanczos matvec (fixed q, s=1).
 * U_host n x s column-major, p_host length m.  *ns_per_pass from %globaltimer. */
int cuhallar_bench_pass(cuhallar_instance* inst, int kind, const double* U_host, int s,
                        const double* p_host, double beta, int iters, int team_ctas,
                        double* ns_per_pass);

/* The trace ring of the last traced launch (events in order, also the debug
 * kinds 9 = fista() call and 10 = parity job-phase results); returns the count. */
int cuhallar_last_trace(const cuhallar_instance* inst, cuhallar_trace_event* out, int cap);

/* Per-phase device time of the last profiled solve (cfg.profile = 1):
 * categories 0 fista_x~, 1 fista_value_grad, 2 fista_y+_map, 3 fista_grad_y+,
 * 4 aipp, 5 lanczos_apply, 6 lanczos_cgs2, 7 jacobi, 8 lanczos_measure,
 * 9 lanczos_restart, 10 gradient_operator, 11 fw_gap, 12 fw_step, 13 outer, 14 other.
 * Returns the number of categories written (0 if none recorded). */
int cuhallar_last_profile(const cuhallar_instance* inst, double* ns, int64_t* counts, int cap);

#ifdef __cplusplus
}
#endif
#endif /* CUHALLAR_H */
