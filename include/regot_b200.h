/* regot_b200.h -- C ABI of the B200-native entropic-OT dual solver.
 *
 * The reference (`regot`, /root/reference/proj/include/regot/) is a header-only
 * C++ library with no FFI layer; its seam is a set of free functions over
 * value structs.  This header is the C-ABI replacement for that
 * seam: plain pointers and sizes, no C++ or torch types.  Each entry point
 * names the reference function it replaces (file:line, relative to
 * proj/include/regot/).  include/regot_b200.hpp re-creates the reference's
 * C++ signatures (regot::run_splr, ...) on top of it; INTEGRATION.md shows the
 * binding a maintainer of the reference would add.
 *
 * Conventions
 *  - All floating point is IEEE binary64.  Indices are int32 (like the
 *    reference's SparseSym, sparsity.h:100-101) or int64 for sizes.
 *  - Host pointers unless a name ends in _device.  The caller owns its inputs;
 *    the library owns device memory until regot_b200_destroy().
 *  - Every function returns a regot_status; on failure regot_b200_last_error()
 *    holds the message the reference would have thrown.
 *  - Dual points obey the gauge beta[m-1] == 0 (dual.h:72-78); a violation is
 *    REGOT_E_VALIDATION exactly as in the reference.
 *  - A context is bound to one CUDA device and is re-entrant per handle
 *    (different handles may be driven from different threads, bench.h:203-211).
 *  - There is no CPU fallback: every compute entry point runs sm_100a kernels.
 */
#ifndef REGOT_B200_H
#define REGOT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One code per reference exception class (core.h:21-37) + StepError
 * (splr.h:315-324) + device-side failure classes. */
typedef enum regot_status {
    REGOT_OK = 0,
    REGOT_E_DEGENERATE_COST = 1,
    REGOT_E_FORMAT = 2,
    REGOT_E_TRUNCATION = 3,
    REGOT_E_VALIDATION = 4,
    REGOT_E_IO = 5,
    REGOT_E_ORACLE_SIZE = 6,
    REGOT_E_STRUCTURE = 7,
    REGOT_E_NOT_POSITIVE_DEFINITE = 8,
    REGOT_E_DIRECTION = 9,
    REGOT_E_LINE_SEARCH = 10,
    REGOT_E_PLOT = 11,
    REGOT_E_STEP = 12,
    REGOT_E_CUDA = 100,
    REGOT_E_NCCL = 101,
    REGOT_E_NOMEM = 102,
    REGOT_E_UNSUPPORTED = 103
} regot_status;

/* Cost-matrix layouts accepted at upload. */
#define REGOT_LAYOUT_COLMAJOR 0 /* Eigen::MatrixXd, the reference's in-memory layout (core.h:16) */
#define REGOT_LAYOUT_ROWMAJOR 1 /* ROTB on-disk layout (problem.h:235-237) */

/* SplrConfig (splr.h:22-60), field for field.  `tile_rows/tile_cols` mirror
 * FusedTiling (dual.h:97-101): they take part in the config hash but are
 * advisory on the device (the GPU reduction tree is fixed).  The cg_* and
 * lse_fused fields are extensions with no reference counterpart. */
typedef struct regot_splr_config {
    double tau_max;
    int64_t S;
    int64_t J;
    double density;
    double c1;
    double c2;
    int64_t max_iter;
    double tol;
    int64_t max_ls_trials;
    int64_t record_every;
    int32_t overlap;   /* 1: Sinkhorn candidate chain on a side CUDA stream (splr.h:373-378) */
    int32_t tile_rows; /* default 8 */
    int32_t tile_cols; /* default 32 */
    /* --- extensions --- */
    int32_t cg_max_iter; /* PCG iteration cap per solve; <=0 -> 20 * dim */
    double cg_rtol;      /* PCG relative preconditioned-residual tolerance; <=0 -> 1e-10 */
} regot_splr_config;

/* SinkhornConfig (sinkhorn.h:16-31). */
typedef struct regot_sinkhorn_config {
    int64_t max_iter;
    int64_t record_every;
    double tol; /* 0 disables the convergence test */
} regot_sinkhorn_config;

/* TraceRow (trace.h:11-18). */
typedef struct regot_trace_row {
    int64_t iter;
    double wall_ms;
    double f;
    double marginal_error;
    double duality_gap;
} regot_trace_row;

/* SplrStepRecord (splr.h:294-312) + cg_iters (extension). */
typedef struct regot_step_record {
    int64_t iter;
    int32_t refresh;
    int32_t sinkhorn_selected;
    double f_before;
    double f_after;
    double f_cand_sinkhorn; /* NaN when no Sinkhorn candidate was produced */
    double f_cand_qn;
    double gamma;
    double g_dot_d;
    double gnew_dot_d;
    int32_t curvature_ok;
    int32_t ls_failed;
    int32_t lowrank_active;
    int32_t factor_retries;
    double tau;
    int32_t ls_evals;
    int32_t cg_iters;
} regot_step_record;

/* SplrResult / SinkhornResult (splr.h:480-485, sinkhorn.h:117-121).  Arrays are
 * malloc'd by the library and released by regot_b200_result_free().  When a
 * step fails, status == REGOT_E_STEP, `message` is the reference's StepError
 * text ("run_splr: step <iter> failed: <what>", splr.h:520-525) and `trace`
 * holds the rows collected so far; alpha/beta are NULL. */
typedef struct regot_result {
    int32_t status;
    int32_t reserved;
    int64_t n;
    int64_t m;
    double* alpha;
    double* beta;
    regot_trace_row* trace;
    int64_t n_trace;
    regot_step_record* steps; /* NULL for Sinkhorn */
    int64_t n_steps;
    double eta;
    char algo[16];        /* "splr" | "sinkhorn" (SolverTrace::algo) */
    char config_hash[24]; /* 16 hex digits, FNV-1a (splr.h:62-70, sinkhorn.h:33-39) */
    char message[256];
    /* measurement extras */
    double device_ms;        /* CUDA-event time of the whole solve on the main stream */
    int64_t gradient_passes; /* fused-gradient launches (K1) */
    int64_t lse_passes;      /* row/column LSE launches (K7/K8) */
    int64_t kernel_launches; /* all kernels of this library launched by the solve */
} regot_result;

/* GradientResult (dual.h:50-56) extras returned with every gradient pass. */
typedef struct regot_gradient_info {
    double f;
    double marginal_error; /* dual.h:219-222 */
    double duality_gap;    /* dual.h:225-229 */
    double grad_norm2;     /* ||grad||_2 over the n+m-1 free coordinates (splr.h:353) */
    double total_mass;     /* sum of T */
} regot_gradient_info;

typedef struct regot_ctx regot_ctx;
typedef struct regot_sparse regot_sparse; /* device H_Omega + tau I (sparsity.h:97-195) */

/* ---- context ---------------------------------------------------------------- */
regot_status regot_b200_create(int device, regot_ctx** out);
void regot_b200_destroy(regot_ctx* ctx);
const char* regot_b200_last_error(const regot_ctx* ctx); /* ctx may be NULL: last create() error */
const char* regot_b200_status_name(regot_status s);       /* reference exception class name */
/* Library identification: "regot_b200 <version> sm_100a". */
const char* regot_b200_version(void);

/* Row-sharded multi-GPU (north_star item 5).  One process per GPU; rank r owns a
 * contiguous block of rows.  `unique_ids` is 256 bytes -- two ncclUniqueIds (one
 * communicator per CUDA stream of the solver) made by
 * regot_b200_comm_unique_id() on rank 0 and broadcast by the host program. */
regot_status regot_b200_comm_unique_id(void* out256);
regot_status regot_b200_comm_init(regot_ctx* ctx, int rank, int world, const void* unique_ids256);

/* ---- problem upload: ProblemInstance (problem.h:20-28) ---------------------- */
/* Full problem on one GPU.  M is n x m with leading dimension ld (elements). */
regot_status regot_b200_set_problem(regot_ctx* ctx, int64_t n, int64_t m, const double* M, int layout,
                                    int64_t ld, const double* a, const double* b, double eta);
/* Row block [row_begin, row_begin+row_count) of a global n x m problem; M points
 * at the first element of the GLOBAL matrix when layout is column-major, or at
 * the first element of the block's first row when row-major.  a has n entries
 * (global), b has m. */
regot_status regot_b200_set_problem_rows(regot_ctx* ctx, int64_t n, int64_t m, int64_t row_begin,
                                         int64_t row_count, const double* M, int layout, int64_t ld,
                                         const double* a, const double* b, double eta);
/* Inputs already resident in HBM: row-major block with pitch ld (elements,
 * multiple of 2), device pointers, borrowed (not copied, not freed). */
regot_status regot_b200_set_problem_device(regot_ctx* ctx, int64_t n, int64_t m, int64_t row_begin,
                                           int64_t row_count, const double* M_device, int64_t ld,
                                           const double* a_device, const double* b_device, double eta);
/* Point-cloud problem: squared-Euclidean cost of X (n x d, row-major) and Y (m x d) divided by its
 * maximum -- what gen_synthetic1 builds (problem.h:124-132) and normalize_cost (problem.h:53-61)
 * scales -- formed ON THE DEVICE with the same arithmetic (coordinates accumulated in order, multiply
 * and add rounded separately, true division), so the cost equals the host generator's bit for bit.
 * on_the_fly == 0 materialises the row block in HBM (no 8 n m bytes over PCIe); on_the_fly != 0 never
 * stores it: every pass over the cost recomputes its tiles in shared memory (BASELINE config E).  Both
 * modes give bitwise identical results.  The row-block variant serves sharded contexts (X holds all
 * n rows; the maximum is taken over all ranks). */
regot_status regot_b200_set_pointcloud(regot_ctx* ctx, int64_t n, int64_t m, int32_t d, const double* X,
                                       const double* Y, const double* a, const double* b, double eta,
                                       int32_t on_the_fly);
regot_status regot_b200_set_pointcloud_rows(regot_ctx* ctx, int64_t n, int64_t m, int64_t row_begin,
                                            int64_t row_count, int32_t d, const double* X, const double* Y,
                                            const double* a, const double* b, double eta, int32_t on_the_fly);
/* The resident (or on-the-fly) cost block of this context, row-major row_count x m, to host memory. */
regot_status regot_b200_get_cost(regot_ctx* ctx, double* M_rowmajor);
/* validate_problem (problem.h:30-50) on the uploaded instance. */
regot_status regot_b200_validate_problem(regot_ctx* ctx);
/* eta override, like `regot solve --eta` (tools/regot.cpp:121-122). */
regot_status regot_b200_set_eta(regot_ctx* ctx, double eta);

/* ---- dual kernels (dual.h) -------------------------------------------------- */
/* fused_gradient (dual.h:106-164): one pass over M.  alpha has n entries
 * (global), beta m.  Any output pointer may be NULL. grad has n+m-1 entries. */
regot_status regot_b200_fused_gradient(regot_ctx* ctx, const double* alpha, const double* beta,
                                       regot_gradient_info* info, double* grad, double* row_sums,
                                       double* col_sums);
/* plan (dual.h:83-94): dense T for tests / diagnostics, written in `layout`. */
regot_status regot_b200_plan(regot_ctx* ctx, const double* alpha, const double* beta, double* T, int layout);

/* ---- Sinkhorn (sinkhorn.h) -------------------------------------------------- */
/* optimal_alpha (sinkhorn.h:44-74) / optimal_beta (:77-101) / sinkhorn_step (:105-115) */
regot_status regot_b200_optimal_alpha(regot_ctx* ctx, const double* alpha, const double* beta, double* alpha_out);
regot_status regot_b200_optimal_beta(regot_ctx* ctx, const double* alpha, double* beta_out);
regot_status regot_b200_sinkhorn_step(regot_ctx* ctx, double* alpha_io, double* beta_io);
/* run_sinkhorn (sinkhorn.h:123-171) */
regot_status regot_b200_run_sinkhorn(regot_ctx* ctx, const double* alpha0, const double* beta0,
                                     const regot_sinkhorn_config* cfg, regot_result* out);

/* ---- sparsification (sparsity.h) -------------------------------------------- */
/* select_topk (sparsity.h:44-91) given a dense plan T (n x m, `layout`): the
 * parity entry point ("pattern bit-exact given identical T").  Writes up to
 * `cap` (i, j) pairs, sorted lexicographically, into coords[2*t], coords[2*t+1];
 * *count receives the pattern size (call with cap = 0 to query). */
regot_status regot_b200_select_topk_dense(regot_ctx* ctx, int64_t n, int64_t m, const double* T, int layout,
                                          int64_t k, int32_t* coords, int64_t cap, int64_t* count);
/* topk_budget (splr.h:336-340) */
int64_t regot_b200_topk_budget(int64_t n, int64_t m, double density);
/* plan + select_topk + assemble (splr.h:361-363) at the current problem: T is
 * formed on the fly, never materialised.  row_sums/col_sums are the gradient
 * sums at (alpha, beta) (GradientResult), tau >= 0. */
regot_status regot_b200_assemble_topk(regot_ctx* ctx, const double* alpha, const double* beta, int64_t k,
                                      double tau, const double* row_sums, const double* col_sums,
                                      regot_sparse** out);
/* assemble (sparsity.h:226-294) at a caller-given pattern (sorted unique pairs
 * containing the first row and column of the block). */
regot_status regot_b200_assemble(regot_ctx* ctx, const double* alpha, const double* beta, const int32_t* coords,
                                 int64_t ncoords, double tau, const double* row_sums, const double* col_sums,
                                 regot_sparse** out);
/* update_values (sparsity.h:305-317) */
regot_status regot_b200_update_values(regot_ctx* ctx, regot_sparse* A, const double* alpha, const double* beta,
                                      double tau, const double* row_sums, const double* col_sums);
/* SparseSym::matvec (sparsity.h:112-125): y = A v, dim = n+m-1 */
regot_status regot_b200_matvec(regot_ctx* ctx, const regot_sparse* A, const double* v, double* y);
/* Pattern and CSC export in the reference layout (sparsity.h:249-289):
 * alpha-column i = [diag, n+j ascending], beta-column n+j = [i ascending, diag]. */
/* dim = n+m-1; nnz / ncoords count this context's rows; pattern_id is 0 on a row-sharded context (the id
 * hashes the global structure). */
regot_status regot_b200_sparse_info(const regot_sparse* A, int32_t* dim, int64_t* nnz, int64_t* ncoords,
                                    uint64_t* pattern_id);
regot_status regot_b200_sparse_export(regot_ctx* ctx, const regot_sparse* A, int32_t* colptr, int32_t* rowidx,
                                      double* values, int32_t* coords);
/* This context's rows of the pattern (global row index, column) with the off-diagonal values B_ij =
 * T_ij / eta, in row-major order -- the one export that also works on a row-sharded context (the
 * concatenation over the ranks is the global pattern).  *count receives the number of local entries;
 * up to `cap` of them are written (coords: 2 ints per entry; either array may be NULL). */
regot_status regot_b200_sparse_export_local(regot_ctx* ctx, const regot_sparse* A, int32_t* coords, double* values,
                                            int64_t cap, int64_t* count);
void regot_b200_sparse_free(regot_sparse* A);

/* ---- SPLR (splr.h) ---------------------------------------------------------- */
/* compute_direction (splr.h:128-167) with the sparse Cholesky solve replaced by
 * device Jacobi-PCG (north_star item 3).  Low-rank term: pass u = v = NULL for
 * an inactive R.  cg_iters (optional) receives the PCG iterations used. */
regot_status regot_b200_compute_direction(regot_ctx* ctx, const regot_sparse* A, const double* g,
                                          const double* u, const double* v, double xi, double zeta,
                                          double cg_rtol, int32_t cg_max_iter, double* d, int32_t* cg_iters);
/* run_splr (splr.h:487-534) */
regot_status regot_b200_run_splr(regot_ctx* ctx, const double* alpha0, const double* beta0,
                                 const regot_splr_config* cfg, regot_result* out);

/* Step-level interface: SplrState (splr.h:82-97) as an opaque device-resident handle -- the iterate, its
 * gradient, the previous accepted iterate, the frozen pattern and its matrix -- with splr_init
 * (splr.h:326-334) and splr_step (splr.h:348-478).  run_splr is exactly init + the loop of splr.h:509-531
 * over step; a caller driving the steps itself gets bitwise the same iterates (the reference's tests do:
 * test_splr.cpp:349-378).  A state belongs to the context and problem it was made with; it is the
 * checkpoint / resume seam (state_point + state_info give everything a restart needs: x and iter --
 * restarting at a multiple of S rebuilds the pattern like the reference would). */
typedef struct regot_splr_state regot_splr_state;
regot_status regot_b200_splr_init(regot_ctx* ctx, const double* alpha0, const double* beta0,
                                  const regot_splr_config* cfg, regot_splr_state** out);
/* One iteration; rec (nullable) receives the step record.  Failures are the reference's exception classes
 * (REGOT_E_DIRECTION, REGOT_E_NOT_POSITIVE_DEFINITE, ...), not REGOT_E_STEP: wrapping is run_splr's job. */
regot_status regot_b200_splr_step(regot_ctx* ctx, regot_splr_state* state, const regot_splr_config* cfg,
                                  regot_step_record* rec);
/* st.iter, st.has_prev and the scalars of st.cur (f, marginal error, duality gap, ||grad||, mass). */
regot_status regot_b200_splr_state_info(regot_ctx* ctx, const regot_splr_state* state, int64_t* iter,
                                        int32_t* has_prev, regot_gradient_info* cur);
/* st.x (alpha: n, beta: m) and, optionally, st.cur's gradient (n+m-1), row sums (n), column sums (m). */
regot_status regot_b200_splr_state_point(regot_ctx* ctx, const regot_splr_state* state, double* alpha,
                                         double* beta, double* grad, double* row_sums, double* col_sums);
/* st.A: borrowed handle to H_Omega + tau I at the frozen pattern (valid until the next refresh step or
 * state_free; NULL before the first step).  Do not free it. */
const regot_sparse* regot_b200_splr_state_matrix(const regot_splr_state* state);
void regot_b200_splr_state_free(regot_splr_state* state);

void regot_b200_splr_config_default(regot_splr_config* cfg);         /* SplrConfig{} */
void regot_b200_sinkhorn_config_default(regot_sinkhorn_config* cfg); /* SinkhornConfig{} */
regot_status regot_b200_splr_config_validate(const regot_splr_config* cfg);         /* splr.h:37-59 */
regot_status regot_b200_sinkhorn_config_validate(const regot_sinkhorn_config* cfg); /* sinkhorn.h:22-30 */
void regot_b200_splr_config_hash(const regot_splr_config* cfg, char out17[17]);         /* splr.h:62-70 */
void regot_b200_sinkhorn_config_hash(const regot_sinkhorn_config* cfg, char out17[17]); /* sinkhorn.h:33-39 */
void regot_b200_result_free(regot_result* r);

/* ---- host-side logic of the row-sharded path (pure functions, no device needed) ---- */
/* Row block of rank `rank` of `world`: [n*rank/world, n*(rank+1)/world). */
void regot_b200_host_row_block(int64_t n, int rank, int world, int64_t* row_begin, int64_t* row_count);
/* Threshold search of the distributed top-k: given the (allreduced) histogram of an
 * order-preserving key digit, the largest bucket b with count(buckets >= b) >= need, and the count
 * strictly above it.  bucket = -1 when the histogram holds fewer than `need` entries. */
void regot_b200_host_pick_bucket(const uint64_t* hist, int nbins, int64_t need, int* bucket, int64_t* above);

/* ---- measurement hooks (bench.py; not part of the reference surface) --------- */
/* Runs `iters` back-to-back launches of one hot kernel on the context's stream
 * at the given dual point and returns the CUDA-event time of each launch (ms).
 * which: 0 fused gradient (K1), 1 row LSE (K7), 2 column LSE (K8). */
regot_status regot_b200_time_kernel(regot_ctx* ctx, int which, const double* alpha, const double* beta,
                                    int iters, float* ms_out);
/* Per-kernel device timing inside solves: when enabled every sweep / SpMV launch
 * is bracketed by CUDA events on its stream.  kind: 0 fused gradient (K1),
 * 1 row LSE (K7), 2 column LSE (K8), 3 top-k sweeps (K2), 4 SpMV (K4), 5 persistent PCG solve (K5),
 * 6 a whole pattern refresh, 7 a whole fused_gradient (K1 sweep + finalize kernels + allreduce).
 * set_profiling() also clears the recorded events. */
regot_status regot_b200_set_profiling(regot_ctx* ctx, int enabled);
regot_status regot_b200_get_profile(regot_ctx* ctx, int kind, int64_t* launches, double* total_ms);
/* Pattern reuse across refreshes -- north_star item (2): "the symbolic structure is reused across iterations and rebuilt
 * only when the pattern drifts".  The reference rebuilds the top-k pattern at every k % S == 0 (splr.h:352, 359-364); with
 * drift_tol > 0 such an iteration keeps pattern, pointer arrays and the direction solve's plans when (i) the duals moved
 * by at most drift_tol x eta in oscillation since the pattern was selected (osc(d_alpha) + osc(d_beta): every T_ij then
 * moved by a factor within exp(+-drift_tol) relative to every other), (ii) the values of the pattern refreshed at the
 * current point (update_values, sparsity.h:305-317) still capture >= (1 - drift_tol) x the share of the Hessian block's
 * mass (sum of the row sums over eta) they captured when the pattern was built, and (iii) fewer than max_skips refreshes
 * in a row kept it; the Sinkhorn candidate chain (splr.h:366-378) runs either way.
 * drift_tol = 0 (default) is the reference's rule, bit for bit.  pattern_counts: rebuilds and reuses since creation. */
regot_status regot_b200_set_pattern_reuse(regot_ctx* ctx, double drift_tol, int max_skips);
void regot_b200_pattern_counts(const regot_ctx* ctx, int64_t* rebuilds, int64_t* reuses);
/* Kernels of this library launched on this context since creation. */
int64_t regot_b200_launch_count(const regot_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* REGOT_B200_H */
