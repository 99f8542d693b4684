// ctx.hpp -- host-side context of the device solver: device buffers, streams,
// error plumbing.  Internal to the library (the public surface is
// include/regot_b200.h).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <ctime>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/regot_b200.h"

struct ncclComm;

namespace rg {

// Error carrying a regot_status; thrown inside the library, converted to a
// status code + message at the C boundary.
struct Error : std::runtime_error {
    regot_status code;
    Error(regot_status c, const std::string& w) : std::runtime_error(w), code(c) {}
};
[[noreturn]] inline void raise(regot_status c, const std::string& w) { throw Error(c, w); }

#define RG_CUDA(expr)                                                                                         \
    do {                                                                                                      \
        cudaError_t e__ = (expr);                                                                             \
        if (e__ != cudaSuccess)                                                                               \
            ::rg::raise(REGOT_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e__) + " (" + __FILE__ + \
                                          ":" + std::to_string(__LINE__) + ")");                              \
    } while (0)

// RAII device buffer of T (grow-only)
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release()
    {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void swap(DevBuf& o)
    {
        std::swap(p, o.p);
        std::swap(n, o.n);
    }
    void ensure(size_t count)
    {
        if (count <= n && p) return;
        // a buffer that grows again gets a quarter of headroom: candidate and pattern sizes creep up from refresh to refresh,
        // and every regrowth is a cudaFree + cudaMalloc (synchronising; tens of ms at the GB sizes of config D)
        const bool regrow = p != nullptr;
        release();
        cudaError_t e = cudaErrorMemoryAllocation;
        if (regrow && count > 1024) {
            const size_t padded = count + count / 4;
            e = cudaMalloc((void**)&p, sizeof(T) * padded);
            if (e == cudaSuccess) {
                n = padded;
                return;
            }
            p = nullptr;
            cudaGetLastError();
        }
        e = cudaMalloc((void**)&p, sizeof(T) * (count ? count : 1));
        if (e != cudaSuccess) {
            p = nullptr;
            cudaGetLastError();
            raise(REGOT_E_NOMEM, std::string("cudaMalloc of ") + std::to_string(sizeof(T) * count) +
                                     " bytes failed: " + cudaGetErrorString(e));
        }
        n = count;
    }
};

// RAII pinned host buffer of T (grow-only): staging for asynchronous copies
template <class T>
struct PinnedBuf {
    T* p = nullptr;
    size_t n = 0;
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    ~PinnedBuf()
    {
        if (p) cudaFreeHost(p);
    }
    void ensure(size_t count)
    {
        if (count <= n && p) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        const size_t want = count + count / 4 + 64;  // slack: sizes drift from refresh to refresh
        RG_CUDA(cudaMallocHost((void**)&p, sizeof(T) * want));
        n = want;
    }
};

// A slot of mapped pinned host memory: the last thread of a kernel writes its scalars there, then a
// sequence number (device side: mailbox_post in common.cuh); the host spins on the sequence number
// instead of paying a copy + stream synchronisation for every decision it takes (a line-search
// evaluation, a set of dot products, the end of a PCG solve: ~6 per quasi-Newton iteration).
struct HostMailbox {
    static constexpr int kSlots = 31;  // payload doubles; the sequence number follows them
    double* data = nullptr;
    unsigned long long expected = 0;
    HostMailbox() = default;
    HostMailbox(const HostMailbox&) = delete;
    HostMailbox& operator=(const HostMailbox&) = delete;
    ~HostMailbox()
    {
        if (data) cudaFreeHost(data);
    }
    void ensure()
    {
        if (data) return;
        RG_CUDA(cudaHostAlloc((void**)&data, sizeof(double) * (kSlots + 1), cudaHostAllocMapped));
        for (int k = 0; k <= kSlots; ++k) data[k] = 0.0;
        reinterpret_cast<volatile unsigned long long*>(data)[kSlots] = 0ULL;
    }
    // the value the next post must carry
    unsigned long long next() { return ++expected; }
    // block until the post with sequence number `expected` has landed (all earlier work of the posting
    // stream is then complete); a failed launch or kernel shows up through cudaStreamQuery
    static double wall_seconds()
    {
        timespec ts;
        clock_gettime(CLOCK_MONOTONIC, &ts);
        return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
    }
    static double timeout_seconds()
    {
        static const double t = std::getenv("REGOT_B200_MAILBOX_TIMEOUT_S") ? std::atof(std::getenv("REGOT_B200_MAILBOX_TIMEOUT_S")) : 300.0;
        return t;
    }
    void wait(cudaStream_t st) const
    {
        const double t_start = wall_seconds();
        const volatile unsigned long long* seq = reinterpret_cast<const volatile unsigned long long*>(data) + kSlots;
        for (unsigned long spins = 0; *seq != expected; ++spins) {
            if ((spins & 0xffffUL) == 0xffffUL) {
                const cudaError_t e = cudaStreamQuery(st);
                if (e != cudaErrorNotReady && *seq != expected) {
                    if (e == cudaSuccess) raise(REGOT_E_CUDA, "mailbox: stream drained without the expected post (internal error)");
                    raise(REGOT_E_CUDA, std::string("mailbox: ") + cudaGetErrorString(e));
                }
                // a kernel that never posts (a persistent kernel waiting on itself) must not hang the caller for ever
                if ((spins & 0xffffffUL) == 0xffffffUL && wall_seconds() - t_start > timeout_seconds())
                    raise(REGOT_E_CUDA, "mailbox: no post within the time limit (REGOT_B200_MAILBOX_TIMEOUT_S); the device is still busy");
            }
        }
        __sync_synchronize();
    }
};

// Geometry of the panel sweep shared by the fused-gradient and LSE kernels:
// M is cut into tiles of tile_rows x tile_cols, ordered column-panel-major
// (tile id = panel * n_row_tiles + row_tile); CTA b owns the contiguous tile
// range [total*b/grid, total*(b+1)/grid).  A "segment" is the part of one
// CTA's range inside one panel; column partials are produced per segment and
// reduced per panel in segment order (deterministic, no atomics).
struct SweepPlan {
    int tile_rows = 0, tile_cols = 0;
    int n_row_tiles = 0, n_panels = 0;
    long total_tiles = 0;
    int grid = 0;
    int n_segments = 0;
    DevBuf<int> d_cta_seg0;      // grid + 1: first segment id of each CTA
    DevBuf<int> d_panel_seg0;    // n_panels + 1: first segment id of each panel
};

// Scalars produced by every gradient pass.
struct GradScalars {
    double f, marginal_error, duality_gap, grad_sqnorm, total_mass, g_dot_d;
    double row_abs, col_abs;  // the two halves of the marginal error
    double lse_flag;          // != 0: a fast Sinkhorn update on this stream left its safe range since the last check
    double f_lo;              // f = f + f_lo to about twice the working precision (one GPU; 0 where the plain sum is used)
};

// Per-stream scratch of one sweep (gradient or LSE) so the main stream and the
// Sinkhorn side stream can run concurrently.
struct SweepWS {
    DevBuf<double> rowpart;   // n_panels x nloc            (gradient row partials / LSE row sums)
    DevBuf<double> rowpart2;  // n_panels x nloc            (LSE row maxima)
    DevBuf<double> colpart;   // n_segments x tile_cols     (column partial sums)
    DevBuf<double> colpart2;  // n_segments x tile_cols     (LSE column maxima)
    DevBuf<double> pack;      // m + 16: column sums + row-side scalars (the allreduce payload)
    DevBuf<double> pack2;     // LSE: second payload
    DevBuf<double> partials;  // per-CTA scalar partials of the finalize kernels
    DevBuf<unsigned int> ticket;
    DevBuf<GradScalars> d_scal;
    DevBuf<unsigned int> sk_flag;  // set by the fast Sinkhorn updates (k7_lse.cu), reported with the next gradient pass
    HostMailbox mbox;  // the pass's scalars, posted by k_gradient_fin2
};

// Problem resident on the device (one row block).
struct DeviceProblem {
    int64_t n = 0, m = 0;             // global sizes
    int64_t row_begin = 0, nloc = 0;  // this rank's row block
    int64_t ld = 0;                   // row pitch of M in elements
    double eta = 0.0;
    const double* M = nullptr;  // row-major nloc x ld
    const double* a = nullptr;  // nloc entries (this block)
    const double* b = nullptr;  // m entries
    DevBuf<double> M_own, a_own, b_own;
    CUtensorMap tmap;  // 2-D map over M for the sweep kernels
    bool loaded = false;
    // point-cloud problems (regot_b200_set_pointcloud): cost = |x_i - y_j|^2 / max.  on_the_fly: M is
    // never materialised (M == nullptr); the sweeps form their tiles from X and Y.
    bool on_the_fly = false;
    int cloud_d = 0;
    double cloud_max = 0.0;
    bool cloud_fast_div = false;  // the reciprocal-based division was verified against true division on this block
    DevBuf<double> X_own, Y_own;  // nloc x d, m x d
};

// A dual-space vector on the device: alpha block (nloc, row-sharded) + beta
// block (m, replicated).  Free vectors use beta[0..m-2]; beta[m-1] is kept 0.
struct DVec {
    DevBuf<double> a, b;
    void ensure(int64_t nloc, int64_t m)
    {
        a.ensure((size_t)nloc);
        b.ensure((size_t)m);
    }
    void swap(DVec& o)
    {
        a.swap(o.a);
        b.swap(o.b);
    }
};

// Outputs of a gradient pass on the device.
struct GradOut {
    DVec g;          // grad: g.a = row_sums - a, g.b[j] = col_sums[j] - b[j] (all m; free part is j < m-1)
    DVec sums;       // sums.a = row_sums, sums.b = col_sums
    GradScalars sc;  // host copy, valid after the stream is synchronised
    void ensure(int64_t nloc, int64_t m)
    {
        g.ensure(nloc, m);
        sums.ensure(nloc, m);
    }
    void swap(GradOut& o)
    {
        g.swap(o.g);
        sums.swap(o.sums);
        std::swap(sc, o.sc);
    }
};

}  // namespace rg

struct regot_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;  // main stream
    cudaStream_t side = nullptr;    // Sinkhorn candidate chain (splr.h:373-378)
    cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_fork = nullptr, ev_join = nullptr;
    std::string err;
    int64_t launches = 0;

    // multi-GPU
    int rank = 0, world = 1;
    bool sharded = false;  // world > 1, or a one-rank communicator driven through the sharded path (REGOT_B200_SHARDED_SINGLE: tests)
    ncclComm* comm = nullptr;       // main-stream collectives
    ncclComm* comm_side = nullptr;  // side-stream collectives (own communicator: no cross-stream ordering hazards)

    rg::DeviceProblem prob;
    rg::SweepPlan plan;
    rg::SweepWS ws_main, ws_side;
    rg::DevBuf<double> exp_table;  // kExpN doubles: 2^(j/N), high word biased (common.cuh)

    // staging for API calls that take host vectors
    rg::DVec api_x, api_y, api_d;
    rg::GradOut api_grad;

    void* solver_ws = nullptr;  // opaque solver workspace (solver.cu)

    // tests: run the sharded (multi-kernel + NCCL) PCG path on one GPU (REGOT_B200_MULTIKERNEL_PCG=1)
    bool force_multikernel_pcg = false;
    // panel mat-vec of the kernel-by-kernel PCG (k4_sparse.cu): -1 auto (large patterns), 0 off, 1 always
    // (REGOT_B200_PANEL_SPMV); panel_width > 0 caps the panel width in entries (REGOT_B200_PANEL_WIDTH, tests)
    int panel_spmv = -1;
    int panel_width = 0;
    int panel_ahead = 0;  // REGOT_B200_PANEL_AHEAD: prefetch distance of the ELL stream in rows of 32 entries (0: off)
    int panel_ell = 1;  // REGOT_B200_PANEL_ELL=0: pieces straight from the CSR / CSC copy (the form before the ELL stream)
    // one GPU: the two finalize kernels of a gradient pass as one (REGOT_B200_FUSED_FINALIZE=0: two kernels, as sharded runs)
    bool fused_finalize = true;
    // the objective's three sums accumulated in double-double and the line search comparing objectives as (hi, lo) pairs, so
    // that decreases below one ulp of f still register near the tolerance (REGOT_B200_EXTENDED_F=0: plain doubles, like the
    // reference); one GPU with the fused finalize kernel only
    bool extended_f = true;
    // block-resident PCG (k6_pcg_blocks.cu): -1 auto (whenever the pattern fits), 0 off (REGOT_B200_PCG_BLOCKS);
    // pcg_blocks_p x pcg_blocks_q > 0 force the block grid (REGOT_B200_PCG_BLOCKS_GRID=PxQ, tests)
    // top-k refresh: the count sweep starts from the previous refresh's threshold bin and histograms the candidates itself;
    // the histogram sweep runs only when that guess turns out too high (REGOT_B200_TOPK_GUESS=0: always three sweeps)
    int topk_guess = 1;
    int topk_prev_bin = -1;
    long long topk_prev_take = -1;
    // pattern reuse across refreshes (north_star item 2, an extension of the reference's fixed-S rule splr.h:352-364): at
    // an iteration with k % S == 0 the top-k pattern is rebuilt only if the share of the Hessian block's mass it holds fell
    // below (1 - pattern_drift) x the share it held when it was built, or after pattern_max_skips refreshes in a row kept it;
    // otherwise the refresh is a value update and the candidate chain.  0 (default): the reference's rule, always rebuild
    // (regot_b200_set_pattern_reuse, REGOT_B200_PATTERN_DRIFT / REGOT_B200_PATTERN_MAX_SKIPS)
    double pattern_drift = 0.0;
    int pattern_max_skips = 4;
    int64_t pattern_rebuilds = 0, pattern_reuses = 0;
    int schur_diag = 1;  // REGOT_B200_SCHUR_DIAG=0: precondition with D2 instead of diag(D2 - B' D1^-1 B)
    int pcg_blocks = -1;
    int pcg_blocks_p = 0, pcg_blocks_q = 0;
    // block rows as thread-block clusters: -1 auto, 0 off (REGOT_B200_PCG_BLOCKS_CLUSTER); patterns up to this many entries
    // take a single cluster (REGOT_B200_PCG_BLOCKS_ONE_CLUSTER_ENTRIES); pcg_blocks_maxcl[q]: clusters of q CTAs the device holds
    int pcg_blocks_cluster = -1;
    long pcg_blocks_one_cluster_entries = 100000;
    long pcg_blocks_cluster_entries = 600000;  // block rows as clusters only up to this many entries (REGOT_B200_PCG_BLOCKS_CLUSTER_ENTRIES)
    bool pcg_blocks_probed = false;
    int pcg_blocks_maxcl[17] = {0};
    // persistent PCG on one thread-block cluster when a CG iteration touches at most this many matrix entries
    // (REGOT_B200_PCG_CLUSTER = 0 | 8 | 16, REGOT_B200_PCG_CLUSTER_ENTRIES)
    int pcg_cluster_size = 0;
    bool pcg_cluster_probed = false;
    long pcg_cluster_max_entries = 0;
    // Sinkhorn updates take the gradient-sweep form (k7_lse.cu: alpha_i += eta (log a_i - log r_i) from K1-speed sweeps,
    // with an exact redo through the log-sum-exp kernels whenever a sum leaves [e^-600, e^600]) in run_sinkhorn
    // (REGOT_B200_EXACT_LSE=1: always the log-sum-exp kernels) and in the candidate chain of run_splr
    // (REGOT_B200_FAST_CHAIN=0: log-sum-exp kernels there); the stand-alone entry points always use the log-sum-exp kernels
    bool fast_sinkhorn = true;
    bool fast_sinkhorn_chain = true;
    // row log-sum-exp kernel: shift by the warp's approximate maximum (one redux instead of five shuffle rounds; same
    // value up to rounding) -- REGOT_B200_LSE_FAST_SHIFT=0: the exact maximum, the reference's arithmetic
    bool lse_fast_shift = true;

    // optional per-kernel timing (regot_b200_set_profiling): event pairs around the sweep kernels
    bool profiling = false;
    struct ProfEvent {
        int kind;
        cudaEvent_t a, b;
    };
    std::vector<ProfEvent> prof_events;
};

namespace rg {

void ctx_require_problem(const regot_ctx* ctx);
// kind: 0 gradient sweep (K1), 1 row LSE (K7), 2 column LSE (K8), 3 top-k sweeps (K2), 4 spmv (K4),
// 5 persistent PCG solve (K5), 6 a whole pattern refresh (top-k sweeps + selection + structure, host gaps included),
// 7 a whole fused_gradient (K1 sweep + finalize kernels + allreduce)
struct ProfScope {
    regot_ctx* ctx;
    cudaStream_t st;
    int idx = -1;
    ProfScope(regot_ctx* c, cudaStream_t s, int kind) : ctx(c), st(s)
    {
        if (!ctx->profiling) return;
        regot_ctx::ProfEvent e;
        e.kind = kind;
        cudaEventCreate(&e.a);
        cudaEventCreate(&e.b);
        cudaEventRecord(e.a, st);
        ctx->prof_events.push_back(e);
        idx = (int)ctx->prof_events.size() - 1;
    }
    ~ProfScope()
    {
        if (idx >= 0) cudaEventRecord(ctx->prof_events[(size_t)idx].b, st);
    }
};
void make_sweep_plan(regot_ctx* ctx);
void ensure_sweep_ws(regot_ctx* ctx, SweepWS& ws);

// ---- kernel launchers (k1_gradient.cu) ----------------------------------------
// Enqueue one fused-gradient pass at (alpha, beta) on `st`.  dir_a/dir_b
// (nullable) give a direction d for phi'(gamma) = grad . d.  Column sums and
// the row-side scalars are allreduced over `comm` when world > 1.  On return
// everything is enqueued; out.sc is valid after sync_scalars().
void launch_gradient(regot_ctx* ctx, cudaStream_t st, SweepWS& ws, ncclComm* comm, const double* alpha,
                     const double* beta, const double* dir_a, const double* dir_b, GradOut& out);
// Wait for the pass enqueued on `st` and copy its scalars into out.sc.
void sync_scalars(regot_ctx* ctx, cudaStream_t st, SweepWS& ws, GradOut& out);
// Only the main sweep kernel, for timing (regot_b200_time_kernel).
void launch_gradient_sweep_only(regot_ctx* ctx, cudaStream_t st, SweepWS& ws, const double* alpha, const double* beta);
// Dense plan T (row-major nloc x m) for tests/diagnostics.
void launch_plan(regot_ctx* ctx, cudaStream_t st, const double* alpha, const double* beta, double* T_rowmajor);

// ---- Sinkhorn launchers (k7_lse.cu) ----------------------------------------------
void launch_row_lse_sweep_only(regot_ctx* ctx, cudaStream_t st, SweepWS& ws, const double* beta);
void launch_col_lse_sweep_only(regot_ctx* ctx, cudaStream_t st, SweepWS& ws, const double* alpha);
void launch_optimal_alpha(regot_ctx* ctx, cudaStream_t st, SweepWS& ws, const double* beta, double* alpha_out);
void launch_optimal_beta(regot_ctx* ctx, cudaStream_t st, SweepWS& ws, ncclComm* comm, double* alpha_io,
                         double* beta_out, int gauge);
void launch_sinkhorn_step(regot_ctx* ctx, cudaStream_t st, SweepWS& ws, ncclComm* comm, double* alpha_io,
                          double* beta_io);
// The same update from two fused-gradient sweeps (row sums at (alpha, beta), column sums at (alpha', beta)):
//   alpha_i += eta (log a_i - log r_i),  beta_j += eta (log b_j - log c_j),  then the gauge shift.
// Identical to the log-sum-exp form whenever every sum lies in [e^-600, e^600] (no entry that matters was
// clamped); otherwise ws.sk_flag is set and the caller must redo the update with launch_sinkhorn_step.
// row_sums_here (nullable): row sums of T at (alpha, beta) from a gradient pass made at this very point.
void launch_sinkhorn_step_fast(regot_ctx* ctx, cudaStream_t st, SweepWS& ws, ncclComm* comm, double* alpha_io,
                               double* beta_io, const double* row_sums_here = nullptr);
// true when every row sum lies in the fast update's safe range (one small kernel + a host round trip on `st`; summed over
// the ranks): a chain whose first update would be flagged goes straight to the log-sum-exp kernels
bool fast_sinkhorn_update_is_safe(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, const double* row_sums, DevBuf<double>& scratch);
void reset_sinkhorn_flag(regot_ctx* ctx, cudaStream_t st, SweepWS& ws);

// host <-> device helpers (ctx.cu)
void upload_dual(regot_ctx* ctx, const double* alpha_host, const double* beta_host, DVec& x, bool check_gauge,
                 const char* who);
void allreduce_sum(regot_ctx* ctx, ncclComm* comm, double* buf, size_t count, cudaStream_t st);
void allreduce_max(regot_ctx* ctx, ncclComm* comm, double* buf, size_t count, cudaStream_t st);

}  // namespace rg
