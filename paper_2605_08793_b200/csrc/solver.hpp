// solver.hpp -- host-side drivers (solver.cu) and their device workspace.
#pragma once

#include "ctx.hpp"
#include "sparse.hpp"
#include "vecops.hpp"

#include <chrono>
#include <vector>

namespace rg {

// Default relative tolerance of the PCG direction solves (preconditioned residual): tight enough
// that the direction matches the reference's exact sparse-Cholesky solve to ~1e-8 and the SPLR
// iteration counts track the oracle's ("PCG tolerance study": 1e-6 is ~30% faster at
// config B but moves small-problem iteration counts by up to 12%).
constexpr double kDefaultCgRtol = 1e-10;

struct WallClock {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    double ms() const
    {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
};

// Host-side result before it is flattened into regot_result.
struct SolveOut {
    regot_status status = REGOT_OK;
    std::string message;
    std::vector<regot_trace_row> trace;
    std::vector<regot_step_record> steps;
    std::vector<double> alpha, beta;  // global n / m (this rank's rows filled when sharded)
    double device_ms = 0.0;
    int64_t gradient_passes = 0, lse_passes = 0, kernel_launches = 0;
};

// SplrState (splr.h:82-97) on the device: the iterate and its gradient, the previous accepted iterate, the
// frozen pattern with its matrix, plus the vectors one step works in (so a step allocates nothing).
struct SplrStateDev {
    DVec x, x_prev, g_prev;
    GradOut cur;  // f, grad, row/col sums at x
    bool has_prev = false;
    regot_sparse A;  // H_Omega + tau I at the frozen pattern
    long iter = 0;
    // pattern reuse (regot_b200_set_pattern_reuse): share of the mass the pattern held when it was built, refreshes that kept it
    double mass_at_build = -1.0;
    int pattern_skips = 0;
    DevBuf<double> mass_scratch, chain_scratch;
    DVec x_build;  // the point the pattern was selected at
    // per-step scratch
    DVec xs, d, sdiff, ydiff, v, ag, au, av;
    GradOut cand;
    DVec tx[3];  // line-search trial points and their gradients (three rotating slots)
    GradOut tg[3];
};

// Everything the solvers keep on the device between calls.
struct SolverWS {
    DVec x, x_prev;  // run_sinkhorn
    GradOut cur;
    DVec ag, au, av, d;  // stand-alone compute_direction
    SplrStateDev splr;  // run_splr's state (splr_init / splr_step own theirs)
    DotScratch dots;
    SparseWS sparse;
};

SolverWS& solver_ws(regot_ctx* ctx);

void solve_sinkhorn(regot_ctx* ctx, const double* alpha0, const double* beta0, const regot_sinkhorn_config& cfg,
                    SolveOut& out);
void solve_splr(regot_ctx* ctx, const double* alpha0, const double* beta0, const regot_splr_config& cfg, SolveOut& out);
// splr_init (splr.h:326-334) / splr_step (splr.h:348-478) on a caller-owned state; stats (nullable) counts passes
void splr_init_state(regot_ctx* ctx, const double* alpha0, const double* beta0, SplrStateDev& S, SolveOut* stats);
void splr_step_state(regot_ctx* ctx, SplrStateDev& S, const regot_splr_config& cfg, regot_step_record& rec, SolveOut* stats);
// st.x to the host (alpha allgathered over the ranks when sharded)
void download_point(regot_ctx* ctx, const DVec& x, std::vector<double>& alpha, std::vector<double>& beta);

// compute_direction alone (regot_b200_compute_direction); false on PCG breakdown
bool compute_direction_api(regot_ctx* ctx, const regot_sparse& A, const DVec& g, double g_sqnorm, bool active, double xi,
                           double zeta, const DVec& u, const DVec& v, double rtol, int max_iter, DVec& d, int& cg_iters);

}  // namespace rg
