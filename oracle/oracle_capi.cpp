// oracle_capi.cpp -- extern "C" surface of the CPU oracle (TEST INFRASTRUCTURE
// ONLY; see the header of regot_oracle.hpp).  Loaded with ctypes by tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs.
//
// Stateless: every call receives the problem arrays (cost matrix COLUMN-MAJOR,
// like the reference's Eigen::MatrixXd).  Struct layouts are shared with the
// product ABI (include/regot_b200.h) so traces and step records can be compared
// field by field.
#include "regot_oracle.hpp"

#include "../include/regot_b200.h"

#include <cstdio>
#include <cstdlib>

using namespace rgo;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& body)
{
    try {
        body();
        return OK;
    } catch (const Failure& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 99;
    }
}

Problem view(long n, long m, const double* M, const double* a, const double* b, double eta)
{
    Problem p;
    p.n = n;
    p.m = m;
    p.eta = eta;
    p.M.assign(M, M + n * m);
    p.a.assign(a, a + n);
    p.b.assign(b, b + m);
    return p;
}

Dual dual_of(long n, long m, const double* alpha, const double* beta)
{
    Dual x;
    x.alpha.assign(alpha, alpha + n);
    x.beta.assign(beta, beta + m);
    return x;
}

SplrConfig cfg_of(const regot_splr_config* c)
{
    SplrConfig k;
    k.tau_max = c->tau_max;
    k.S = c->S;
    k.J = c->J;
    k.density = c->density;
    k.c1 = c->c1;
    k.c2 = c->c2;
    k.max_iter = c->max_iter;
    k.tol = c->tol;
    k.max_ls_trials = c->max_ls_trials;
    k.record_every = c->record_every;
    k.overlap = c->overlap != 0;
    k.tile_rows = c->tile_rows;
    k.tile_cols = c->tile_cols;
    return k;
}

void fill_trace(regot_result* out, const std::vector<TraceRow>& rows)
{
    out->n_trace = (int64_t)rows.size();
    out->trace = (regot_trace_row*)std::malloc(sizeof(regot_trace_row) * std::max<std::size_t>(1, rows.size()));
    for (std::size_t r = 0; r < rows.size(); ++r)
        out->trace[r] = {rows[r].iter, rows[r].wall_ms, rows[r].f, rows[r].marginal_error, rows[r].duality_gap};
}

void fill_point(regot_result* out, const Dual& x)
{
    out->alpha = (double*)std::malloc(sizeof(double) * x.alpha.size());
    out->beta = (double*)std::malloc(sizeof(double) * x.beta.size());
    std::memcpy(out->alpha, x.alpha.data(), sizeof(double) * x.alpha.size());
    std::memcpy(out->beta, x.beta.data(), sizeof(double) * x.beta.size());
}

}  // namespace

extern "C" {

const char* rgo_last_error() { return g_err.c_str(); }

// kinds: synth1-iid, synth1-diff, synth2 (problem.h), rand (tests/oracles.h),
// image (config B; n = m = side^2, pass side in d), gmm / uniform (configs D/E)
int rgo_gen_problem(const char* kind, long n, long m, long d, unsigned long long seed, double eta, double* M,
                    double* a, double* b)
{
    return guarded([&] {
        const std::string k(kind);
        Problem p;
        if (k == "synth1-iid") p = gen_synthetic1(n, m, 0, d, seed, eta);
        else if (k == "synth1-diff") p = gen_synthetic1(n, m, 1, d, seed, eta);
        else if (k == "synth2") p = gen_synthetic2(n, m, eta);
        else if (k == "rand") p = rand_instance(n, m, eta, seed);
        else if (k == "image") p = gen_image(d, eta);
        else if (k == "gmm" || k == "uniform") {
            vec X, Y;
            if (k == "gmm") gen_gmm_points(X, Y, n, m, d, seed);
            else gen_uniform_points(X, Y, n, m, d, seed);
            p = problem_from_points(X, Y, n, m, d, eta);
        } else fail(E_VALIDATION, "make_problem: unknown generator kind '" + k + "'");
        if (p.n != n || p.m != m) fail(E_VALIDATION, "rgo_gen_problem: size mismatch");
        std::memcpy(M, p.M.data(), sizeof(double) * p.M.size());
        std::memcpy(a, p.a.data(), sizeof(double) * p.a.size());
        std::memcpy(b, p.b.data(), sizeof(double) * p.b.size());
    });
}

int rgo_gen_points(const char* kind, long n, long m, long d, unsigned long long seed, double* X, double* Y)
{
    return guarded([&] {
        vec x, y;
        if (std::string(kind) == "gmm") gen_gmm_points(x, y, n, m, d, seed);
        else gen_uniform_points(x, y, n, m, d, seed);
        std::memcpy(X, x.data(), sizeof(double) * x.size());
        std::memcpy(Y, y.data(), sizeof(double) * y.size());
    });
}

int rgo_validate_problem(long n, long m, const double* M, const double* a, const double* b, double eta)
{
    return guarded([&] { validate_problem(view(n, m, M, a, b, eta)); });
}

int rgo_rand_dual(long n, long m, double scale, unsigned long long seed, double* alpha, double* beta)
{
    return guarded([&] {
        const Dual x = rand_dual(n, m, scale, seed);
        std::memcpy(alpha, x.alpha.data(), sizeof(double) * (std::size_t)n);
        std::memcpy(beta, x.beta.data(), sizeof(double) * (std::size_t)m);
    });
}

double rgo_rng_uniform_nth(unsigned long long seed, long nth)
{
    Rng r(seed);
    double v = 0.0;
    for (long i = 0; i <= nth; ++i) v = r.uniform();
    return v;
}

int rgo_plan(long n, long m, const double* M, const double* a, const double* b, double eta, const double* alpha,
             const double* beta, double* T)
{
    return guarded([&] {
        const vec t = plan(dual_of(n, m, alpha, beta), view(n, m, M, a, b, eta));
        std::memcpy(T, t.data(), sizeof(double) * t.size());
    });
}

// which: 0 fused (tile tr x tc), 1 naive two-pass
int rgo_gradient(int which, long n, long m, const double* M, const double* a, const double* b, double eta,
                 const double* alpha, const double* beta, int tr, int tc, regot_gradient_info* info, double* grad,
                 double* row, double* col)
{
    return guarded([&] {
        const Problem p = view(n, m, M, a, b, eta);
        const Dual x = dual_of(n, m, alpha, beta);
        const Grad g = which == 0 ? fused_gradient(x, p, tr, tc) : naive_gradient(x, p);
        if (info) {
            info->f = g.f;
            info->marginal_error = marginal_error(g, p);
            info->duality_gap = duality_gap(x, g, p);
            info->grad_norm2 = norm2(g.grad);
            info->total_mass = pairwise_sum(g.row.data(), n);
        }
        if (grad) std::memcpy(grad, g.grad.data(), sizeof(double) * g.grad.size());
        if (row) std::memcpy(row, g.row.data(), sizeof(double) * g.row.size());
        if (col) std::memcpy(col, g.col.data(), sizeof(double) * g.col.size());
    });
}

int rgo_optimal_alpha(long n, long m, const double* M, const double* a, const double* b, double eta,
                      const double* alpha, const double* beta, double* out)
{
    return guarded([&] {
        const vec r = optimal_alpha(dual_of(n, m, alpha, beta), view(n, m, M, a, b, eta));
        std::memcpy(out, r.data(), sizeof(double) * r.size());
    });
}

int rgo_optimal_beta(long n, long m, const double* M, const double* a, const double* b, double eta,
                     const double* alpha, double* out)
{
    return guarded([&] {
        const vec r = optimal_beta(vec(alpha, alpha + n), view(n, m, M, a, b, eta));
        std::memcpy(out, r.data(), sizeof(double) * r.size());
    });
}

int rgo_sinkhorn_step(long n, long m, const double* M, const double* a, const double* b, double eta,
                      double* alpha_io, double* beta_io)
{
    return guarded([&] {
        const Dual r = sinkhorn_step(dual_of(n, m, alpha_io, beta_io), view(n, m, M, a, b, eta));
        std::memcpy(alpha_io, r.alpha.data(), sizeof(double) * (std::size_t)n);
        std::memcpy(beta_io, r.beta.data(), sizeof(double) * (std::size_t)m);
    });
}

// T column-major n x m.  coords receives (i, j) pairs.
int rgo_select_topk(long n, long m, const double* T, long k, int* coords, long cap, long* count)
{
    return guarded([&] {
        const Pattern om = select_topk(vec(T, T + n * m), n, m, k);
        *count = (long)om.coords.size();
        for (long t = 0; t < std::min<long>(cap, *count); ++t) {
            coords[2 * t] = om.coords[(std::size_t)t].first;
            coords[2 * t + 1] = om.coords[(std::size_t)t].second;
        }
    });
}

long rgo_topk_budget(long n, long m, double density)
{
    Problem p;
    p.n = n;
    p.m = m;
    return topk_budget(p, density);
}

// ---- sparse handle ------------------------------------------------------------
struct rgo_sparse {
    SparseSym A;
    Problem p;
};

int rgo_assemble(long n, long m, const double* M, const double* a, const double* b, double eta,
                 const double* alpha, const double* beta, const int* coords, long ncoords, double tau,
                 rgo_sparse** out)
{
    return guarded([&] {
        auto h = std::make_unique<rgo_sparse>();
        h->p = view(n, m, M, a, b, eta);
        const Dual x = dual_of(n, m, alpha, beta);
        Pattern om;
        om.n = n;
        om.mm1 = m - 1;
        for (long t = 0; t < ncoords; ++t) om.coords.emplace_back(coords[2 * t], coords[2 * t + 1]);
        h->A = assemble(x, h->p, om, tau, fused_gradient(x, h->p));
        *out = h.release();
    });
}

int rgo_update_values(rgo_sparse* h, const double* alpha, const double* beta, double tau)
{
    return guarded([&] {
        const Dual x = dual_of(h->p.n, h->p.m, alpha, beta);
        update_values(h->A, x, h->p, tau, fused_gradient(x, h->p));
    });
}

void rgo_sparse_info(const rgo_sparse* h, int* dim, long* nnz, long* ncoords, unsigned long long* pattern_id)
{
    *dim = h->A.dim;
    *nnz = (long)h->A.rowidx.size();
    *ncoords = (long)h->A.coords.size();
    *pattern_id = h->A.pattern_id;
}

void rgo_sparse_export(const rgo_sparse* h, int* colptr, int* rowidx, double* values)
{
    std::memcpy(colptr, h->A.colptr.data(), sizeof(int) * h->A.colptr.size());
    std::memcpy(rowidx, h->A.rowidx.data(), sizeof(int) * h->A.rowidx.size());
    std::memcpy(values, h->A.values.data(), sizeof(double) * h->A.values.size());
}

int rgo_matvec(const rgo_sparse* h, const double* v, double* y)
{
    return guarded([&] {
        const vec r = h->A.matvec(vec(v, v + h->A.dim));
        std::memcpy(y, r.data(), sizeof(double) * r.size());
    });
}

// compute_direction through the reference's sparse Cholesky route (solver = 0)
// or the PCG model (solver = 1).  u == NULL -> inactive low-rank term.
int rgo_compute_direction(const rgo_sparse* h, const double* g, const double* u, const double* v, double xi,
                          double zeta, int solver, double cg_rtol, int cg_max_iter, double* d, int* cg_iters)
{
    return guarded([&] {
        const int dim = h->A.dim;
        LowRank R;
        if (u && v) {
            R.active = true;
            R.u.assign(u, u + dim);
            R.v.assign(v, v + dim);
            R.xi = xi;
            R.zeta = zeta;
        }
        const vec gv(g, g + dim);
        vec dir;
        int used = 0;
        if (solver == 0) {
            auto sym = std::make_shared<const Symbolic>(symbolic_analyze(h->A));
            const Numeric F = numeric_factorize(sym, h->A);
            dir = compute_direction(F, R, gv);
        } else {
            dir = compute_direction_with(
                [&](const vec& r) {
                    vec s;
                    const int it = pcg_solve(h->A, r, s, cg_rtol, cg_max_iter);
                    if (it < 0) fail(E_NOT_POSITIVE_DEFINITE, "pcg breakdown");
                    used += it;
                    return s;
                },
                R, gv);
        }
        if (cg_iters) *cg_iters = used;
        std::memcpy(d, dir.data(), sizeof(double) * dir.size());
    });
}

void rgo_sparse_free(rgo_sparse* h) { delete h; }

// ---- solvers -----------------------------------------------------------------
// direction_solver: 0 reference sparse Cholesky, 1 PCG model of the device path
int rgo_run_splr(long n, long m, const double* M, const double* a, const double* b, double eta,
                 const double* alpha0, const double* beta0, const regot_splr_config* cfg, int direction_solver,
                 regot_result* out)
{
    std::memset(out, 0, sizeof(*out));
    return guarded([&] {
        const Problem p = view(n, m, M, a, b, eta);
        SplrConfig k = cfg_of(cfg);
        k.direction_solver = direction_solver;
        if (cfg->cg_rtol > 0.0) k.cg_rtol = cfg->cg_rtol;
        if (cfg->cg_max_iter > 0) k.cg_max_iter = cfg->cg_max_iter;
        const SplrResult r = run_splr(dual_of(n, m, alpha0, beta0), p, k);
        out->status = r.status;
        out->n = n;
        out->m = m;
        out->eta = eta;
        std::snprintf(out->algo, sizeof(out->algo), "splr");
        std::snprintf(out->message, sizeof(out->message), "%s", r.message.c_str());
        fill_trace(out, r.trace);
        out->n_steps = (int64_t)r.steps.size();
        out->steps = (regot_step_record*)std::malloc(sizeof(regot_step_record) * std::max<std::size_t>(1, r.steps.size()));
        for (std::size_t s = 0; s < r.steps.size(); ++s) {
            const StepRecord& q = r.steps[s];
            regot_step_record& o = out->steps[s];
            o.iter = q.iter;
            o.refresh = q.refresh;
            o.sinkhorn_selected = q.sinkhorn_selected;
            o.f_before = q.f_before;
            o.f_after = q.f_after;
            o.f_cand_sinkhorn = q.f_cand_sinkhorn;
            o.f_cand_qn = q.f_cand_qn;
            o.gamma = q.gamma;
            o.g_dot_d = q.g_dot_d;
            o.gnew_dot_d = q.gnew_dot_d;
            o.curvature_ok = q.curvature_ok;
            o.ls_failed = q.ls_failed;
            o.lowrank_active = q.lowrank_active;
            o.factor_retries = q.factor_retries;
            o.tau = q.tau;
            o.ls_evals = q.ls_evals;
            o.cg_iters = q.cg_iters;
        }
        if (r.status == OK) fill_point(out, r.x);
    });
}

int rgo_run_sinkhorn(long n, long m, const double* M, const double* a, const double* b, double eta,
                     const double* alpha0, const double* beta0, const regot_sinkhorn_config* cfg, regot_result* out)
{
    std::memset(out, 0, sizeof(*out));
    return guarded([&] {
        const Problem p = view(n, m, M, a, b, eta);
        SinkhornConfig k;
        k.max_iter = cfg->max_iter;
        k.record_every = cfg->record_every;
        k.tol = cfg->tol;
        const SinkhornResult r = run_sinkhorn(dual_of(n, m, alpha0, beta0), p, k);
        out->status = OK;
        out->n = n;
        out->m = m;
        out->eta = eta;
        std::snprintf(out->algo, sizeof(out->algo), "sinkhorn");
        fill_trace(out, r.trace);
        fill_point(out, r.x);
    });
}

void rgo_result_free(regot_result* r)
{
    std::free(r->alpha);
    std::free(r->beta);
    std::free(r->trace);
    std::free(r->steps);
    std::memset(r, 0, sizeof(*r));
}

// Timed loops for bench.py's cpu_baseline leg: `reps` fused-gradient passes (or
// Sinkhorn steps) on one thread; returns seconds per call.
double rgo_time_gradient(long n, long m, const double* M, const double* a, const double* b, double eta,
                         const double* alpha, const double* beta, int reps)
{
    const Problem p = view(n, m, M, a, b, eta);
    const Dual x = dual_of(n, m, alpha, beta);
    WallClock clk;
    double sink = 0.0;
    for (int r = 0; r < reps; ++r) sink += fused_gradient(x, p).f;
    const double s = clk.ms() * 1e-3 / reps;
    return sink == 12345.678 ? -s : s;
}

}  // extern "C"
