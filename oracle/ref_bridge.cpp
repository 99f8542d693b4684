// ref_bridge.cpp -- exposes the reference's OWN implementation (headers included unmodified from
// /root/reference/proj/include/regot, compiled over oracle/eigen_shim) through the same extern "C"
// surface as oracle_capi.cpp, so tests can run the restatement and the real reference code side by
// side and bench.py can time the reference itself.  TEST INFRASTRUCTURE ONLY; built by
// `make -C oracle ref` into oracle/_ref/libregot_ref.so, only where the reference tree is mounted.
#include "regot/core.h"
#include "regot/problem.h"
#include "regot/dual.h"
#include "regot/trace.h"
#include "regot/sinkhorn.h"
#include "regot/sparsity.h"
#include "regot/sparse_chol.h"
#include "regot/splr.h"
#include "regot/bench.h"

#include "../include/regot_b200.h"

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>

using namespace regot;

namespace {

thread_local std::string g_err;

int code_of(const std::exception& e)
{
    if (dynamic_cast<const DegenerateCostError*>(&e)) return 1;
    if (dynamic_cast<const FormatError*>(&e)) return 2;
    if (dynamic_cast<const TruncationError*>(&e)) return 3;
    if (dynamic_cast<const ValidationError*>(&e)) return 4;
    if (dynamic_cast<const IoError*>(&e)) return 5;
    if (dynamic_cast<const OracleSizeError*>(&e)) return 6;
    if (dynamic_cast<const StructureError*>(&e)) return 7;
    if (dynamic_cast<const NotPositiveDefiniteError*>(&e)) return 8;
    if (dynamic_cast<const DirectionError*>(&e)) return 9;
    if (dynamic_cast<const LineSearchError*>(&e)) return 10;
    if (dynamic_cast<const PlotError*>(&e)) return 11;
    if (dynamic_cast<const StepError*>(&e)) return 12;
    return 99;
}

template <class F>
int guarded(F&& body)
{
    try {
        body();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

ProblemInstance view(long n, long m, const double* M, const double* a, const double* b, double eta)
{
    ProblemInstance p;
    p.n = n;
    p.m = m;
    p.eta = eta;
    p.M.resize(n, m);
    std::memcpy(p.M.data(), M, sizeof(double) * (size_t)(n * m));
    p.a.resize(n);
    p.b.resize(m);
    std::memcpy(p.a.data(), a, sizeof(double) * (size_t)n);
    std::memcpy(p.b.data(), b, sizeof(double) * (size_t)m);
    return p;
}

DualPoint dual_of(long n, long m, const double* alpha, const double* beta)
{
    DualPoint x = DualPoint::zeros(n, m);
    std::memcpy(x.alpha.data(), alpha, sizeof(double) * (size_t)n);
    std::memcpy(x.beta.data(), beta, sizeof(double) * (size_t)m);
    return x;
}

void put(double* dst, const Vector& v)
{
    std::memcpy(dst, v.data(), sizeof(double) * (size_t)v.size());
}

void fill_trace(regot_result* out, const SolverTrace& t)
{
    out->n_trace = (int64_t)t.rows.size();
    out->trace = (regot_trace_row*)std::malloc(sizeof(regot_trace_row) * std::max<size_t>(1, t.rows.size()));
    for (size_t r = 0; r < t.rows.size(); ++r)
        out->trace[r] = {t.rows[r].iter, t.rows[r].wall_ms, t.rows[r].f, t.rows[r].marginal_error, t.rows[r].duality_gap};
    std::snprintf(out->algo, sizeof(out->algo), "%s", t.algo.c_str());
    std::snprintf(out->config_hash, sizeof(out->config_hash), "%s", t.config_hash.c_str());
}

void fill_point(regot_result* out, const DualPoint& x)
{
    out->alpha = (double*)std::malloc(sizeof(double) * (size_t)x.alpha.size());
    out->beta = (double*)std::malloc(sizeof(double) * (size_t)x.beta.size());
    put(out->alpha, x.alpha);
    put(out->beta, x.beta);
}

}  // namespace

extern "C" {

const char* rgo_last_error() { return g_err.c_str(); }

int rgo_gen_problem(const char* kind, long n, long m, long d, unsigned long long seed, double eta, double* M, double* a,
                    double* b)
{
    return guarded([&] {
        GeneratorSpec spec;
        spec.kind = kind;
        spec.n = n;
        spec.m = m;
        spec.d = d;
        spec.seed = seed;
        const ProblemInstance p = make_problem(spec, eta);  // synth1-iid | synth1-diff | synth2
        std::memcpy(M, p.M.data(), sizeof(double) * (size_t)(n * m));
        put(a, p.a);
        put(b, p.b);
    });
}

int rgo_plan(long n, long m, const double* M, const double* a, const double* b, double eta, const double* alpha,
             const double* beta, double* T)
{
    return guarded([&] {
        const Matrix t = plan(dual_of(n, m, alpha, beta), view(n, m, M, a, b, eta));
        std::memcpy(T, t.data(), sizeof(double) * (size_t)(n * m));
    });
}

int rgo_gradient(int which, long n, long m, const double* M, const double* a, const double* b, double eta,
                 const double* alpha, const double* beta, int tr, int tc, regot_gradient_info* info, double* grad,
                 double* row, double* col)
{
    return guarded([&] {
        const ProblemInstance p = view(n, m, M, a, b, eta);
        const DualPoint x = dual_of(n, m, alpha, beta);
        const GradientResult g = which == 0 ? fused_gradient(x, p, FusedTiling{tr, tc}) : naive_gradient(x, p);
        if (info) {
            info->f = g.f;
            info->marginal_error = marginal_error(g, p);
            info->duality_gap = duality_gap(x, g, p);
            info->grad_norm2 = g.grad.norm();
            info->total_mass = detail::pairwise_sum(g.row_sums.data(), n);
        }
        if (grad) put(grad, g.grad);
        if (row) put(row, g.row_sums);
        if (col) put(col, g.col_sums);
    });
}

int rgo_optimal_alpha(long n, long m, const double* M, const double* a, const double* b, double eta,
                      const double* alpha, const double* beta, double* out)
{
    return guarded([&] { put(out, optimal_alpha(dual_of(n, m, alpha, beta), view(n, m, M, a, b, eta))); });
}

int rgo_optimal_beta(long n, long m, const double* M, const double* a, const double* b, double eta,
                     const double* alpha, double* out)
{
    return guarded([&] {
        Vector al(n);
        std::memcpy(al.data(), alpha, sizeof(double) * (size_t)n);
        put(out, optimal_beta(al, view(n, m, M, a, b, eta)));
    });
}

int rgo_sinkhorn_step(long n, long m, const double* M, const double* a, const double* b, double eta, double* alpha_io,
                      double* beta_io)
{
    return guarded([&] {
        const DualPoint r = sinkhorn_step(dual_of(n, m, alpha_io, beta_io), view(n, m, M, a, b, eta));
        put(alpha_io, r.alpha);
        put(beta_io, r.beta);
    });
}

int rgo_select_topk(long n, long m, const double* T, long k, int* coords, long cap, long* count)
{
    return guarded([&] {
        Matrix Tm(n, m);
        std::memcpy(Tm.data(), T, sizeof(double) * (size_t)(n * m));
        const SparsityPattern om = select_topk(Tm, k);
        *count = (long)om.coords.size();
        for (long t = 0; t < std::min<long>(cap, *count); ++t) {
            coords[2 * t] = om.coords[(size_t)t].first;
            coords[2 * t + 1] = om.coords[(size_t)t].second;
        }
    });
}

long rgo_topk_budget(long n, long m, double density)
{
    ProblemInstance p;
    p.n = n;
    p.m = m;
    return topk_budget(p, density);
}

struct rgo_sparse {
    SparseSym A;
    ProblemInstance p;
};

int rgo_assemble(long n, long m, const double* M, const double* a, const double* b, double eta, const double* alpha,
                 const double* beta, const int* coords, long ncoords, double tau, rgo_sparse** out)
{
    return guarded([&] {
        auto h = std::make_unique<rgo_sparse>();
        h->p = view(n, m, M, a, b, eta);
        SparsityPattern om;
        om.n = n;
        om.mm1 = m - 1;
        for (long t = 0; t < ncoords; ++t) om.coords.emplace_back(coords[2 * t], coords[2 * t + 1]);
        h->A = assemble(dual_of(n, m, alpha, beta), h->p, om, tau);
        *out = h.release();
    });
}

int rgo_update_values(rgo_sparse* h, const double* alpha, const double* beta, double tau)
{
    return guarded([&] { update_values(h->A, dual_of(h->p.n, h->p.m, alpha, beta), h->p, tau); });
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
        Vector x(h->A.dim);
        std::memcpy(x.data(), v, sizeof(double) * (size_t)h->A.dim);
        put(y, h->A.matvec(x));
    });
}

int rgo_compute_direction(const rgo_sparse* h, const double* g, const double* u, const double* v, double xi, double zeta,
                          int solver, double, int, double* d, int* cg_iters)
{
    return guarded([&] {
        if (solver != 0) throw ValidationError("the reference has no PCG direction solver");
        const int dim = h->A.dim;
        LowRankTerm R;
        if (u && v) {
            R.active = true;
            R.u.resize(dim);
            R.v.resize(dim);
            std::memcpy(R.u.data(), u, sizeof(double) * (size_t)dim);
            std::memcpy(R.v.data(), v, sizeof(double) * (size_t)dim);
            R.xi = xi;
            R.zeta = zeta;
        }
        Vector gv(dim);
        std::memcpy(gv.data(), g, sizeof(double) * (size_t)dim);
        auto sym = std::make_shared<const SymbolicFactor>(symbolic_analyze(h->A));
        const NumericFactor F = numeric_factorize(sym, h->A);
        put(d, compute_direction(F, R, gv));
        if (cg_iters) *cg_iters = 0;
    });
}

void rgo_sparse_free(rgo_sparse* h) { delete h; }

int rgo_run_splr(long n, long m, const double* M, const double* a, const double* b, double eta, const double* alpha0,
                 const double* beta0, const regot_splr_config* c, int direction_solver, regot_result* out)
{
    std::memset(out, 0, sizeof(*out));
    return guarded([&] {
        if (direction_solver != 0) throw ValidationError("the reference has no PCG direction solver");
        const ProblemInstance p = view(n, m, M, a, b, eta);
        SplrConfig cfg;
        cfg.tau_max = c->tau_max;
        cfg.S = c->S;
        cfg.J = c->J;
        cfg.density = c->density;
        cfg.c1 = c->c1;
        cfg.c2 = c->c2;
        cfg.max_iter = c->max_iter;
        cfg.tol = c->tol;
        cfg.max_ls_trials = c->max_ls_trials;
        cfg.record_every = c->record_every;
        cfg.overlap = c->overlap != 0;
        cfg.tiling = FusedTiling{c->tile_rows, c->tile_cols};
        out->n = n;
        out->m = m;
        out->eta = eta;
        SplrResult r;
        try {
            r = run_splr(dual_of(n, m, alpha0, beta0), p, cfg);
        } catch (const StepError& e) {
            out->status = 12;
            std::snprintf(out->message, sizeof(out->message), "%s", e.what());
            fill_trace(out, e.trace());
            return;
        }
        fill_trace(out, r.trace);
        out->n_steps = (int64_t)r.steps.size();
        out->steps = (regot_step_record*)std::malloc(sizeof(regot_step_record) * std::max<size_t>(1, r.steps.size()));
        for (size_t s = 0; s < r.steps.size(); ++s) {
            const SplrStepRecord& q = r.steps[s];
            regot_step_record& o = out->steps[s];
            std::memset(&o, 0, sizeof(o));
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
        }
        fill_point(out, r.x);
    });
}

int rgo_run_sinkhorn(long n, long m, const double* M, const double* a, const double* b, double eta, const double* alpha0,
                     const double* beta0, const regot_sinkhorn_config* c, regot_result* out)
{
    std::memset(out, 0, sizeof(*out));
    return guarded([&] {
        SinkhornConfig cfg;
        cfg.max_iter = c->max_iter;
        cfg.record_every = c->record_every;
        cfg.tol = c->tol;
        const SinkhornResult r = run_sinkhorn(dual_of(n, m, alpha0, beta0), view(n, m, M, a, b, eta), cfg);
        out->n = n;
        out->m = m;
        out->eta = eta;
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

double rgo_time_gradient(long n, long m, const double* M, const double* a, const double* b, double eta,
                         const double* alpha, const double* beta, int reps)
{
    const ProblemInstance p = view(n, m, M, a, b, eta);
    const DualPoint x = dual_of(n, m, alpha, beta);
    const auto t0 = std::chrono::steady_clock::now();
    double sink = 0.0;
    for (int r = 0; r < reps; ++r) sink += fused_gradient(x, p).f;
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / reps;
    return sink == 12345.678 ? -s : s;
}

// ---- data formats either side of the path (problem.h:218-280, bench.h:243-256): used once, here, to
// write the golden ROTB / CSV fixtures under tests/golden with the reference's own writers ----
int rgo_save_problem(const char* path, long n, long m, const double* M, const double* a, const double* b, double eta)
{
    return guarded([&] { save_problem(view(n, m, M, a, b, eta), path); });
}

// M (column-major like every matrix on this surface), a, b may be NULL to query the dimensions first
int rgo_load_problem(const char* path, long* n, long* m, double* eta, double* M, double* a, double* b)
{
    return guarded([&] {
        const ProblemInstance p = load_problem(path);
        *n = (long)p.n;
        *m = (long)p.m;
        *eta = p.eta;
        if (M) std::memcpy(M, p.M.data(), sizeof(double) * (size_t)(p.n * p.m));
        if (a) put(a, p.a);
        if (b) put(b, p.b);
    });
}

int rgo_emit_trace_csv(const char* path, long nrows, const regot_trace_row* rows)
{
    return guarded([&] {
        SolverTrace t;
        t.algo = "splr";
        for (long r = 0; r < nrows; ++r)
            t.rows.push_back(TraceRow{(long)rows[r].iter, rows[r].wall_ms, rows[r].f, rows[r].marginal_error, rows[r].duality_gap});
        emit_csv(t, path);
    });
}

}  // extern "C"
