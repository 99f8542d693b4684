// regot_b200.hpp -- header-only C++ mirror of the reference's solver interface over the C ABI
// (include/regot_b200.h).  Same names, argument meaning and error behaviour as `namespace regot`
// (/root/reference/proj/include/regot/*.h), so code written against the reference changes one
// namespace:
//
//     regot::ProblemInstance / DualPoint / GradientResult      problem.h:20-28, dual.h:14-56
//     regot::SplrConfig / SinkhornConfig / SolverTrace          splr.h:22-60, sinkhorn.h:16-31, trace.h:22-41
//     regot::run_splr / run_sinkhorn / fused_gradient / ...      splr.h:487, sinkhorn.h:123, dual.h:106
//
// Differences forced by the device: the cost matrix is a flat std::vector<double> with an explicit
// layout flag (the reference's Eigen::MatrixXd is column-major: layout 0), and a Solver object owns
// the GPU context + the uploaded problem.  The free functions below keep the reference's
// `(x, problem, config)` signatures by binding a process-wide Solver to the problem on first use.
//
// Link with -lregot_b200.  There is no CPU fallback: construction throws CudaError without a GPU.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "regot_b200.h"

namespace regot_b200 {

using Vector = std::vector<double>;
using Index = std::int64_t;

// ---- errors: one class per reference exception (core.h:21-37) ---------------------------------
class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
#define REGOT_B200_ERROR(name) \
    class name : public Error { \
    public: \
        using Error::Error; \
    }
REGOT_B200_ERROR(DegenerateCostError);
REGOT_B200_ERROR(FormatError);
REGOT_B200_ERROR(TruncationError);
REGOT_B200_ERROR(ValidationError);
REGOT_B200_ERROR(IoError);
REGOT_B200_ERROR(OracleSizeError);
REGOT_B200_ERROR(StructureError);
REGOT_B200_ERROR(NotPositiveDefiniteError);
REGOT_B200_ERROR(DirectionError);
REGOT_B200_ERROR(LineSearchError);
REGOT_B200_ERROR(PlotError);
REGOT_B200_ERROR(CudaError);
REGOT_B200_ERROR(NcclError);
REGOT_B200_ERROR(DeviceMemoryError);
REGOT_B200_ERROR(UnsupportedError);
#undef REGOT_B200_ERROR

[[noreturn]] inline void throw_status(regot_status st, const std::string& msg)
{
    switch (st) {
    case REGOT_E_DEGENERATE_COST: throw DegenerateCostError(msg);
    case REGOT_E_FORMAT: throw FormatError(msg);
    case REGOT_E_TRUNCATION: throw TruncationError(msg);
    case REGOT_E_VALIDATION: throw ValidationError(msg);
    case REGOT_E_IO: throw IoError(msg);
    case REGOT_E_ORACLE_SIZE: throw OracleSizeError(msg);
    case REGOT_E_STRUCTURE: throw StructureError(msg);
    case REGOT_E_NOT_POSITIVE_DEFINITE: throw NotPositiveDefiniteError(msg);
    case REGOT_E_DIRECTION: throw DirectionError(msg);
    case REGOT_E_LINE_SEARCH: throw LineSearchError(msg);
    case REGOT_E_PLOT: throw PlotError(msg);
    case REGOT_E_NCCL: throw NcclError(msg);
    case REGOT_E_NOMEM: throw DeviceMemoryError(msg);
    case REGOT_E_UNSUPPORTED: throw UnsupportedError(msg);
    default: throw CudaError(msg);
    }
}

// ---- value types ------------------------------------------------------------------------------------
// problem.h:20-28.  M holds n*m doubles in `layout` (REGOT_LAYOUT_COLMAJOR like Eigen, or ROWMAJOR).
struct ProblemInstance {
    Index n = 0, m = 0;
    Vector M;
    int layout = REGOT_LAYOUT_COLMAJOR;
    Vector a, b;
    double eta = 0.0;
};

// dual.h:14-47
struct DualPoint {
    Vector alpha, beta;
    static DualPoint zeros(Index n, Index m)
    {
        DualPoint x;
        x.alpha.assign((std::size_t)n, 0.0);
        x.beta.assign((std::size_t)m, 0.0);
        return x;
    }
    static DualPoint from_free(const Vector& xf, Index n, Index m)
    {
        if ((Index)xf.size() != n + m - 1) throw ValidationError("DualPoint::from_free: length mismatch");
        DualPoint x;
        x.alpha.assign(xf.begin(), xf.begin() + n);
        x.beta.assign(xf.begin() + n, xf.end());
        x.beta.push_back(0.0);
        return x;
    }
    Vector to_free() const
    {
        Vector xf(alpha);
        xf.insert(xf.end(), beta.begin(), beta.end() - 1);
        return xf;
    }
};

// dual.h:50-56 (+ the scalars the device epilogue produces in the same pass)
struct GradientResult {
    double f = 0.0;
    Vector grad, row_sums, col_sums;
    double marginal_error = 0.0, duality_gap = 0.0, grad_norm2 = 0.0;
};

struct FusedTiling {
    int rows = 8, cols = 32;
};

// splr.h:22-60
struct SplrConfig {
    double tau_max = 1.0;
    long S = 10, J = 5;
    double density = 0.01, c1 = 1e-4, c2 = 0.9;
    long max_iter = 1000;
    double tol = 1e-8;
    long max_ls_trials = 30, record_every = 1;
    bool overlap = false;
    FusedTiling tiling;
    int cg_max_iter = 0;   // extension: 0 -> library default
    double cg_rtol = 0.0;  // extension: 0 -> library default

    regot_splr_config c() const
    {
        regot_splr_config k;
        regot_b200_splr_config_default(&k);
        k.tau_max = tau_max; k.S = S; k.J = J; k.density = density; k.c1 = c1; k.c2 = c2; k.max_iter = max_iter;
        k.tol = tol; k.max_ls_trials = max_ls_trials; k.record_every = record_every; k.overlap = overlap ? 1 : 0;
        k.tile_rows = tiling.rows; k.tile_cols = tiling.cols; k.cg_max_iter = cg_max_iter; k.cg_rtol = cg_rtol;
        return k;
    }
    void validate() const
    {
        const regot_splr_config k = c();
        const regot_status st = regot_b200_splr_config_validate(&k);
        if (st != REGOT_OK) throw_status(st, regot_b200_last_error(nullptr));
    }
};

// sinkhorn.h:16-31
struct SinkhornConfig {
    long max_iter = 1000, record_every = 1;
    double tol = 0.0;
    regot_sinkhorn_config c() const { return regot_sinkhorn_config{max_iter, record_every, tol}; }
    void validate() const
    {
        const regot_sinkhorn_config k = c();
        const regot_status st = regot_b200_sinkhorn_config_validate(&k);
        if (st != REGOT_OK) throw_status(st, regot_b200_last_error(nullptr));
    }
};

inline std::string splr_config_hash(const SplrConfig& cfg)
{
    char buf[17];
    const regot_splr_config k = cfg.c();
    regot_b200_splr_config_hash(&k, buf);
    return buf;
}
inline std::string sinkhorn_config_hash(const SinkhornConfig& cfg)
{
    char buf[17];
    const regot_sinkhorn_config k = cfg.c();
    regot_b200_sinkhorn_config_hash(&k, buf);
    return buf;
}

// trace.h:11-41
struct TraceRow {
    long iter = 0;
    double wall_ms = 0.0, f = 0.0, marginal_error = 0.0, duality_gap = 0.0;
};
struct SolverTrace {
    std::string algo, problem;
    double eta = 0.0;
    std::string config_hash;
    std::vector<TraceRow> rows;
    void append(const TraceRow& r)
    {
        if (!rows.empty()) {
            if (r.iter <= rows.back().iter) throw ValidationError("SolverTrace: iter must be strictly increasing");
            if (r.wall_ms < rows.back().wall_ms) throw ValidationError("SolverTrace: wall_ms must be nondecreasing");
        }
        rows.push_back(r);
    }
};

// splr.h:294-312 (+ cg_iters)
struct SplrStepRecord {
    long iter = 0;
    bool refresh = false, sinkhorn_selected = false;
    double f_before = 0.0, f_after = 0.0;
    double f_cand_sinkhorn = std::numeric_limits<double>::quiet_NaN();
    double f_cand_qn = 0.0, gamma = 0.0, g_dot_d = 0.0, gnew_dot_d = 0.0;
    bool curvature_ok = false, ls_failed = false, lowrank_active = false;
    double tau = 0.0;
    int factor_retries = 0, ls_evals = 0, cg_iters = 0;
};

// splr.h:315-324
class StepError : public Error {
public:
    StepError(const std::string& msg, SolverTrace trace) : Error(msg), m_trace(std::move(trace)) {}
    const SolverTrace& trace() const { return m_trace; }

private:
    SolverTrace m_trace;
};

struct SplrResult {
    DualPoint x;
    SolverTrace trace;
    std::vector<SplrStepRecord> steps;
    double device_ms = 0.0;
};
struct SinkhornResult {
    DualPoint x;
    SolverTrace trace;
    double device_ms = 0.0;
};

// ---- device handle ----------------------------------------------------------------------------------
class Solver {
public:
    explicit Solver(int device = 0)
    {
        const regot_status st = regot_b200_create(device, &m_ctx);
        if (st != REGOT_OK) throw_status(st, regot_b200_last_error(nullptr));
    }
    ~Solver() { regot_b200_destroy(m_ctx); }
    Solver(const Solver&) = delete;
    Solver& operator=(const Solver&) = delete;

    void set_problem(const ProblemInstance& p)
    {
        if ((Index)p.M.size() != p.n * p.m) throw ValidationError("problem: cost matrix shape mismatch");
        if ((Index)p.a.size() != p.n || (Index)p.b.size() != p.m) throw ValidationError("problem: marginal length mismatch");
        check(regot_b200_set_problem(m_ctx, p.n, p.m, p.M.data(), p.layout, p.layout == REGOT_LAYOUT_COLMAJOR ? p.n : p.m,
                                     p.a.data(), p.b.data(), p.eta));
        m_n = p.n;
        m_m = p.m;
        m_bound = &p;
    }
    // squared-Euclidean cost of point clouds / max, formed on the device (problem.h:124-132, 53-61);
    // on_the_fly: the matrix is never stored (every pass recomputes its tiles)
    void set_pointcloud(Index n, Index m, int d, const Vector& X, const Vector& Y, const Vector& a, const Vector& b,
                        double eta, bool on_the_fly = false)
    {
        if ((Index)X.size() != n * d || (Index)Y.size() != m * d) throw ValidationError("set_pointcloud: cloud shape mismatch");
        if ((Index)a.size() != n || (Index)b.size() != m) throw ValidationError("problem: marginal length mismatch");
        check(regot_b200_set_pointcloud(m_ctx, n, m, d, X.data(), Y.data(), a.data(), b.data(), eta, on_the_fly ? 1 : 0));
        m_n = n;
        m_m = m;
        m_bound = nullptr;
    }
    void ensure_problem(const ProblemInstance& p)
    {
        if (m_bound != &p) set_problem(p);
    }
    void validate_problem() { check(regot_b200_validate_problem(m_ctx)); }
    // north_star item (2): rebuild the top-k pattern at k % S == 0 only when it drifted (0: the reference's fixed rule)
    void set_pattern_reuse(double drift_tol, int max_skips = 4) { check(regot_b200_set_pattern_reuse(m_ctx, drift_tol, max_skips)); }

    // dual.h:106-164
    GradientResult fused_gradient(const DualPoint& x)
    {
        dims(x, "fused_gradient");
        GradientResult g;
        g.grad.resize((std::size_t)(m_n + m_m - 1));
        g.row_sums.resize((std::size_t)m_n);
        g.col_sums.resize((std::size_t)m_m);
        regot_gradient_info info;
        check(regot_b200_fused_gradient(m_ctx, x.alpha.data(), x.beta.data(), &info, g.grad.data(), g.row_sums.data(),
                                        g.col_sums.data()));
        g.f = info.f;
        g.marginal_error = info.marginal_error;
        g.duality_gap = info.duality_gap;
        g.grad_norm2 = info.grad_norm2;
        return g;
    }
    // sinkhorn.h:105-115
    DualPoint sinkhorn_step(const DualPoint& x)
    {
        dims(x, "sinkhorn_step");
        DualPoint y = x;
        check(regot_b200_sinkhorn_step(m_ctx, y.alpha.data(), y.beta.data()));
        return y;
    }
    // sinkhorn.h:123-171
    SinkhornResult run_sinkhorn(const DualPoint& x0, const SinkhornConfig& cfg)
    {
        dims(x0, "run_sinkhorn");
        const regot_sinkhorn_config k = cfg.c();
        regot_result r;
        const regot_status st = regot_b200_run_sinkhorn(m_ctx, x0.alpha.data(), x0.beta.data(), &k, &r);
        Holder h{&r};
        check(st);
        SinkhornResult out;
        out.trace = trace_of(r);
        out.x = point_of(r);
        out.device_ms = r.device_ms;
        return out;
    }
    // splr.h:487-534
    SplrResult run_splr(const DualPoint& x0, const SplrConfig& cfg)
    {
        dims(x0, "run_splr");
        const regot_splr_config k = cfg.c();
        regot_result r;
        const regot_status st = regot_b200_run_splr(m_ctx, x0.alpha.data(), x0.beta.data(), &k, &r);
        Holder h{&r};
        if (st == REGOT_E_STEP) throw StepError(r.message, trace_of(r));
        check(st);
        SplrResult out;
        out.trace = trace_of(r);
        out.x = point_of(r);
        out.device_ms = r.device_ms;
        for (std::int64_t s = 0; s < r.n_steps; ++s) {
            const regot_step_record& q = r.steps[s];
            SplrStepRecord o;
            o.iter = (long)q.iter; o.refresh = q.refresh != 0; o.sinkhorn_selected = q.sinkhorn_selected != 0;
            o.f_before = q.f_before; o.f_after = q.f_after; o.f_cand_sinkhorn = q.f_cand_sinkhorn; o.f_cand_qn = q.f_cand_qn;
            o.gamma = q.gamma; o.g_dot_d = q.g_dot_d; o.gnew_dot_d = q.gnew_dot_d; o.curvature_ok = q.curvature_ok != 0;
            o.ls_failed = q.ls_failed != 0; o.lowrank_active = q.lowrank_active != 0; o.tau = q.tau;
            o.factor_retries = q.factor_retries; o.ls_evals = q.ls_evals; o.cg_iters = q.cg_iters;
            out.steps.push_back(o);
        }
        return out;
    }
    regot_ctx* handle() const { return m_ctx; }

private:
    struct Holder {
        regot_result* r;
        ~Holder() { regot_b200_result_free(r); }
    };
    void check(regot_status st) const
    {
        if (st != REGOT_OK) throw_status(st, regot_b200_last_error(m_ctx));
    }
    void dims(const DualPoint& x, const char* who) const
    {
        if ((Index)x.alpha.size() != m_n || (Index)x.beta.size() != m_m)
            throw ValidationError(std::string(who) + ": dual point/problem dimension mismatch");
    }
    static SolverTrace trace_of(const regot_result& r)
    {
        SolverTrace t;
        t.algo = r.algo;
        t.eta = r.eta;
        t.config_hash = r.config_hash;
        for (std::int64_t k = 0; k < r.n_trace; ++k)
            t.rows.push_back({(long)r.trace[k].iter, r.trace[k].wall_ms, r.trace[k].f, r.trace[k].marginal_error,
                              r.trace[k].duality_gap});
        return t;
    }
    static DualPoint point_of(const regot_result& r)
    {
        DualPoint x;
        if (r.alpha && r.beta) {
            x.alpha.assign(r.alpha, r.alpha + r.n);
            x.beta.assign(r.beta, r.beta + r.m);
        }
        return x;
    }
    regot_ctx* m_ctx = nullptr;
    Index m_n = 0, m_m = 0;
    const ProblemInstance* m_bound = nullptr;
};

// ---- free functions with the reference's signatures -------------------------------------------------------
inline Solver& default_solver()
{
    static Solver s(0);
    return s;
}
inline GradientResult fused_gradient(const DualPoint& x, const ProblemInstance& p, const FusedTiling& tile = FusedTiling())
{
    if (tile.rows < 1 || tile.cols < 1) throw ValidationError("fused_gradient: invalid tile shape");
    default_solver().ensure_problem(p);
    return default_solver().fused_gradient(x);
}
inline double objective(const DualPoint& x, const ProblemInstance& p) { return fused_gradient(x, p).f; }
inline double marginal_error(const GradientResult& gr, const ProblemInstance&) { return gr.marginal_error; }
inline double duality_gap(const DualPoint&, const GradientResult& gr, const ProblemInstance&) { return gr.duality_gap; }
inline DualPoint sinkhorn_step(const DualPoint& x, const ProblemInstance& p)
{
    default_solver().ensure_problem(p);
    return default_solver().sinkhorn_step(x);
}
inline SinkhornResult run_sinkhorn(const DualPoint& x0, const ProblemInstance& p, const SinkhornConfig& cfg)
{
    default_solver().ensure_problem(p);
    return default_solver().run_sinkhorn(x0, cfg);
}
inline SplrResult run_splr(const DualPoint& x0, const ProblemInstance& p, const SplrConfig& cfg)
{
    default_solver().ensure_problem(p);
    return default_solver().run_splr(x0, cfg);
}
inline long topk_budget(const ProblemInstance& p, double density) { return (long)regot_b200_topk_budget(p.n, p.m, density); }

}  // namespace regot_b200
