// capi.cu -- extern "C" boundary (include/regot_b200.h): context, problem upload,
// dual kernels, configuration structs.  Solver and sparse entry points live in
// capi_solver.cu.
#include "ctx.hpp"
#include "capi_util.hpp"

#include <cmath>
#include <cstring>
#include <sstream>

namespace rg {
regot_ctx* ctx_create(int device);
void ctx_destroy(regot_ctx* ctx);
void nccl_unique_id(void* out128);
void comm_init(regot_ctx* ctx, int rank, int world, const void* id256);
void set_problem_host(regot_ctx* ctx, int64_t n, int64_t m, int64_t row_begin, int64_t row_count, const double* M,
                      int layout, int64_t ld, const double* a, const double* b, double eta);
void set_problem_device(regot_ctx* ctx, int64_t n, int64_t m, int64_t row_begin, int64_t row_count,
                        const double* M_dev, int64_t ld, const double* a_dev, const double* b_dev, double eta);
void validate_problem_device(regot_ctx* ctx);
void set_pointcloud(regot_ctx* ctx, int64_t n, int64_t m, int64_t row_begin, int64_t row_count, int d, const double* X,
                    const double* Y, const double* a, const double* b, double eta, bool on_the_fly);
void get_cost_host(regot_ctx* ctx, double* out);
thread_local std::string g_create_error;  // last create()/unique_id() failure of the calling thread
}  // namespace rg

using namespace rg;

extern "C" {

const char* regot_b200_version(void) { return "regot_b200 0.1.0 sm_100a"; }

const char* regot_b200_status_name(regot_status s)
{
    switch (s) {
    case REGOT_OK: return "OK";
    case REGOT_E_DEGENERATE_COST: return "DegenerateCostError";
    case REGOT_E_FORMAT: return "FormatError";
    case REGOT_E_TRUNCATION: return "TruncationError";
    case REGOT_E_VALIDATION: return "ValidationError";
    case REGOT_E_IO: return "IoError";
    case REGOT_E_ORACLE_SIZE: return "OracleSizeError";
    case REGOT_E_STRUCTURE: return "StructureError";
    case REGOT_E_NOT_POSITIVE_DEFINITE: return "NotPositiveDefiniteError";
    case REGOT_E_DIRECTION: return "DirectionError";
    case REGOT_E_LINE_SEARCH: return "LineSearchError";
    case REGOT_E_PLOT: return "PlotError";
    case REGOT_E_STEP: return "StepError";
    case REGOT_E_CUDA: return "CudaError";
    case REGOT_E_NCCL: return "NcclError";
    case REGOT_E_NOMEM: return "DeviceMemoryError";
    case REGOT_E_UNSUPPORTED: return "UnsupportedError";
    }
    return "UnknownError";
}

regot_status regot_b200_create(int device, regot_ctx** out)
{
    if (!out) return REGOT_E_VALIDATION;
    *out = nullptr;
    try {
        *out = ctx_create(device);
        return REGOT_OK;
    } catch (const Error& e) {
        g_create_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_create_error = e.what();
        return REGOT_E_CUDA;
    }
}

void regot_b200_destroy(regot_ctx* ctx) { ctx_destroy(ctx); }

const char* regot_b200_last_error(const regot_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_error.c_str(); }

int64_t regot_b200_launch_count(const regot_ctx* ctx) { return ctx ? ctx->launches : 0; }

regot_status regot_b200_set_pattern_reuse(regot_ctx* ctx, double drift_tol, int max_skips)
{
    return guard(ctx, [&] {
        if (!(drift_tol >= 0.0) || drift_tol >= 1.0 || max_skips < 0)
            rg::raise(REGOT_E_VALIDATION, "set_pattern_reuse: need 0 <= drift_tol < 1 and max_skips >= 0");
        ctx->pattern_drift = drift_tol;
        ctx->pattern_max_skips = max_skips;
    });
}

void regot_b200_pattern_counts(const regot_ctx* ctx, int64_t* rebuilds, int64_t* reuses)
{
    if (rebuilds) *rebuilds = ctx ? ctx->pattern_rebuilds : 0;
    if (reuses) *reuses = ctx ? ctx->pattern_reuses : 0;
}

regot_status regot_b200_set_profiling(regot_ctx* ctx, int enabled)
{
    return guard(ctx, [&] {
        RG_CUDA(cudaDeviceSynchronize());
        for (auto& e : ctx->prof_events) {
            cudaEventDestroy(e.a);
            cudaEventDestroy(e.b);
        }
        ctx->prof_events.clear();
        ctx->profiling = enabled != 0;
    });
}

regot_status regot_b200_get_profile(regot_ctx* ctx, int kind, int64_t* launches, double* total_ms)
{
    return guard(ctx, [&] {
        RG_CUDA(cudaDeviceSynchronize());
        int64_t n = 0;
        double tot = 0.0;
        for (const auto& e : ctx->prof_events) {
            if (e.kind != kind) continue;
            float ms = 0.f;
            RG_CUDA(cudaEventElapsedTime(&ms, e.a, e.b));
            tot += ms;
            ++n;
        }
        if (launches) *launches = n;
        if (total_ms) *total_ms = tot;
    });
}

regot_status regot_b200_comm_unique_id(void* out256)
{
    try {
        nccl_unique_id(out256);
        nccl_unique_id(static_cast<char*>(out256) + 128);
        return REGOT_OK;
    } catch (const Error& e) {
        g_create_error = e.what();
        return e.code;
    }
}

regot_status regot_b200_comm_init(regot_ctx* ctx, int rank, int world, const void* ids256)
{
    return guard(ctx, [&] { comm_init(ctx, rank, world, ids256); });
}

regot_status regot_b200_set_problem(regot_ctx* ctx, int64_t n, int64_t m, const double* M, int layout, int64_t ld,
                                    const double* a, const double* b, double eta)
{
    return guard(ctx, [&] {
        if (ctx->sharded) raise(REGOT_E_VALIDATION, "set_problem: use set_problem_rows on a sharded context");
        set_problem_host(ctx, n, m, 0, n, M, layout, ld, a, b, eta);
    });
}

regot_status regot_b200_set_problem_rows(regot_ctx* ctx, int64_t n, int64_t m, int64_t row_begin, int64_t row_count,
                                         const double* M, int layout, int64_t ld, const double* a, const double* b,
                                         double eta)
{
    return guard(ctx, [&] {
        // row-major: M is the block's first row; column-major: M is the global matrix
        set_problem_host(ctx, n, m, row_begin, row_count, M, layout, ld, a, b, eta);
    });
}

regot_status regot_b200_set_problem_device(regot_ctx* ctx, int64_t n, int64_t m, int64_t row_begin,
                                           int64_t row_count, const double* M_device, int64_t ld,
                                           const double* a_device, const double* b_device, double eta)
{
    return guard(ctx, [&] { set_problem_device(ctx, n, m, row_begin, row_count, M_device, ld, a_device, b_device, eta); });
}

regot_status regot_b200_set_pointcloud(regot_ctx* ctx, int64_t n, int64_t m, int32_t d, const double* X, const double* Y,
                                       const double* a, const double* b, double eta, int32_t on_the_fly)
{
    return guard(ctx, [&] {
        if (ctx->sharded) raise(REGOT_E_VALIDATION, "set_pointcloud: use set_pointcloud_rows on a sharded context");
        set_pointcloud(ctx, n, m, 0, n, d, X, Y, a, b, eta, on_the_fly != 0);
    });
}

regot_status regot_b200_set_pointcloud_rows(regot_ctx* ctx, int64_t n, int64_t m, int64_t row_begin, int64_t row_count,
                                            int32_t d, const double* X, const double* Y, const double* a,
                                            const double* b, double eta, int32_t on_the_fly)
{
    return guard(ctx, [&] { set_pointcloud(ctx, n, m, row_begin, row_count, d, X, Y, a, b, eta, on_the_fly != 0); });
}

regot_status regot_b200_get_cost(regot_ctx* ctx, double* M_rowmajor)
{
    return guard(ctx, [&] {
        ctx_require_problem(ctx);
        if (!M_rowmajor) raise(REGOT_E_VALIDATION, "get_cost: null output");
        get_cost_host(ctx, M_rowmajor);
    });
}

regot_status regot_b200_validate_problem(regot_ctx* ctx)
{
    return guard(ctx, [&] {
        ctx_require_problem(ctx);
        validate_problem_device(ctx);
    });
}

regot_status regot_b200_set_eta(regot_ctx* ctx, double eta)
{
    return guard(ctx, [&] {
        ctx_require_problem(ctx);
        if (!(eta > 0.0) || !std::isfinite(eta)) raise(REGOT_E_VALIDATION, "problem: eta must be positive and finite");
        ctx->prob.eta = eta;
    });
}

regot_status regot_b200_fused_gradient(regot_ctx* ctx, const double* alpha, const double* beta,
                                       regot_gradient_info* info, double* grad, double* row_sums, double* col_sums)
{
    return guard(ctx, [&] {
        ctx_require_problem(ctx);
        const DeviceProblem& pr = ctx->prob;
        upload_dual(ctx, alpha, beta, ctx->api_x, true, "fused_gradient");
        GradOut& go = ctx->api_grad;
        launch_gradient(ctx, ctx->stream, ctx->ws_main, ctx->comm, ctx->api_x.a.p, ctx->api_x.b.p, nullptr, nullptr, go);
        sync_scalars(ctx, ctx->stream, ctx->ws_main, go);
        if (info) {
            info->f = go.sc.f;
            info->marginal_error = go.sc.marginal_error;
            info->duality_gap = go.sc.duality_gap;
            info->grad_norm2 = std::sqrt(go.sc.grad_sqnorm);
            info->total_mass = go.sc.total_mass;
        }
        // sharded contexts fill only their own row slice of the n-long outputs
        if (grad) {
            download(ctx, grad + pr.row_begin, go.g.a.p, (size_t)pr.nloc);
            download(ctx, grad + pr.n, go.g.b.p, (size_t)pr.m - 1);
        }
        if (row_sums) download(ctx, row_sums + pr.row_begin, go.sums.a.p, (size_t)pr.nloc);
        if (col_sums) download(ctx, col_sums, go.sums.b.p, (size_t)pr.m);
        RG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

regot_status regot_b200_plan(regot_ctx* ctx, const double* alpha, const double* beta, double* T, int layout)
{
    return guard(ctx, [&] {
        ctx_require_problem(ctx);
        const DeviceProblem& pr = ctx->prob;
        if (!T) raise(REGOT_E_VALIDATION, "plan: null output");
        upload_dual(ctx, alpha, beta, ctx->api_x, true, "plan");
        DevBuf<double> Td;
        Td.ensure((size_t)pr.nloc * (size_t)pr.m);
        launch_plan(ctx, ctx->stream, ctx->api_x.a.p, ctx->api_x.b.p, Td.p);
        std::vector<double> h((size_t)pr.nloc * (size_t)pr.m);
        download(ctx, h.data(), Td.p, h.size());
        RG_CUDA(cudaStreamSynchronize(ctx->stream));
        if (layout == REGOT_LAYOUT_ROWMAJOR) {
            std::memcpy(T + (size_t)pr.row_begin * pr.m, h.data(), sizeof(double) * h.size());
        } else {
            for (int64_t i = 0; i < pr.nloc; ++i)
                for (int64_t j = 0; j < pr.m; ++j)
                    T[(size_t)j * pr.n + pr.row_begin + i] = h[(size_t)i * pr.m + j];
        }
    });
}

regot_status regot_b200_time_kernel(regot_ctx* ctx, int which, const double* alpha, const double* beta, int iters,
                                    float* ms_out)
{
    return guard(ctx, [&] {
        ctx_require_problem(ctx);
        if (iters < 1 || !ms_out) raise(REGOT_E_VALIDATION, "time_kernel: bad arguments");
        upload_dual(ctx, alpha, beta, ctx->api_x, true, "time_kernel");
        RG_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int it = 0; it < iters; ++it) {
            RG_CUDA(cudaEventRecord(ctx->ev_a, ctx->stream));
            time_kernel_once(ctx, which);
            RG_CUDA(cudaEventRecord(ctx->ev_b, ctx->stream));
            RG_CUDA(cudaEventSynchronize(ctx->ev_b));
            RG_CUDA(cudaEventElapsedTime(&ms_out[it], ctx->ev_a, ctx->ev_b));
        }
    });
}

// ---- configuration structs ---------------------------------------------------------------------
void regot_b200_splr_config_default(regot_splr_config* c)
{
    // SplrConfig{} (splr.h:24-35)
    std::memset(c, 0, sizeof(*c));
    c->tau_max = 1.0;
    c->S = 10;
    c->J = 5;
    c->density = 0.01;
    c->c1 = 1e-4;
    c->c2 = 0.9;
    c->max_iter = 1000;
    c->tol = 1e-8;
    c->max_ls_trials = 30;
    c->record_every = 1;
    c->overlap = 0;
    c->tile_rows = 8;
    c->tile_cols = 32;
    c->cg_max_iter = 0;
    c->cg_rtol = 0.0;
}

void regot_b200_sinkhorn_config_default(regot_sinkhorn_config* c)
{
    // SinkhornConfig{} (sinkhorn.h:18-20)
    c->max_iter = 1000;
    c->record_every = 1;
    c->tol = 0.0;
}

regot_status regot_b200_splr_config_validate(const regot_splr_config* c)
{
    try {
        validate_splr_config(*c);
        return REGOT_OK;
    } catch (const Error& e) {
        g_create_error = e.what();
        return e.code;
    }
}

regot_status regot_b200_sinkhorn_config_validate(const regot_sinkhorn_config* c)
{
    try {
        validate_sinkhorn_config(*c);
        return REGOT_OK;
    } catch (const Error& e) {
        g_create_error = e.what();
        return e.code;
    }
}

void regot_b200_splr_config_hash(const regot_splr_config* c, char out17[17])
{
    const std::string h = splr_config_hash(*c);
    std::memcpy(out17, h.c_str(), 17);
}

void regot_b200_sinkhorn_config_hash(const regot_sinkhorn_config* c, char out17[17])
{
    const std::string h = sinkhorn_config_hash(*c);
    std::memcpy(out17, h.c_str(), 17);
}

void regot_b200_result_free(regot_result* r)
{
    if (!r) return;
    std::free(r->alpha);
    std::free(r->beta);
    std::free(r->trace);
    std::free(r->steps);
    r->alpha = r->beta = nullptr;
    r->trace = nullptr;
    r->steps = nullptr;
    r->n_trace = r->n_steps = 0;
}

void regot_b200_host_row_block(int64_t n, int rank, int world, int64_t* row_begin, int64_t* row_count)
{
    const int64_t r0 = n * rank / world, r1 = n * (rank + 1) / world;
    *row_begin = r0;
    *row_count = r1 - r0;
}

void regot_b200_host_pick_bucket(const uint64_t* hist, int nbins, int64_t need, int* bucket, int64_t* above)
{
    // largest bucket b with count(buckets >= b) >= need; above = count(buckets > b)
    int64_t acc = 0;
    int b = nbins - 1;
    for (; b >= 0; --b) {
        if (acc + (int64_t)hist[b] >= need) break;
        acc += (int64_t)hist[b];
    }
    *bucket = b;
    *above = b >= 0 ? acc : 0;
}

int64_t regot_b200_topk_budget(int64_t n, int64_t m, double density)
{
    // splr.h:336-340
    return (int64_t)std::ceil(density * ((double)n * (double)(m - 1)));
}

}  // extern "C"
