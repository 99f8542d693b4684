// capi_solver.cu -- extern "C" boundary: Sinkhorn, sparsification, SPLR.
#include "capi_util.hpp"
#include "solver.hpp"

#include <cstring>
#include <memory>

namespace rg {
regot_ctx* ctx_create(int device);
void ctx_destroy(regot_ctx* ctx);
void set_problem_host(regot_ctx* ctx, int64_t n, int64_t m, int64_t row_begin, int64_t row_count, const double* M,
                      int layout, int64_t ld, const double* a, const double* b, double eta);
}  // namespace rg

using namespace rg;

namespace {

void fill_result(regot_ctx* ctx, const SolveOut& so, const char* algo, const std::string& hash, regot_result* out)
{
    std::memset(out, 0, sizeof(*out));
    out->status = so.status;
    out->n = ctx->prob.n;
    out->m = ctx->prob.m;
    out->eta = ctx->prob.eta;
    std::snprintf(out->algo, sizeof(out->algo), "%s", algo);
    std::snprintf(out->config_hash, sizeof(out->config_hash), "%s", hash.c_str());
    std::snprintf(out->message, sizeof(out->message), "%s", so.message.c_str());
    out->n_trace = (int64_t)so.trace.size();
    out->trace = (regot_trace_row*)std::malloc(sizeof(regot_trace_row) * std::max<size_t>(1, so.trace.size()));
    std::memcpy(out->trace, so.trace.data(), sizeof(regot_trace_row) * so.trace.size());
    if (!so.steps.empty()) {
        out->n_steps = (int64_t)so.steps.size();
        out->steps = (regot_step_record*)std::malloc(sizeof(regot_step_record) * so.steps.size());
        std::memcpy(out->steps, so.steps.data(), sizeof(regot_step_record) * so.steps.size());
    }
    if (so.status == REGOT_OK) {
        out->alpha = (double*)std::malloc(sizeof(double) * std::max<size_t>(1, so.alpha.size()));
        out->beta = (double*)std::malloc(sizeof(double) * std::max<size_t>(1, so.beta.size()));
        std::memcpy(out->alpha, so.alpha.data(), sizeof(double) * so.alpha.size());
        std::memcpy(out->beta, so.beta.data(), sizeof(double) * so.beta.size());
    }
    out->device_ms = so.device_ms;
    out->gradient_passes = so.gradient_passes;
    out->lse_passes = so.lse_passes;
    out->kernel_launches = so.kernel_launches;
}

// gradient sums (row_sums global n, col_sums m) from the host into a DVec
void upload_sums(regot_ctx* ctx, const double* row_sums, const double* col_sums, DVec& s)
{
    const DeviceProblem& pr = ctx->prob;
    if (!row_sums || !col_sums) raise(REGOT_E_VALIDATION, "assemble: null gradient sums");
    s.ensure(pr.nloc, pr.m);
    RG_CUDA(cudaMemcpyAsync(s.a.p, row_sums + pr.row_begin, sizeof(double) * (size_t)pr.nloc, cudaMemcpyHostToDevice, ctx->stream));
    RG_CUDA(cudaMemcpyAsync(s.b.p, col_sums, sizeof(double) * (size_t)pr.m, cudaMemcpyHostToDevice, ctx->stream));
}

void upload_free(regot_ctx* ctx, const double* v, DVec& out, const char* who)
{
    const DeviceProblem& pr = ctx->prob;
    if (!v) raise(REGOT_E_VALIDATION, std::string(who) + ": null vector");
    out.ensure(pr.nloc, pr.m);
    RG_CUDA(cudaMemcpyAsync(out.a.p, v + pr.row_begin, sizeof(double) * (size_t)pr.nloc, cudaMemcpyHostToDevice, ctx->stream));
    RG_CUDA(cudaMemcpyAsync(out.b.p, v + pr.n, sizeof(double) * (size_t)(pr.m - 1), cudaMemcpyHostToDevice, ctx->stream));
    RG_CUDA(cudaMemsetAsync(out.b.p + (pr.m - 1), 0, sizeof(double), ctx->stream));
}

void download_free(regot_ctx* ctx, const DVec& v, double* out)
{
    const DeviceProblem& pr = ctx->prob;
    download(ctx, out + pr.row_begin, v.a.p, (size_t)pr.nloc);
    download(ctx, out + pr.n, v.b.p, (size_t)pr.m - 1);
    RG_CUDA(cudaStreamSynchronize(ctx->stream));
}

void check_sparse(const regot_ctx* ctx, const regot_sparse* A, const char* who)
{
    if (!A) raise(REGOT_E_VALIDATION, std::string(who) + ": null matrix");
    // update_values (sparsity.h:308-313): the matrix must come from this problem shape
    if (A->n != ctx->prob.n || A->m != ctx->prob.m || A->nloc != ctx->prob.nloc)
        raise(REGOT_E_VALIDATION, std::string(who) + ": problem shape mismatch");
}

// host copy of the structure in the reference's CSC layout (sparsity.h:249-289)
struct HostCsc {
    std::vector<int> colptr, rowidx, coords;
    std::vector<double> values;
    uint64_t pattern_id = 0;
};

HostCsc export_csc(regot_ctx* ctx, const regot_sparse& S, bool with_values)
{
    if (ctx->sharded) raise(REGOT_E_UNSUPPORTED, "sparse export: only on an unsharded context");
    const int n = (int)S.nloc, mm1 = (int)S.m - 1, nnz = (int)S.nnz, dim = n + mm1;
    std::vector<int> rowptr((size_t)n + 1), col((size_t)nnz), cscptr((size_t)mm1 + 1), cscrow((size_t)nnz);
    std::vector<double> val((size_t)nnz), cscval((size_t)nnz), dA((size_t)n), dB((size_t)std::max(mm1, 0));
    auto get = [&](void* dst, const void* src, size_t bytes) {
        if (bytes) RG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    };
    get(rowptr.data(), S.rowptr.p, sizeof(int) * rowptr.size());
    get(col.data(), S.col.p, sizeof(int) * col.size());
    get(cscptr.data(), S.cscptr.p, sizeof(int) * cscptr.size());
    get(cscrow.data(), S.cscrow.p, sizeof(int) * cscrow.size());
    if (with_values) {
        get(val.data(), S.val.p, sizeof(double) * val.size());
        get(cscval.data(), S.cscval.p, sizeof(double) * cscval.size());
        get(dA.data(), S.dA.p, sizeof(double) * dA.size());
        get(dB.data(), S.dB.p, sizeof(double) * dB.size());
    }
    RG_CUDA(cudaStreamSynchronize(ctx->stream));
    HostCsc H;
    H.colptr.assign((size_t)dim + 1, 0);
    H.rowidx.reserve((size_t)dim + 2 * (size_t)nnz);
    H.values.reserve((size_t)dim + 2 * (size_t)nnz);
    H.coords.reserve(2 * (size_t)nnz);
    for (int i = 0; i < n; ++i) {  // alpha column i: diagonal, then rows n + j ascending
        H.rowidx.push_back(i);
        H.values.push_back(with_values ? dA[(size_t)i] : 0.0);
        for (int t = rowptr[(size_t)i]; t < rowptr[(size_t)i + 1]; ++t) {
            H.rowidx.push_back(n + col[(size_t)t]);
            H.values.push_back(with_values ? val[(size_t)t] : 0.0);
            H.coords.push_back(i);
            H.coords.push_back(col[(size_t)t]);
        }
        H.colptr[(size_t)i + 1] = (int)H.rowidx.size();
    }
    for (int j = 0; j < mm1; ++j) {  // beta column n + j: rows i ascending, diagonal last
        for (int q = cscptr[(size_t)j]; q < cscptr[(size_t)j + 1]; ++q) {
            H.rowidx.push_back(cscrow[(size_t)q]);
            H.values.push_back(with_values ? cscval[(size_t)q] : 0.0);
        }
        H.rowidx.push_back(n + j);
        H.values.push_back(with_values ? dB[(size_t)j] : 0.0);
        H.colptr[(size_t)n + j + 1] = (int)H.rowidx.size();
    }
    // compute_pattern_id (sparsity.h:160-166): FNV-1a over dim, colptr, rowidx
    auto fnv = [](const void* data, size_t len, uint64_t h) {
        const unsigned char* p = static_cast<const unsigned char*>(data);
        for (size_t i = 0; i < len; ++i) {
            h ^= p[i];
            h *= 0x100000001b3ULL;
        }
        return h;
    };
    uint64_t h = fnv(&dim, sizeof(dim), 0xcbf29ce484222325ULL);
    h = fnv(H.colptr.data(), H.colptr.size() * sizeof(int), h);
    if (!H.rowidx.empty()) h = fnv(H.rowidx.data(), H.rowidx.size() * sizeof(int), h);
    H.pattern_id = h;
    return H;
}

}  // namespace

extern "C" {

regot_status regot_b200_optimal_alpha(regot_ctx* ctx, const double* alpha, const double* beta, double* alpha_out)
{
    return guard(ctx, [&] {
        ctx_require_problem(ctx);
        const DeviceProblem& pr = ctx->prob;
        if (!alpha_out) raise(REGOT_E_VALIDATION, "optimal_alpha: null output");
        upload_dual(ctx, alpha, beta, ctx->api_x, true, "optimal_alpha");
        ctx->api_y.ensure(pr.nloc, pr.m);
        launch_optimal_alpha(ctx, ctx->stream, ctx->ws_main, ctx->api_x.b.p, ctx->api_y.a.p);
        download(ctx, alpha_out + pr.row_begin, ctx->api_y.a.p, (size_t)pr.nloc);
        RG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

regot_status regot_b200_optimal_beta(regot_ctx* ctx, const double* alpha, double* beta_out)
{
    return guard(ctx, [&] {
        ctx_require_problem(ctx);
        const DeviceProblem& pr = ctx->prob;
        if (!alpha || !beta_out) raise(REGOT_E_VALIDATION, "optimal_beta: alpha length mismatch");
        ctx->api_x.ensure(pr.nloc, pr.m);
        RG_CUDA(cudaMemcpyAsync(ctx->api_x.a.p, alpha + pr.row_begin, sizeof(double) * (size_t)pr.nloc,
                                cudaMemcpyHostToDevice, ctx->stream));
        launch_optimal_beta(ctx, ctx->stream, ctx->ws_main, ctx->comm, ctx->api_x.a.p, ctx->api_x.b.p, 0);
        download(ctx, beta_out, ctx->api_x.b.p, (size_t)pr.m);
        RG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

regot_status regot_b200_sinkhorn_step(regot_ctx* ctx, double* alpha_io, double* beta_io)
{
    return guard(ctx, [&] {
        ctx_require_problem(ctx);
        const DeviceProblem& pr = ctx->prob;
        upload_dual(ctx, alpha_io, beta_io, ctx->api_x, true, "optimal_alpha");
        launch_sinkhorn_step(ctx, ctx->stream, ctx->ws_main, ctx->comm, ctx->api_x.a.p, ctx->api_x.b.p);
        download(ctx, alpha_io + pr.row_begin, ctx->api_x.a.p, (size_t)pr.nloc);
        download(ctx, beta_io, ctx->api_x.b.p, (size_t)pr.m);
        RG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

regot_status regot_b200_run_sinkhorn(regot_ctx* ctx, const double* alpha0, const double* beta0,
                                     const regot_sinkhorn_config* cfg, regot_result* out)
{
    if (out) std::memset(out, 0, sizeof(*out));
    return guard(ctx, [&] {
        if (!cfg || !out) raise(REGOT_E_VALIDATION, "run_sinkhorn: null argument");
        SolveOut so;
        solve_sinkhorn(ctx, alpha0, beta0, *cfg, so);
        fill_result(ctx, so, "sinkhorn", sinkhorn_config_hash(*cfg), out);
    });
}

regot_status regot_b200_run_splr(regot_ctx* ctx, const double* alpha0, const double* beta0, const regot_splr_config* cfg,
                                 regot_result* out)
{
    if (out) std::memset(out, 0, sizeof(*out));
    regot_status step = REGOT_OK;
    const regot_status st = guard(ctx, [&] {
        if (!cfg || !out) raise(REGOT_E_VALIDATION, "run_splr: null argument");
        SolveOut so;
        solve_splr(ctx, alpha0, beta0, *cfg, so);
        fill_result(ctx, so, "splr", splr_config_hash(*cfg), out);
        if (so.status != REGOT_OK) {
            step = so.status;
            ctx->err = so.message;
        }
    });
    if (st == REGOT_OK && step != REGOT_OK) {
        ctx->err = out->message;
        return step;
    }
    return st;
}

}  // extern "C"

// SplrState (splr.h:82-97): the device state plus the context it belongs to
struct regot_splr_state {
    regot_ctx* ctx = nullptr;
    int device = 0;
    int64_t n = 0, m = 0, nloc = 0;
    SplrStateDev dev;
};

namespace {
void check_state(const regot_ctx* ctx, const regot_splr_state* s, const char* who)
{
    if (!s) raise(REGOT_E_VALIDATION, std::string(who) + ": null state");
    if (s->ctx != ctx || s->n != ctx->prob.n || s->m != ctx->prob.m || s->nloc != ctx->prob.nloc)
        raise(REGOT_E_VALIDATION, std::string(who) + ": dual point/problem dimension mismatch");
}
}  // namespace

extern "C" {

regot_status regot_b200_splr_init(regot_ctx* ctx, const double* alpha0, const double* beta0, const regot_splr_config* cfg,
                                  regot_splr_state** out)
{
    return guard(ctx, [&] {
        if (!cfg || !out) raise(REGOT_E_VALIDATION, "splr_init: null argument");
        *out = nullptr;
        ctx_require_problem(ctx);
        auto s = std::make_unique<regot_splr_state>();
        s->ctx = ctx;
        s->device = ctx->device;
        s->n = ctx->prob.n;
        s->m = ctx->prob.m;
        s->nloc = ctx->prob.nloc;
        splr_init_state(ctx, alpha0, beta0, s->dev, nullptr);
        *out = s.release();
    });
}

regot_status regot_b200_splr_step(regot_ctx* ctx, regot_splr_state* state, const regot_splr_config* cfg,
                                  regot_step_record* rec)
{
    return guard(ctx, [&] {
        if (!cfg) raise(REGOT_E_VALIDATION, "splr_step: null argument");
        validate_splr_config(*cfg);
        ctx_require_problem(ctx);
        check_state(ctx, state, "splr_step");
        regot_step_record r;
        splr_step_state(ctx, state->dev, *cfg, r, nullptr);
        if (rec) *rec = r;
    });
}

regot_status regot_b200_splr_state_info(regot_ctx* ctx, const regot_splr_state* state, int64_t* iter, int32_t* has_prev,
                                        regot_gradient_info* cur)
{
    return guard(ctx, [&] {
        check_state(ctx, state, "splr_state_info");
        if (iter) *iter = state->dev.iter;
        if (has_prev) *has_prev = state->dev.has_prev ? 1 : 0;
        if (cur) {
            const GradScalars& sc = state->dev.cur.sc;
            cur->f = sc.f;
            cur->marginal_error = sc.marginal_error;
            cur->duality_gap = sc.duality_gap;
            cur->grad_norm2 = std::sqrt(sc.grad_sqnorm);
            cur->total_mass = sc.total_mass;
        }
    });
}

regot_status regot_b200_splr_state_point(regot_ctx* ctx, const regot_splr_state* state, double* alpha, double* beta,
                                         double* grad, double* row_sums, double* col_sums)
{
    return guard(ctx, [&] {
        check_state(ctx, state, "splr_state_point");
        const DeviceProblem& pr = ctx->prob;
        const SplrStateDev& S = state->dev;
        if (alpha || beta) {
            std::vector<double> a, b;
            download_point(ctx, S.x, a, b);
            if (alpha) std::memcpy(alpha, a.data(), sizeof(double) * a.size());
            if (beta) std::memcpy(beta, b.data(), sizeof(double) * b.size());
        }
        // like fused_gradient: a sharded context fills its own row slice of the n-long outputs
        if (grad) {
            download(ctx, grad + pr.row_begin, S.cur.g.a.p, (size_t)pr.nloc);
            download(ctx, grad + pr.n, S.cur.g.b.p, (size_t)pr.m - 1);
        }
        if (row_sums) download(ctx, row_sums + pr.row_begin, S.cur.sums.a.p, (size_t)pr.nloc);
        if (col_sums) download(ctx, col_sums, S.cur.sums.b.p, (size_t)pr.m);
        RG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

const regot_sparse* regot_b200_splr_state_matrix(const regot_splr_state* state)
{
    return (state && state->dev.A.ctx) ? &state->dev.A : nullptr;
}

void regot_b200_splr_state_free(regot_splr_state* state)
{
    if (!state) return;
    cudaSetDevice(state->device);
    delete state;
}

regot_status regot_b200_select_topk_dense(regot_ctx* ctx, int64_t n, int64_t m, const double* T, int layout, int64_t k,
                                          int32_t* coords, int64_t cap, int64_t* count)
{
    return guard(ctx, [&] {
        if (k < 0) raise(REGOT_E_VALIDATION, "select_topk: k must be >= 0");
        if (!T || !count || n < 1 || m < 1) raise(REGOT_E_VALIDATION, "select_topk: bad arguments");
        if (m - 1 <= 0) {  // sparsity.h:55-56
            *count = 0;
            return;
        }
        // the dense plan becomes the "cost matrix" of a scratch context so the
        // selection sweeps run unchanged (kFromDenseT)
        std::unique_ptr<regot_ctx, void (*)(regot_ctx*)> tmp(ctx_create(ctx->device), ctx_destroy);
        std::vector<double> a((size_t)n, 1.0 / (double)n), b((size_t)m, 1.0 / (double)m);
        set_problem_host(tmp.get(), n, m, 0, n, T, layout, layout == REGOT_LAYOUT_COLMAJOR ? n : m, a.data(), b.data(), 1.0);
        regot_sparse S;
        SparseWS ws;
        topk_build_pattern(tmp.get(), tmp->stream, ws, kFromDenseT, nullptr, nullptr, k, S);
        ctx->launches += tmp->launches;
        *count = S.nnz;
        if (coords && cap > 0) {
            const int64_t take = std::min<int64_t>(cap, S.nnz);
            std::vector<int> row((size_t)take), col((size_t)take);
            RG_CUDA(cudaMemcpy(row.data(), S.row.p, sizeof(int) * (size_t)take, cudaMemcpyDeviceToHost));
            RG_CUDA(cudaMemcpy(col.data(), S.col.p, sizeof(int) * (size_t)take, cudaMemcpyDeviceToHost));
            for (int64_t t = 0; t < take; ++t) {
                coords[2 * t] = row[(size_t)t];
                coords[2 * t + 1] = col[(size_t)t];
            }
        }
    });
}

regot_status regot_b200_assemble_topk(regot_ctx* ctx, const double* alpha, const double* beta, int64_t k, double tau,
                                      const double* row_sums, const double* col_sums, regot_sparse** out)
{
    return guard(ctx, [&] {
        ctx_require_problem(ctx);
        if (!out) raise(REGOT_E_VALIDATION, "assemble: null output");
        if (tau < 0.0) raise(REGOT_E_VALIDATION, "assemble: tau must be >= 0");
        upload_dual(ctx, alpha, beta, ctx->api_x, true, "assemble");
        upload_sums(ctx, row_sums, col_sums, ctx->api_y);
        auto S = std::make_unique<regot_sparse>();
        topk_build_pattern(ctx, ctx->stream, solver_ws(ctx).sparse, kFromDual, ctx->api_x.a.p, ctx->api_x.b.p, k, *S);
        sparse_fill_values(ctx, ctx->stream, *S, ctx->api_x.a.p, ctx->api_x.b.p, tau, ctx->api_y.a.p, ctx->api_y.b.p);
        RG_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = S.release();
    });
}

regot_status regot_b200_assemble(regot_ctx* ctx, const double* alpha, const double* beta, const int32_t* coords,
                                 int64_t ncoords, double tau, const double* row_sums, const double* col_sums,
                                 regot_sparse** out)
{
    return guard(ctx, [&] {
        ctx_require_problem(ctx);
        if (!out || (!coords && ncoords > 0)) raise(REGOT_E_VALIDATION, "assemble: null argument");
        if (tau < 0.0) raise(REGOT_E_VALIDATION, "assemble: tau must be >= 0");
        upload_dual(ctx, alpha, beta, ctx->api_x, true, "assemble");
        upload_sums(ctx, row_sums, col_sums, ctx->api_y);
        auto S = std::make_unique<regot_sparse>();
        pattern_from_coords(ctx, ctx->stream, solver_ws(ctx).sparse, coords, ncoords, *S);
        sparse_fill_values(ctx, ctx->stream, *S, ctx->api_x.a.p, ctx->api_x.b.p, tau, ctx->api_y.a.p, ctx->api_y.b.p);
        RG_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = S.release();
    });
}

regot_status regot_b200_update_values(regot_ctx* ctx, regot_sparse* A, const double* alpha, const double* beta, double tau,
                                      const double* row_sums, const double* col_sums)
{
    return guard(ctx, [&] {
        ctx_require_problem(ctx);
        if (!A) raise(REGOT_E_VALIDATION, "update_values: matrix was not assembled from a problem");
        check_sparse(ctx, A, "update_values");
        if (tau < 0.0) raise(REGOT_E_VALIDATION, "update_values: tau must be >= 0");
        upload_dual(ctx, alpha, beta, ctx->api_x, true, "update_values");
        upload_sums(ctx, row_sums, col_sums, ctx->api_y);
        sparse_fill_values(ctx, ctx->stream, *A, ctx->api_x.a.p, ctx->api_x.b.p, tau, ctx->api_y.a.p, ctx->api_y.b.p);
        RG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

regot_status regot_b200_matvec(regot_ctx* ctx, const regot_sparse* A, const double* v, double* y)
{
    return guard(ctx, [&] {
        ctx_require_problem(ctx);
        check_sparse(ctx, A, "SparseSym::matvec");
        if (!y) raise(REGOT_E_VALIDATION, "SparseSym::matvec: length mismatch");
        upload_free(ctx, v, ctx->api_x, "SparseSym::matvec");
        ctx->api_y.ensure(ctx->prob.nloc, ctx->prob.m);
        sparse_matvec(ctx, ctx->stream, ctx->comm, *A, 1, ctx->api_x.a.p, ctx->api_x.b.p, ctx->api_y.a.p, ctx->api_y.b.p, 0, 0);
        download_free(ctx, ctx->api_y, y);
    });
}

regot_status regot_b200_sparse_info(const regot_sparse* A, int32_t* dim, int64_t* nnz, int64_t* ncoords,
                                    uint64_t* pattern_id)
{
    if (!A || !A->ctx) return REGOT_E_VALIDATION;
    regot_ctx* ctx = A->ctx;
    return guard(ctx, [&] {
        if (dim) *dim = (int32_t)(A->n + A->m - 1);
        if (ncoords) *ncoords = A->nnz;
        if (nnz) *nnz = (A->n + A->m - 1) + 2 * A->nnz;
        // the id hashes the GLOBAL structure (sparsity.h:160-166): a row-sharded context holds only its rows -> 0
        if (pattern_id) *pattern_id = !ctx->sharded ? export_csc(ctx, *A, false).pattern_id : 0;
    });
}

regot_status regot_b200_sparse_export(regot_ctx* ctx, const regot_sparse* A, int32_t* colptr, int32_t* rowidx,
                                      double* values, int32_t* coords)
{
    return guard(ctx, [&] {
        if (!A) raise(REGOT_E_VALIDATION, "sparse_export: null matrix");
        const HostCsc H = export_csc(ctx, *A, true);
        if (colptr) std::memcpy(colptr, H.colptr.data(), sizeof(int) * H.colptr.size());
        if (rowidx) std::memcpy(rowidx, H.rowidx.data(), sizeof(int) * H.rowidx.size());
        if (values) std::memcpy(values, H.values.data(), sizeof(double) * H.values.size());
        if (coords) std::memcpy(coords, H.coords.data(), sizeof(int) * H.coords.size());
    });
}

regot_status regot_b200_sparse_export_local(regot_ctx* ctx, const regot_sparse* A, int32_t* coords, double* values,
                                            int64_t cap, int64_t* count)
{
    return guard(ctx, [&] {
        if (!A || !count) raise(REGOT_E_VALIDATION, "sparse_export_local: null argument");
        *count = A->nnz;
        const size_t take = (size_t)std::max<int64_t>(0, std::min<int64_t>(cap, A->nnz));
        if (take == 0) return;
        std::vector<int> row(take), col(take);
        RG_CUDA(cudaMemcpyAsync(row.data(), A->row.p, sizeof(int) * take, cudaMemcpyDeviceToHost, ctx->stream));
        RG_CUDA(cudaMemcpyAsync(col.data(), A->col.p, sizeof(int) * take, cudaMemcpyDeviceToHost, ctx->stream));
        if (values) RG_CUDA(cudaMemcpyAsync(values, A->val.p, sizeof(double) * take, cudaMemcpyDeviceToHost, ctx->stream));
        RG_CUDA(cudaStreamSynchronize(ctx->stream));
        if (coords)
            for (size_t t = 0; t < take; ++t) {
                coords[2 * t] = (int32_t)(row[t] + A->row_begin);
                coords[2 * t + 1] = col[t];
            }
    });
}

void regot_b200_sparse_free(regot_sparse* A)
{
    if (!A) return;
    cudaSetDevice(A->device);  // not A->ctx->device: the context may already have been destroyed
    delete A;
}

regot_status regot_b200_compute_direction(regot_ctx* ctx, const regot_sparse* A, const double* g, const double* u,
                                          const double* v, double xi, double zeta, double cg_rtol, int32_t cg_max_iter,
                                          double* d, int32_t* cg_iters)
{
    return guard(ctx, [&] {
        ctx_require_problem(ctx);
        check_sparse(ctx, A, "compute_direction");
        if (!d) raise(REGOT_E_VALIDATION, "compute_direction: null output");
        SolverWS& W = solver_ws(ctx);
        const DeviceProblem& pr = ctx->prob;
        upload_free(ctx, g, ctx->api_x, "compute_direction");
        const bool active = u && v;
        if (active) {
            upload_free(ctx, u, ctx->api_y, "compute_direction");
            upload_free(ctx, v, ctx->api_d, "compute_direction");
        }
        // same body as solver.cu's compute_direction, through the public pieces
        const DVec* gx[1] = {&ctx->api_x};
        double gg = 0.0;
        vec_dots(ctx, ctx->stream, ctx->comm, W.dots, 1, gx, gx, &gg);
        int its = 0;
        const double rtol = cg_rtol > 0.0 ? cg_rtol : kDefaultCgRtol;
        const long dim = (long)pr.n + pr.m - 1;
        const int maxit = cg_max_iter > 0 ? cg_max_iter : (int)std::min<long>(20 * dim, 200000);
        if (!compute_direction_api(ctx, *A, ctx->api_x, gg, active, xi, zeta, ctx->api_y, ctx->api_d, rtol, maxit, W.d, its))
            raise(REGOT_E_NOT_POSITIVE_DEFINITE, "pcg: matrix is not positive definite");
        if (cg_iters) *cg_iters = its;
        download_free(ctx, W.d, d);
    });
}

}  // extern "C"
