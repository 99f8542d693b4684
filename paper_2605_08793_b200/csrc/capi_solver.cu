// capi_solver.cu -- extern "C" boundary: Sinkhorn, sparsification, SPLR.
#include "capi_util.hpp"

using namespace rg;

#define RG_TODO(name) return guard(ctx, [&] { raise(REGOT_E_UNSUPPORTED, name ": not implemented yet"); })

extern "C" {
regot_status regot_b200_optimal_alpha(regot_ctx* ctx, const double*, const double*, double*) { RG_TODO("optimal_alpha"); }
regot_status regot_b200_optimal_beta(regot_ctx* ctx, const double*, double*) { RG_TODO("optimal_beta"); }
regot_status regot_b200_sinkhorn_step(regot_ctx* ctx, double*, double*) { RG_TODO("sinkhorn_step"); }
regot_status regot_b200_run_sinkhorn(regot_ctx* ctx, const double*, const double*, const regot_sinkhorn_config*, regot_result*) { RG_TODO("run_sinkhorn"); }
regot_status regot_b200_select_topk_dense(regot_ctx* ctx, int64_t, int64_t, const double*, int, int64_t, int32_t*, int64_t, int64_t*) { RG_TODO("select_topk"); }
regot_status regot_b200_assemble_topk(regot_ctx* ctx, const double*, const double*, int64_t, double, const double*, const double*, regot_sparse**) { RG_TODO("assemble_topk"); }
regot_status regot_b200_assemble(regot_ctx* ctx, const double*, const double*, const int32_t*, int64_t, double, const double*, const double*, regot_sparse**) { RG_TODO("assemble"); }
regot_status regot_b200_update_values(regot_ctx* ctx, regot_sparse*, const double*, const double*, double, const double*, const double*) { RG_TODO("update_values"); }
regot_status regot_b200_matvec(regot_ctx* ctx, const regot_sparse*, const double*, double*) { RG_TODO("matvec"); }
regot_status regot_b200_sparse_info(const regot_sparse*, int32_t*, int64_t*, int64_t*, uint64_t*) { return REGOT_E_UNSUPPORTED; }
regot_status regot_b200_sparse_export(regot_ctx* ctx, const regot_sparse*, int32_t*, int32_t*, double*, int32_t*) { RG_TODO("sparse_export"); }
void regot_b200_sparse_free(regot_sparse*) {}
regot_status regot_b200_compute_direction(regot_ctx* ctx, const regot_sparse*, const double*, const double*, const double*, double, double, double, int32_t, double*, int32_t*) { RG_TODO("compute_direction"); }
regot_status regot_b200_run_splr(regot_ctx* ctx, const double*, const double*, const regot_splr_config*, regot_result*) { RG_TODO("run_splr"); }
}
