// timing.cu -- single launches of the hot kernels for regot_b200_time_kernel.
#include "capi_util.hpp"

namespace rg {

void time_kernel_once(regot_ctx* ctx, int which)
{
    switch (which) {
    case 0:
        launch_gradient_sweep_only(ctx, ctx->stream, ctx->ws_main, ctx->api_x.a.p, ctx->api_x.b.p);
        break;
    case 1:
        launch_row_lse_sweep_only(ctx, ctx->stream, ctx->ws_main, ctx->api_x.b.p);
        break;
    case 2:
        launch_col_lse_sweep_only(ctx, ctx->stream, ctx->ws_main, ctx->api_x.a.p);
        break;
    default:
        raise(REGOT_E_VALIDATION, "time_kernel: unknown kernel id");
    }
}

}  // namespace rg
