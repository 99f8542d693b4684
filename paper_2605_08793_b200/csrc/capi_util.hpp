// capi_util.hpp -- helpers shared by the extern "C" translation units.
#pragma once

#include "ctx.hpp"

#include <cmath>
#include <new>
#include <sstream>

namespace rg {

extern thread_local std::string g_create_error;

// Run `body`, translate exceptions into a status + ctx->err.
template <class F>
regot_status guard(regot_ctx* ctx, F&& body)
{
    if (!ctx) return REGOT_E_VALIDATION;
    try {
        RG_CUDA(cudaSetDevice(ctx->device));
        body();
        ctx->err.clear();
        return REGOT_OK;
    } catch (const Error& e) {
        ctx->err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        ctx->err = "host allocation failed";
        return REGOT_E_NOMEM;
    } catch (const std::exception& e) {
        ctx->err = e.what();
        return REGOT_E_CUDA;
    }
}

inline void download(regot_ctx* ctx, double* host, const double* dev, size_t count)
{
    if (count == 0) return;
    RG_CUDA(cudaMemcpyAsync(host, dev, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx->stream));
}

// splr.h:37-59
inline void validate_splr_config(const regot_splr_config& c)
{
    if (!(c.c1 > 0.0 && c.c1 < 0.5)) raise(REGOT_E_VALIDATION, "SplrConfig: need 0 < c1 < 1/2");
    if (!(c.c2 > c.c1 && c.c2 < 1.0)) raise(REGOT_E_VALIDATION, "SplrConfig: need c1 < c2 < 1");
    if (c.S < 1) raise(REGOT_E_VALIDATION, "SplrConfig: need S >= 1");
    if (c.J < 0) raise(REGOT_E_VALIDATION, "SplrConfig: need J >= 0");
    if (!(c.tau_max > 0.0)) raise(REGOT_E_VALIDATION, "SplrConfig: need tau_max > 0");
    if (!(c.density > 0.0 && c.density <= 1.0)) raise(REGOT_E_VALIDATION, "SplrConfig: need 0 < density <= 1");
    if (c.max_iter < 1) raise(REGOT_E_VALIDATION, "SplrConfig: need max_iter >= 1");
    if (c.tol < 0.0) raise(REGOT_E_VALIDATION, "SplrConfig: need tol >= 0");
    if (c.max_ls_trials < 1) raise(REGOT_E_VALIDATION, "SplrConfig: need max_ls_trials >= 1");
    if (c.record_every < 1) raise(REGOT_E_VALIDATION, "SplrConfig: need record_every >= 1");
}

// sinkhorn.h:22-30
inline void validate_sinkhorn_config(const regot_sinkhorn_config& c)
{
    if (c.max_iter < 1) raise(REGOT_E_VALIDATION, "SinkhornConfig: max_iter must be >= 1");
    if (c.record_every < 1) raise(REGOT_E_VALIDATION, "SinkhornConfig: record_every must be >= 1");
    if (c.tol < 0.0) raise(REGOT_E_VALIDATION, "SinkhornConfig: tol must be >= 0");
}

inline std::string fnv_hex(const std::string& s)
{
    // core.h:42-66
    std::uint64_t h = 0xcbf29ce484222325ULL;
    for (unsigned char ch : s) {
        h ^= ch;
        h *= 0x100000001b3ULL;
    }
    static const char* dig = "0123456789abcdef";
    std::string out(16, '0');
    for (int i = 15; i >= 0; --i, h >>= 4) out[(size_t)i] = dig[h & 0xf];
    return out;
}

// splr.h:62-70: canonical string streamed with default ostream formatting
inline std::string splr_config_hash(const regot_splr_config& c)
{
    std::ostringstream os;
    os << "tau_max=" << c.tau_max << ";S=" << (long)c.S << ";J=" << (long)c.J << ";density=" << c.density
       << ";c1=" << c.c1 << ";c2=" << c.c2 << ";tile=" << c.tile_rows << "x" << c.tile_cols;
    return fnv_hex(os.str());
}

// sinkhorn.h:33-39
inline std::string sinkhorn_config_hash(const regot_sinkhorn_config& c)
{
    std::ostringstream os;
    os << "max_iter=" << (long)c.max_iter << ";tol=" << c.tol;
    return fnv_hex(os.str());
}

// one launch of hot kernel `which` at ctx->api_x (k1_gradient.cu / k7_lse.cu)
void time_kernel_once(regot_ctx* ctx, int which);

}  // namespace rg
