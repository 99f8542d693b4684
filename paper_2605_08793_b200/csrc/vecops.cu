// vecops.cu -- BLAS-1 helpers on dual-space vectors (alpha block row-sharded,
// beta block replicated): axpy, fused multi-dot with a deterministic two-stage
// reduction.  These replace the Eigen BLAS-1 calls of splr.h (dot, norm,
// squaredNorm, x0 + gamma * d).
#include "ctx.hpp"
#include "vecops.hpp"

#include <algorithm>

namespace rg {

// out = x + gamma * d with the reference's rounding (product rounded, then sum:
// splr.h:207 `x0 + gamma * d`); beta[m-1] stays 0 (DualPoint::from_free).
__global__ void k_axpy(int nloc, int m, double gamma, const double* __restrict__ xa, const double* __restrict__ xb,
                       const double* __restrict__ da, const double* __restrict__ db, double* __restrict__ oa,
                       double* __restrict__ ob)
{
    const int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += stride)
        oa[i] = __dadd_rn(xa[i], __dmul_rn(gamma, da[i]));
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += stride)
        ob[j] = (j == m - 1) ? 0.0 : __dadd_rn(xb[j], __dmul_rn(gamma, db[j]));
}

// out = a - b on free vectors (s- = x - x_prev, y- = g - g_prev; splr.h:95-96)
__global__ void k_sub(int nloc, int mfree, const double* __restrict__ aa, const double* __restrict__ ab,
                      const double* __restrict__ ba, const double* __restrict__ bb, double* __restrict__ oa,
                      double* __restrict__ ob)
{
    const int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += stride) oa[i] = aa[i] - ba[i];
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < mfree; j += stride) ob[j] = ab[j] - bb[j];
}

// y = sa * a + sb * b + sc * c on free vectors (any of b, c may be null)
__global__ void k_lincomb(int nloc, int mfree, double sa, const double* __restrict__ aa, const double* __restrict__ ab,
                          double sb, const double* __restrict__ ba, const double* __restrict__ bb, double sc,
                          const double* __restrict__ ca, const double* __restrict__ cb, double* __restrict__ oa,
                          double* __restrict__ ob)
{
    const int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += stride) {
        double v = sa * aa[i];
        if (ba) v += sb * ba[i];
        if (ca) v += sc * ca[i];
        oa[i] = v;
    }
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < mfree; j += stride) {
        double v = sa * ab[j];
        if (bb) v += sb * bb[j];
        if (cb) v += sc * cb[j];
        ob[j] = v;
    }
}

// Up to kMaxDots dot products in one launch.  Output layout: out[k] = alpha
// part (partial over this rank's rows), out[kMaxDots + k] = beta part (replicated).
__global__ void __launch_bounds__(256) k_multidot(const DotJob job)
{
    __shared__ double scratch[2 * kMaxDots * 8];
    double acc[2 * kMaxDots];
#pragma unroll
    for (int k = 0; k < 2 * kMaxDots; ++k) acc[k] = 0.0;
    const int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < job.nloc; i += stride) {
#pragma unroll
        for (int k = 0; k < kMaxDots; ++k)
            if (k < job.count) acc[k] += job.xa[k][i] * job.ya[k][i];
    }
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < job.mfree; j += stride) {
#pragma unroll
        for (int k = 0; k < kMaxDots; ++k)
            if (k < job.count) acc[kMaxDots + k] += job.xb[k][j] * job.yb[k][j];
    }
    block_sum<2 * kMaxDots>(acc, scratch);
    if (threadIdx.x == 0)
        for (int k = 0; k < 2 * kMaxDots; ++k) job.partials[(size_t)blockIdx.x * 2 * kMaxDots + k] = acc[k];
    // last block: ordered sum of the per-block partials
    __shared__ bool is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = (atomicAdd(job.ticket, 1u) == gridDim.x - 1);
    __syncthreads();
    if (is_last) {
        __threadfence();
        if (threadIdx.x < 32) {
            for (int k = 0; k < 2 * kMaxDots; ++k) {
                double s = 0.0;
                for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) s += job.partials[(size_t)b * 2 * kMaxDots + k];
                s = warp_sum(s);
                if (threadIdx.x == 0) job.out[k] = s;
            }
            if (threadIdx.x == 0) {
                *job.ticket = 0u;
                if (job.mbox) mailbox_post(job.mbox, job.out, 2 * kMaxDots, job.seq);
            }
        }
    }
}

static int vgrid(const regot_ctx* ctx, long work)
{
    return (int)std::max<long>(1, std::min<long>((work + 255) / 256, 2L * ctx->sm_count));
}

void vec_axpy(regot_ctx* ctx, cudaStream_t st, double gamma, const DVec& x, const DVec& d, DVec& out)
{
    const DeviceProblem& pr = ctx->prob;
    out.ensure(pr.nloc, pr.m);
    k_axpy<<<vgrid(ctx, std::max(pr.nloc, pr.m)), 256, 0, st>>>((int)pr.nloc, (int)pr.m, gamma, x.a.p, x.b.p, d.a.p, d.b.p,
                                                               out.a.p, out.b.p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
}

void vec_sub(regot_ctx* ctx, cudaStream_t st, const DVec& a, const DVec& b, DVec& out)
{
    const DeviceProblem& pr = ctx->prob;
    out.ensure(pr.nloc, pr.m);
    k_sub<<<vgrid(ctx, std::max(pr.nloc, pr.m)), 256, 0, st>>>((int)pr.nloc, (int)pr.m - 1, a.a.p, a.b.p, b.a.p, b.b.p,
                                                              out.a.p, out.b.p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
}

void vec_lincomb(regot_ctx* ctx, cudaStream_t st, double sa, const DVec& a, double sb, const DVec* b, double sc,
                 const DVec* c, DVec& out)
{
    const DeviceProblem& pr = ctx->prob;
    out.ensure(pr.nloc, pr.m);
    k_lincomb<<<vgrid(ctx, std::max(pr.nloc, pr.m)), 256, 0, st>>>(
        (int)pr.nloc, (int)pr.m - 1, sa, a.a.p, a.b.p, sb, b ? b->a.p : nullptr, b ? b->b.p : nullptr, sc,
        c ? c->a.p : nullptr, c ? c->b.p : nullptr, out.a.p, out.b.p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
}

void vec_copy(regot_ctx* ctx, cudaStream_t st, const DVec& src, DVec& dst)
{
    const DeviceProblem& pr = ctx->prob;
    dst.ensure(pr.nloc, pr.m);
    RG_CUDA(cudaMemcpyAsync(dst.a.p, src.a.p, sizeof(double) * (size_t)pr.nloc, cudaMemcpyDeviceToDevice, st));
    RG_CUDA(cudaMemcpyAsync(dst.b.p, src.b.p, sizeof(double) * (size_t)pr.m, cudaMemcpyDeviceToDevice, st));
}

void vec_zero(regot_ctx* ctx, cudaStream_t st, DVec& v)
{
    const DeviceProblem& pr = ctx->prob;
    v.ensure(pr.nloc, pr.m);
    RG_CUDA(cudaMemsetAsync(v.a.p, 0, sizeof(double) * (size_t)pr.nloc, st));
    RG_CUDA(cudaMemsetAsync(v.b.p, 0, sizeof(double) * (size_t)pr.m, st));
}

// Synchronous: returns the dots on the host.  The alpha parts are summed over
// ranks (allreduce) when the context is sharded; the beta parts are replicated.
void vec_dots(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, DotScratch& ws, int count, const DVec* const* xs, const DVec* const* ys,
              double* out_host)
{
    const DeviceProblem& pr = ctx->prob;
    if (count < 1 || count > kMaxDots) raise(REGOT_E_VALIDATION, "vec_dots: bad count");
    const int grid = vgrid(ctx, std::max(pr.nloc, pr.m));
    ws.partials.ensure((size_t)(2 * ctx->sm_count + 8) * 2 * kMaxDots);
    ws.out.ensure(2 * kMaxDots);
    if (!ws.ticket.p) {
        ws.ticket.ensure(1);
        RG_CUDA(cudaMemsetAsync(ws.ticket.p, 0, sizeof(unsigned int), st));
    }
    if (!ws.h_out) RG_CUDA(cudaMallocHost((void**)&ws.h_out, sizeof(double) * 2 * kMaxDots));
    DotJob job;
    job.nloc = (int)pr.nloc;
    job.mfree = (int)pr.m - 1;
    job.count = count;
    for (int k = 0; k < kMaxDots; ++k) {
        const int q = k < count ? k : 0;
        job.xa[k] = xs[q]->a.p;
        job.xb[k] = xs[q]->b.p;
        job.ya[k] = ys[q]->a.p;
        job.yb[k] = ys[q]->b.p;
    }
    job.partials = ws.partials.p;
    job.out = ws.out.p;
    job.ticket = ws.ticket.p;
    const bool post = !ctx->sharded;  // sharded: the alpha parts are summed over ranks first
    ws.mbox.ensure();
    job.mbox = post ? ws.mbox.data : nullptr;
    job.seq = post ? ws.mbox.next() : 0ULL;
    k_multidot<<<grid, 256, 0, st>>>(job);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
    if (post) {
        ws.mbox.wait(st);
        for (int k = 0; k < count; ++k) out_host[k] = ws.mbox.data[k] + ws.mbox.data[kMaxDots + k];
        return;
    }
    // alpha parts are partial sums over this rank's rows; beta parts are replicated
    allreduce_sum(ctx, comm, ws.out.p, (size_t)count, st);
    RG_CUDA(cudaMemcpyAsync(ws.h_out, ws.out.p, sizeof(double) * 2 * kMaxDots, cudaMemcpyDeviceToHost, st));
    RG_CUDA(cudaStreamSynchronize(st));
    for (int k = 0; k < count; ++k) out_host[k] = ws.h_out[k] + ws.h_out[kMaxDots + k];
}

}  // namespace rg
