// vecops.hpp -- BLAS-1 helpers on dual-space device vectors (vecops.cu).
#pragma once

#include "common.cuh"
#include "ctx.hpp"

namespace rg {

constexpr int kMaxDots = 8;

struct DotJob {
    int nloc, mfree, count;
    const double* xa[kMaxDots];
    const double* xb[kMaxDots];
    const double* ya[kMaxDots];
    const double* yb[kMaxDots];
    double* partials;
    double* out;
    unsigned int* ticket;
    double* mbox;  // nullable: host mailbox for the 2 kMaxDots results (single-rank runs)
    unsigned long long seq;
};

struct DotScratch {
    DevBuf<double> partials, out;
    DevBuf<unsigned int> ticket;
    double* h_out = nullptr;
    HostMailbox mbox;
    ~DotScratch()
    {
        if (h_out) cudaFreeHost(h_out);
    }
};

void vec_axpy(regot_ctx* ctx, cudaStream_t st, double gamma, const DVec& x, const DVec& d, DVec& out);
void vec_sub(regot_ctx* ctx, cudaStream_t st, const DVec& a, const DVec& b, DVec& out);
void vec_lincomb(regot_ctx* ctx, cudaStream_t st, double sa, const DVec& a, double sb, const DVec* b, double sc,
                 const DVec* c, DVec& out);
void vec_copy(regot_ctx* ctx, cudaStream_t st, const DVec& src, DVec& dst);
void vec_zero(regot_ctx* ctx, cudaStream_t st, DVec& v);
void vec_dots(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, DotScratch& ws, int count, const DVec* const* xs,
              const DVec* const* ys, double* out_host);

}  // namespace rg
