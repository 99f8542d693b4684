// k4_sparse.cu -- K3 value refresh, K4 sparse mat-vec, K5 Jacobi-PCG.
//
// K3 replaces fill_transport_values / update_values (sparsity.h:202-220,
// 305-317): values at the frozen pattern from the costs gathered at compaction
// time (no random reads of M).  K4 replaces SparseSym::matvec
// (sparsity.h:112-125).  K5 replaces the sparse Cholesky solve
// (sparse_chol.h:330-427) with preconditioned conjugate gradients on the SPD
// matrix A = H_Omega + tau I, up to 3 right-hand sides at once (the three solves
// of the Woodbury direction, splr.h:134-140, share every pass over A).
#include "common.cuh"
#include "ctx.hpp"
#include "sparse.hpp"

#include <algorithm>
#include <cmath>

namespace rg {

// ---- K3 -----------------------------------------------------------------------------------
__global__ void k_fill_values(int nnz, int nloc, int mm1, double eta, double tau, const int* __restrict__ row,
                              const int* __restrict__ col, const int* __restrict__ slot,
                              const double* __restrict__ mval, const double* __restrict__ alpha,
                              const double* __restrict__ beta, const double* __restrict__ row_sums,
                              const double* __restrict__ col_sums, const double* __restrict__ exp_table,
                              double* __restrict__ val, double* __restrict__ cscval, double* __restrict__ dA,
                              double* __restrict__ dB)
{
    const double inv_eta = 1.0 / eta;
    const int stride = gridDim.x * blockDim.x;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nnz; t += stride) {
        // plan_entry(...) / eta (sparsity.h:216): same T arithmetic as K1, true division by eta
        const double tt = ((alpha[row[t]] + beta[col[t]]) - mval[t]) * inv_eta;
        const double v = __ddiv_rn(exp_tbl_g(clamp700(tt), exp_table), eta);
        val[t] = v;
        cscval[slot[t]] = v;
    }
    // diagonal: full row / column sums over eta plus tau (sparsity.h:208-212)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += stride)
        dA[i] = __dadd_rn(__ddiv_rn(row_sums[i], eta), tau);
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < mm1; j += stride)
        dB[j] = __dadd_rn(__ddiv_rn(col_sums[j], eta), tau);
}

void sparse_fill_values(regot_ctx* ctx, cudaStream_t st, regot_sparse& S, const double* alpha, const double* beta,
                        double tau, const double* row_sums, const double* col_sums)
{
    if (tau < 0.0) raise(REGOT_E_VALIDATION, "assemble: tau must be >= 0");
    S.tau = tau;
    const long work = std::max<long>(S.nnz, std::max<long>(S.nloc, S.m));
    const int grid = (int)std::max<long>(1, std::min<long>((work + 255) / 256, 8L * ctx->sm_count));
    k_fill_values<<<grid, 256, 0, st>>>((int)S.nnz, (int)S.nloc, (int)S.m - 1, ctx->prob.eta, tau, S.row.p, S.col.p,
                                        S.slot.p, S.mval.p, alpha, beta, row_sums, col_sums, ctx->exp_table.p, S.val.p,
                                        S.cscval.p, S.dA.p, S.dB.p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
}

// ---- K4 -----------------------------------------------------------------------------------
constexpr int kMaxRhs = 3;
constexpr int kSpmvThreads = 256;
constexpr int kLongLen = 1024;  // must match finish_structure

struct SpmvParams {
    int nloc, mm1, nrhs;
    const int* rowptr;
    const int* col;
    const double* val;
    const int* cscptr;
    const int* cscrow;
    const double* cscval;
    const double* dA;
    const double* dB;
    const int* long_rows;
    const int* long_cols;
    int n_long_rows, n_long_cols;
    int warp_blocks;  // blocks doing the warp-per-line part
    int add_diag_b;   // sharded runs: only rank 0 adds diag(dB) v_beta before the allreduce
    const double* va;
    const double* vb;
    double* ya;
    double* yb;
    long sa, sb;  // strides between right-hand sides
};

// one matrix line (row of B or column of B) against nrhs vectors, strided by `step` lanes
template <int kStep>
__device__ __forceinline__ void line_dot(int beg, int end, int lane, const int* __restrict__ idx,
                                         const double* __restrict__ v, const double* __restrict__ x, long sx, int nrhs,
                                         double (&acc)[kMaxRhs])
{
    for (int t = beg + lane; t < end; t += kStep) {
        const int c = idx[t];
        const double a = v[t];
#pragma unroll
        for (int k = 0; k < kMaxRhs; ++k)
            if (k < nrhs) acc[k] += a * x[(size_t)k * sx + c];
    }
}

__global__ void __launch_bounds__(kSpmvThreads) k_spmv(const SpmvParams p)
{
    __shared__ double scratch[kMaxRhs * (kSpmvThreads / 32)];
    const int lane = threadIdx.x & 31;
    if ((int)blockIdx.x < p.warp_blocks) {
        const int wpb = kSpmvThreads / 32;
        const int nlines = p.nloc + p.mm1;
        for (int line = blockIdx.x * wpb + (threadIdx.x >> 5); line < nlines; line += p.warp_blocks * wpb) {
            double acc[kMaxRhs] = {0.0, 0.0, 0.0};
            if (line < p.nloc) {
                const int beg = p.rowptr[line], end = p.rowptr[line + 1];
                if (end - beg > kLongLen) continue;  // done by a whole CTA below
                line_dot<32>(beg, end, lane, p.col, p.val, p.vb, p.sb, p.nrhs, acc);
#pragma unroll
                for (int k = 0; k < kMaxRhs; ++k) {
                    if (k < p.nrhs) {
                        const double s = warp_sum(acc[k]);
                        if (lane == 0) p.ya[(size_t)k * p.sa + line] = p.dA[line] * p.va[(size_t)k * p.sa + line] + s;
                    }
                }
            } else {
                const int j = line - p.nloc;
                const int beg = p.cscptr[j], end = p.cscptr[j + 1];
                if (end - beg > kLongLen) continue;
                line_dot<32>(beg, end, lane, p.cscrow, p.cscval, p.va, p.sa, p.nrhs, acc);
#pragma unroll
                for (int k = 0; k < kMaxRhs; ++k) {
                    if (k < p.nrhs) {
                        const double s = warp_sum(acc[k]);
                        if (lane == 0)
                            p.yb[(size_t)k * p.sb + j] = (p.add_diag_b ? p.dB[j] * p.vb[(size_t)k * p.sb + j] : 0.0) + s;
                    }
                }
            }
        }
        return;
    }
    // long lines: one CTA each (row 0 and column 0 of Omega* are always here at scale)
    const int li = blockIdx.x - p.warp_blocks;
    double acc[kMaxRhs] = {0.0, 0.0, 0.0};
    if (li < p.n_long_rows) {
        const int i = p.long_rows[li];
        line_dot<kSpmvThreads>(p.rowptr[i], p.rowptr[i + 1], threadIdx.x, p.col, p.val, p.vb, p.sb, p.nrhs, acc);
        block_sum<kMaxRhs>(acc, scratch);
        if (threadIdx.x == 0)
            for (int k = 0; k < p.nrhs; ++k)
                p.ya[(size_t)k * p.sa + i] = p.dA[i] * p.va[(size_t)k * p.sa + i] + acc[k];
    } else {
        const int j = p.long_cols[li - p.n_long_rows];
        line_dot<kSpmvThreads>(p.cscptr[j], p.cscptr[j + 1], threadIdx.x, p.cscrow, p.cscval, p.va, p.sa, p.nrhs, acc);
        block_sum<kMaxRhs>(acc, scratch);
        if (threadIdx.x == 0)
            for (int k = 0; k < p.nrhs; ++k)
                p.yb[(size_t)k * p.sb + j] = (p.add_diag_b ? p.dB[j] * p.vb[(size_t)k * p.sb + j] : 0.0) + acc[k];
    }
}

void sparse_matvec(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, const regot_sparse& S, int nrhs, const double* va,
                   const double* vb, double* ya, double* yb, int64_t stride_a, int64_t stride_b)
{
    if (nrhs < 1 || nrhs > kMaxRhs) raise(REGOT_E_VALIDATION, "matvec: bad number of right-hand sides");
    SpmvParams p;
    p.nloc = (int)S.nloc;
    p.mm1 = (int)S.m - 1;
    p.nrhs = nrhs;
    p.rowptr = S.rowptr.p;
    p.col = S.col.p;
    p.val = S.val.p;
    p.cscptr = S.cscptr.p;
    p.cscrow = S.cscrow.p;
    p.cscval = S.cscval.p;
    p.dA = S.dA.p;
    p.dB = S.dB.p;
    p.long_rows = S.long_rows.p;
    p.long_cols = S.long_cols.p;
    p.n_long_rows = S.n_long_rows;
    p.n_long_cols = S.n_long_cols;
    const long lines = (long)p.nloc + p.mm1;
    p.warp_blocks = (int)std::max<long>(1, std::min<long>((lines + 7) / 8, 8L * ctx->sm_count));
    p.add_diag_b = (ctx->world == 1 || ctx->rank == 0) ? 1 : 0;
    p.va = va;
    p.vb = vb;
    p.ya = ya;
    p.yb = yb;
    p.sa = stride_a;
    p.sb = stride_b;
    k_spmv<<<p.warp_blocks + p.n_long_rows + p.n_long_cols, kSpmvThreads, 0, st>>>(p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
    // column results are partial sums over the row blocks
    if (ctx->world > 1) {
        for (int k = 0; k < nrhs; ++k) allreduce_sum(ctx, comm, yb + (size_t)k * stride_b, (size_t)p.mm1, st);
    }
}

// ---- K5: batched Jacobi-PCG -----------------------------------------------------------------
// scalars (device): per rhs k
//   rz[2][k] (double-buffered by iteration parity), pAp[k], rz0[k], done[k], flag
constexpr int kScalRz = 0;               // 2 * kMaxRhs
constexpr int kScalPap = 2 * kMaxRhs;    // kMaxRhs
constexpr int kScalRz0 = 3 * kMaxRhs;    // kMaxRhs
constexpr int kScalDone = 4 * kMaxRhs;   // kMaxRhs (0/1)
constexpr int kScalBreak = 5 * kMaxRhs;  // 1: breakdown flag
constexpr int kScalIters = 5 * kMaxRhs + 1;  // kMaxRhs: iterations taken by each system
constexpr int kScalCount = 6 * kMaxRhs + 4;
constexpr int kCgThreads = 256;

struct CgVecs {
    int nloc, mfree, nrhs;
    long sa, sb;
    double *xa, *xb, *ra, *rb, *pa, *pb, *qa, *qb;  // x, r, p, q = A p
    const double *dA, *dB;
    double* scal;
    double* partials;
    unsigned int* ticket;
    int beta_owner;  // this rank counts the replicated beta block in dot products
};

template <int NV>
__device__ __forceinline__ void two_stage_store(double (&acc)[NV], double* scratch, double* partials,
                                                unsigned int* ticket, double* out)
{
    block_sum<NV>(acc, scratch);
    if (threadIdx.x == 0)
        for (int k = 0; k < NV; ++k) partials[(size_t)blockIdx.x * NV + k] = acc[k];
    __shared__ bool is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
    __syncthreads();
    if (is_last) {
        __threadfence();
        if (threadIdx.x < 32) {
            for (int k = 0; k < NV; ++k) {
                double s = 0.0;
                for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) s += partials[(size_t)b * NV + k];
                s = warp_sum(s);
                if (threadIdx.x == 0) out[k] = s;
            }
            if (threadIdx.x == 0) *ticket = 0u;
        }
    }
}

// r = rhs, x = 0, p = z = D^{-1} r, rz[0] = r.z
__global__ void __launch_bounds__(kCgThreads) k_cg_init(const CgVecs v, const double* const* rhs_a,
                                                        const double* const* rhs_b)
{
    __shared__ double scratch[kMaxRhs * (kCgThreads / 32)];
    double acc[kMaxRhs] = {0.0, 0.0, 0.0};
    const int stride = gridDim.x * blockDim.x;
    for (int k = 0; k < v.nrhs; ++k) {
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < v.nloc; i += stride) {
            const double r = rhs_a[k][i], z = r / v.dA[i];
            v.xa[k * v.sa + i] = 0.0;
            v.ra[k * v.sa + i] = r;
            v.pa[k * v.sa + i] = z;
            acc[k] += r * z;
        }
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < v.mfree; j += stride) {
            const double r = rhs_b[k][j], z = r / v.dB[j];
            v.xb[k * v.sb + j] = 0.0;
            v.rb[k * v.sb + j] = r;
            v.pb[k * v.sb + j] = z;
            if (v.beta_owner) acc[k] += r * z;
        }
    }
    two_stage_store<kMaxRhs>(acc, scratch, v.partials, v.ticket, v.scal + kScalRz);
}

// pAp[k] = p_k . q_k
__global__ void __launch_bounds__(kCgThreads) k_cg_pap(const CgVecs v)
{
    __shared__ double scratch[kMaxRhs * (kCgThreads / 32)];
    double acc[kMaxRhs] = {0.0, 0.0, 0.0};
    const int stride = gridDim.x * blockDim.x;
    for (int k = 0; k < v.nrhs; ++k) {
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < v.nloc; i += stride)
            acc[k] += v.pa[k * v.sa + i] * v.qa[k * v.sa + i];
        if (v.beta_owner)
            for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < v.mfree; j += stride)
                acc[k] += v.pb[k * v.sb + j] * v.qb[k * v.sb + j];
    }
    two_stage_store<kMaxRhs>(acc, scratch, v.partials, v.ticket, v.scal + kScalPap);
}

// x += a p, r -= a q, rz_new = r . D^{-1} r ; a = rz / pAp (0 once the system is done)
__global__ void __launch_bounds__(kCgThreads) k_cg_update(const CgVecs v, int parity)
{
    __shared__ double scratch[kMaxRhs * (kCgThreads / 32)];
    double acc[kMaxRhs] = {0.0, 0.0, 0.0};
    const int stride = gridDim.x * blockDim.x;
    for (int k = 0; k < v.nrhs; ++k) {
        const double pap = v.scal[kScalPap + k];
        const bool live = v.scal[kScalDone + k] == 0.0 && pap > 0.0;
        const double a = live ? v.scal[kScalRz + parity * kMaxRhs + k] / pap : 0.0;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < v.nloc; i += stride) {
            v.xa[k * v.sa + i] += a * v.pa[k * v.sa + i];
            const double r = v.ra[k * v.sa + i] - a * v.qa[k * v.sa + i];
            v.ra[k * v.sa + i] = r;
            acc[k] += r * (r / v.dA[i]);
        }
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < v.mfree; j += stride) {
            v.xb[k * v.sb + j] += a * v.pb[k * v.sb + j];
            const double r = v.rb[k * v.sb + j] - a * v.qb[k * v.sb + j];
            v.rb[k * v.sb + j] = r;
            if (v.beta_owner) acc[k] += r * (r / v.dB[j]);
        }
    }
    two_stage_store<kMaxRhs>(acc, scratch, v.partials, v.ticket, v.scal + kScalRz + (parity ^ 1) * kMaxRhs);
}

// p = z + b p with b = rz_new / rz; block 0 also updates the done / breakdown flags
__global__ void __launch_bounds__(kCgThreads) k_cg_direction(const CgVecs v, int parity, double tol2)
{
    const int stride = gridDim.x * blockDim.x;
    for (int k = 0; k < v.nrhs; ++k) {
        const double rz = v.scal[kScalRz + parity * kMaxRhs + k];
        const double rzn = v.scal[kScalRz + (parity ^ 1) * kMaxRhs + k];
        const bool done = v.scal[kScalDone + k] != 0.0;
        const double b = (!done && rz > 0.0) ? rzn / rz : 0.0;
        if (!done) {
            for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < v.nloc; i += stride)
                v.pa[k * v.sa + i] = v.ra[k * v.sa + i] / v.dA[i] + b * v.pa[k * v.sa + i];
            for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < v.mfree; j += stride)
                v.pb[k * v.sb + j] = v.rb[k * v.sb + j] / v.dB[j] + b * v.pb[k * v.sb + j];
        }
    }
}

// single thread: bookkeeping between iterations (runs after k_cg_direction)
__global__ void k_cg_flags(double* scal, int nrhs, int parity, double tol2, int first)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int k = 0; k < nrhs; ++k) {
        if (first) {
            const double rz0 = scal[kScalRz + k];
            scal[kScalRz0 + k] = rz0;
            scal[kScalDone + k] = (rz0 == 0.0) ? 1.0 : 0.0;
            continue;
        }
        if (scal[kScalDone + k] != 0.0) {
            // keep the buffered rz equal so a finished system stays finished
            scal[kScalRz + (parity ^ 1) * kMaxRhs + k] = scal[kScalRz + parity * kMaxRhs + k];
            continue;
        }
        const double pap = scal[kScalPap + k];
        if (!(pap > 0.0)) scal[kScalBreak] = 1.0;  // not positive definite (or NaN)
        scal[kScalIters + k] += 1.0;
        const double rzn = scal[kScalRz + (parity ^ 1) * kMaxRhs + k];
        if (rzn <= tol2 * scal[kScalRz0 + k]) scal[kScalDone + k] = 1.0;
    }
}

int sparse_pcg(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, SparseWS& ws, const regot_sparse& S, int nrhs,
               const DVec* const* rhs, DVec* const* sol, double rtol, int max_iter)
{
    if (nrhs < 1 || nrhs > kMaxRhs) raise(REGOT_E_VALIDATION, "pcg: bad number of right-hand sides");
    const int nloc = (int)S.nloc, mfree = (int)S.m - 1;
    const long sa = nloc, sb = std::max(mfree, 1);
    // layout of ws.cg: x | r | p | q, each nrhs * (sa + sb)
    const size_t per = (size_t)kMaxRhs * (size_t)(sa + sb);
    ws.cg.ensure(4 * per + 16);
    ws.cg_scal.ensure(kScalCount + 2 * kMaxRhs);
    ws.cg_partials.ensure((size_t)(2 * ctx->sm_count + 8) * kMaxRhs);
    if (!ws.cg_ticket.p) {
        ws.cg_ticket.ensure(1);
        RG_CUDA(cudaMemsetAsync(ws.cg_ticket.p, 0, sizeof(unsigned int), st));
    }
    if (!ws.h_cg) RG_CUDA(cudaMallocHost((void**)&ws.h_cg, sizeof(double) * (kScalCount + 8 + 4 * kMaxRhs)));
    RG_CUDA(cudaMemsetAsync(ws.cg_scal.p, 0, sizeof(double) * (kScalCount + 2 * kMaxRhs), st));

    CgVecs v;
    v.nloc = nloc;
    v.mfree = mfree;
    v.nrhs = nrhs;
    v.sa = sa;
    v.sb = sb;
    double* base = ws.cg.p;
    v.xa = base;
    v.xb = base + (size_t)kMaxRhs * sa;
    v.ra = base + per;
    v.rb = v.ra + (size_t)kMaxRhs * sa;
    v.pa = base + 2 * per;
    v.pb = v.pa + (size_t)kMaxRhs * sa;
    v.qa = base + 3 * per;
    v.qb = v.qa + (size_t)kMaxRhs * sa;
    v.dA = S.dA.p;
    v.dB = S.dB.p;
    v.scal = ws.cg_scal.p;
    v.partials = ws.cg_partials.p;
    v.ticket = ws.cg_ticket.p;
    v.beta_owner = (ctx->world == 1 || ctx->rank == 0) ? 1 : 0;

    // right-hand-side pointer tables live behind the scalars on the device
    const double* h_ptrs[2 * kMaxRhs];
    for (int k = 0; k < kMaxRhs; ++k) {
        h_ptrs[k] = rhs[k < nrhs ? k : 0]->a.p;
        h_ptrs[kMaxRhs + k] = rhs[k < nrhs ? k : 0]->b.p;
    }
    const double** d_ptrs = reinterpret_cast<const double**>(ws.cg_scal.p + kScalCount);
    RG_CUDA(cudaMemcpyAsync((void*)d_ptrs, h_ptrs, sizeof(h_ptrs), cudaMemcpyHostToDevice, st));

    const long work = std::max<long>(nloc, mfree);
    const int grid = (int)std::max<long>(1, std::min<long>((work + kCgThreads - 1) / kCgThreads, 2L * ctx->sm_count));
    const double tol2 = rtol * rtol;
    auto reduce_scal = [&](int off) {  // sharded: sum the partial dot products over ranks
        if (ctx->world > 1) allreduce_sum(ctx, comm, ws.cg_scal.p + off, kMaxRhs, st);
    };

    k_cg_init<<<grid, kCgThreads, 0, st>>>(v, d_ptrs, d_ptrs + kMaxRhs);
    RG_CUDA(cudaGetLastError());
    reduce_scal(kScalRz);
    k_cg_flags<<<1, 32, 0, st>>>(ws.cg_scal.p, nrhs, 0, tol2, 1);
    RG_CUDA(cudaGetLastError());
    ctx->launches += 2;

    const int check_every = 8;
    int it = 0, parity = 0;
    bool finished = false, broke = false;
    while (it < max_iter && !finished) {
        const int burst = std::min(check_every, max_iter - it);
        for (int b = 0; b < burst; ++b, ++it) {
            sparse_matvec(ctx, st, comm, S, nrhs, v.pa, v.pb, v.qa, v.qb, sa, sb);
            k_cg_pap<<<grid, kCgThreads, 0, st>>>(v);
            reduce_scal(kScalPap);
            k_cg_update<<<grid, kCgThreads, 0, st>>>(v, parity);
            reduce_scal(kScalRz + (parity ^ 1) * kMaxRhs);
            k_cg_flags<<<1, 32, 0, st>>>(ws.cg_scal.p, nrhs, parity, tol2, 0);
            k_cg_direction<<<grid, kCgThreads, 0, st>>>(v, parity, tol2);
            RG_CUDA(cudaGetLastError());
            ctx->launches += 4;
            parity ^= 1;
        }
        RG_CUDA(cudaMemcpyAsync(ws.h_cg, ws.cg_scal.p, sizeof(double) * kScalCount, cudaMemcpyDeviceToHost, st));
        RG_CUDA(cudaStreamSynchronize(st));
        broke = ws.h_cg[kScalBreak] != 0.0;
        finished = true;
        for (int k = 0; k < nrhs; ++k) finished &= ws.h_cg[kScalDone + k] != 0.0;
        if (broke) break;
    }
    if (broke) return -1;
    it = 0;  // report the slowest system's exact count, not the burst-rounded loop count
    for (int k = 0; k < nrhs; ++k) it = std::max(it, (int)ws.h_cg[kScalIters + k]);
    for (int k = 0; k < nrhs; ++k) {
        sol[k]->ensure(S.nloc, S.m);
        RG_CUDA(cudaMemcpyAsync(sol[k]->a.p, v.xa + (size_t)k * sa, sizeof(double) * (size_t)nloc, cudaMemcpyDeviceToDevice, st));
        RG_CUDA(cudaMemcpyAsync(sol[k]->b.p, v.xb + (size_t)k * sb, sizeof(double) * (size_t)mfree, cudaMemcpyDeviceToDevice, st));
        RG_CUDA(cudaMemsetAsync(sol[k]->b.p + mfree, 0, sizeof(double), st));
    }
    return it;
}

}  // namespace rg
