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

#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

namespace rg {

// ---- K3 -----------------------------------------------------------------------------------
__global__ void k_fill_values(int nnz, int nloc, int mm1, double eta, const ExpScale E, double tau, const int* __restrict__ row,
                              const int* __restrict__ col, const int* __restrict__ slot,
                              const double* __restrict__ mval, const double* __restrict__ alpha,
                              const double* __restrict__ beta, const double* __restrict__ row_sums,
                              const double* __restrict__ col_sums, const double* __restrict__ exp_table,
                              double* __restrict__ val, double* __restrict__ cscval, double* __restrict__ dA,
                              double* __restrict__ dB)
{
    const int stride = gridDim.x * blockDim.x;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nnz; t += stride) {
        // plan_entry(...) / eta (sparsity.h:216): same T arithmetic as K1, true division by eta
        const double v = __ddiv_rn(plan_entry_dev_g((alpha[row[t]] + beta[col[t]]) - mval[t], E, exp_table), eta);
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
    k_fill_values<<<grid, 256, 0, st>>>((int)S.nnz, (int)S.nloc, (int)S.m - 1, ctx->prob.eta, make_exp_scale(ctx->prob.eta), tau, S.row.p, S.col.p,
                                        S.slot.p, S.mval.p, alpha, beta, row_sums, col_sums, ctx->exp_table.p, S.val.p,
                                        S.cscval.p, S.dA.p, S.dB.p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
}

// ---- K4 -----------------------------------------------------------------------------------
constexpr int kMaxRhs = 3;
constexpr int kSpmvThreads = 256;

// matrix view shared by the stand-alone mat-vec and the persistent PCG kernel
struct SpmvMat {
    int nloc, mm1;
    const int* rowptr;
    const int* col;
    const double* val;
    const int* cscptr;
    const int* cscrow;
    const double* cscval;
    const double* dA;
    const double* dB;
    const int* chunks;     // {line, beg, end, slot} per chunk of a long line
    const int* longlines;  // {first chunk, count} per long line
    int n_chunks;
    const int* lines_s;  // lines with <= kShortLine entries
    const int* lines_m;  // lines with <= kLongLine entries
    int n_lines_s, n_lines_m;
    double* chunk_part;       // n_chunks x kMaxRhs
    unsigned int* chunk_cnt;  // arrivals per long line
    int add_diag_b;           // sharded runs: only rank 0 adds diag(dB) v_beta before the allreduce
    int dbg;                  // experiments: 1 skip chunks, 2 skip medium lines, 4 skip short lines
};

// part of one matrix line (row of B or column of B) against nrhs vectors: kLanes lanes stride
// over [beg, end) with kUnroll independent index/value loads and gathers in flight per lane
// (the mat-vec is latency-bound, not bandwidth-bound: everything lives in L2)
template <int kLanes, int kUnroll>
__device__ __forceinline__ void line_dot(int beg, int end, int gl, const int* __restrict__ idx,
                                         const double* __restrict__ v, const double* x, long sx, int nrhs,
                                         double (&acc)[kMaxRhs])
{
    for (int t = beg + gl; t < end; t += kLanes * kUnroll) {
        int c[kUnroll];
        double a[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int tt = t + kLanes * u;
            const bool ok = tt < end;
            c[u] = ok ? __ldg(idx + tt) : 0;
            a[u] = ok ? __ldg(v + tt) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
#pragma unroll
            for (int k = 0; k < kMaxRhs; ++k)
                if (k < nrhs) acc[k] += a[u] * x[(size_t)k * sx + c[u]];
        }
    }
}

// epilogue of one finished line: y = diag * v_line + s, optional v . y accumulation
template <bool kDot>
__device__ __forceinline__ void line_store(const SpmvMat& A, int line, int k, double s, double diag, double vi,
                                           long sa, long sb, double* ya, double* yb, double& pq)
{
    const double y = diag * vi + s;
    if (line < A.nloc) ya[(size_t)k * sa + line] = y;
    else yb[(size_t)k * sb + (line - A.nloc)] = y;
    if (kDot) pq += vi * y;
}

// line pointers, diagonal entry and the line's own vector entries; issued before the gather
// loop so their latency overlaps it
__device__ __forceinline__ void line_head(const SpmvMat& A, int line, int nrhs, const double* va,
                                          const double* vb, long sa, long sb, int& beg, int& end,
                                          double& diag, double (&vi)[kMaxRhs])
{
    if (line < A.nloc) {
        beg = __ldg(A.rowptr + line);
        end = __ldg(A.rowptr + line + 1);
        diag = __ldg(A.dA + line);
#pragma unroll
        for (int k = 0; k < kMaxRhs; ++k)
            if (k < nrhs) vi[k] = va[(size_t)k * sa + line];
    } else {
        const int j = line - A.nloc;
        beg = __ldg(A.cscptr + j);
        end = __ldg(A.cscptr + j + 1);
        diag = A.add_diag_b ? __ldg(A.dB + j) : 0.0;
#pragma unroll
        for (int k = 0; k < kMaxRhs; ++k)
            if (k < nrhs) vi[k] = vb[(size_t)k * sb + j];
    }
}

// y = A v for nrhs vectors.  Lines are binned by length (finish_structure): long lines are cut into
// chunks spread over warps and combined in chunk order by the last warp to arrive; medium lines
// get a warp; short lines get 8 lanes, four lines in flight per warp.  Longest work first.  With
// kDot, one lane per line also accumulates v . y into pq (the z'Az of conjugate gradients).  Every
// sum has a fixed order (lane-strided partials, butterfly, chunk order): bitwise reproducible for
// a fixed grid.
template <bool kDot>
__device__ __forceinline__ void spmv_warp(const SpmvMat& A, int nrhs, const double* va, const double* vb, long sa,
                                          long sb, double* ya, double* yb, int gw, int nw, int lane,
                                          double (&pq)[kMaxRhs], double* long_pq = nullptr)
{
    // ---- long lines: chunk partials ----
    for (int c = gw; c < ((A.dbg & 1) ? 0 : A.n_chunks); c += nw) {
        const int line = A.chunks[4 * c], beg = A.chunks[4 * c + 1], end = A.chunks[4 * c + 2], slot = A.chunks[4 * c + 3];
        const bool is_row = line < A.nloc;
        double acc[kMaxRhs] = {0.0, 0.0, 0.0};
        if (is_row) line_dot<32, 4>(beg, end, lane, A.col, A.val, vb, sb, nrhs, acc);
        else line_dot<32, 4>(beg, end, lane, A.cscrow, A.cscval, va, sa, nrhs, acc);
#pragma unroll
        for (int k = 0; k < kMaxRhs; ++k) {
            if (k < nrhs) {
                const double s = warp_sum(acc[k]);
                if (lane == 0) A.chunk_part[(size_t)c * kMaxRhs + k] = s;
            }
        }
        __threadfence();
        unsigned prev = 0;
        if (lane == 0) prev = atomicAdd(&A.chunk_cnt[slot], 1u);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        const int first = A.longlines[2 * slot], cnt = A.longlines[2 * slot + 1];
        if ((int)prev == cnt - 1) {  // last chunk of the line to finish: ordered sum of all partials
            __threadfence();
            int b2, e2;
            double diag, vi[kMaxRhs] = {0.0, 0.0, 0.0};
            line_head(A, line, nrhs, va, vb, sa, sb, b2, e2, diag, vi);
#pragma unroll
            for (int k = 0; k < kMaxRhs; ++k) {
                if (k < nrhs) {
                    double s = 0.0;
                    for (int q = lane; q < cnt; q += 32) s += __ldcg(A.chunk_part + (size_t)(first + q) * kMaxRhs + k);
                    s = warp_sum(s);
                    if (lane == 0) {
                        // which warp arrives last varies from run to run, so the line's v . y goes to a
                        // fixed slot of the ordered grid reduction instead of this warp's partial
                        double dotk = 0.0;
                        line_store<kDot>(A, line, k, s, diag, vi[k], sa, sb, ya, yb, dotk);
                        if (kDot) {
                            long_pq[(size_t)slot * 2 * kMaxRhs + k] = 0.0;
                            long_pq[(size_t)slot * 2 * kMaxRhs + kMaxRhs + k] = dotk;
                        }
                    }
                } else if (kDot && lane == 0) {
                    long_pq[(size_t)slot * 2 * kMaxRhs + k] = 0.0;
                    long_pq[(size_t)slot * 2 * kMaxRhs + kMaxRhs + k] = 0.0;
                }
            }
            if (lane == 0) A.chunk_cnt[slot] = 0u;
        }
    }
    // ---- medium lines: one warp each (handed out from the far end so chunk-laden warps get fewer) ----
    for (int q = nw - 1 - gw; q < ((A.dbg & 2) ? 0 : A.n_lines_m); q += nw) {
        const int line = A.lines_m[q];
        int beg, end;
        double diag, vi[kMaxRhs] = {0.0, 0.0, 0.0}, acc[kMaxRhs] = {0.0, 0.0, 0.0};
        line_head(A, line, nrhs, va, vb, sa, sb, beg, end, diag, vi);
        if (line < A.nloc) line_dot<32, 4>(beg, end, lane, A.col, A.val, vb, sb, nrhs, acc);
        else line_dot<32, 4>(beg, end, lane, A.cscrow, A.cscval, va, sa, nrhs, acc);
#pragma unroll
        for (int k = 0; k < kMaxRhs; ++k) {
            if (k < nrhs) {
                const double s = warp_sum(acc[k]);
                if (lane == 0) line_store<kDot>(A, line, k, s, diag, vi[k], sa, sb, ya, yb, pq[k]);
            }
        }
    }
    // ---- short lines: 8 lanes each, four lines in flight per warp ----
    const int sub = lane >> 3, gl = lane & 7;
    for (int base = gw * 4; base < ((A.dbg & 4) ? 0 : A.n_lines_s); base += nw * 4) {
        const bool valid = base + sub < A.n_lines_s;
        int line = 0, beg = 0, end = 0;
        double diag = 0.0, vi[kMaxRhs] = {0.0, 0.0, 0.0}, acc[kMaxRhs] = {0.0, 0.0, 0.0};
        if (valid) {
            line = A.lines_s[base + sub];
            line_head(A, line, nrhs, va, vb, sa, sb, beg, end, diag, vi);
            if (line < A.nloc) line_dot<8, 8>(beg, end, gl, A.col, A.val, vb, sb, nrhs, acc);
            else line_dot<8, 8>(beg, end, gl, A.cscrow, A.cscval, va, sa, nrhs, acc);
        }
#pragma unroll
        for (int k = 0; k < kMaxRhs; ++k) {
            if (k < nrhs) {
                double s = acc[k];
                s += shfl_xor_d(s, 4);
                s += shfl_xor_d(s, 2);
                s += shfl_xor_d(s, 1);
                if (valid && gl == 0) line_store<kDot>(A, line, k, s, diag, vi[k], sa, sb, ya, yb, pq[k]);
            }
        }
    }
}

struct SpmvParams {
    SpmvMat A;
    int nrhs;
    const double* va;
    const double* vb;
    double* ya;
    double* yb;
    long sa, sb;
};

__global__ void __launch_bounds__(kSpmvThreads, 4) k_spmv(const SpmvParams p)
{
    double pq[kMaxRhs] = {0.0, 0.0, 0.0};
    const int wpb = kSpmvThreads / 32;
    spmv_warp<false>(p.A, p.nrhs, p.va, p.vb, p.sa, p.sb, p.ya, p.yb, blockIdx.x * wpb + (threadIdx.x >> 5),
                     gridDim.x * wpb, threadIdx.x & 31, pq);
}

static SpmvMat mat_view(const regot_ctx* ctx, const regot_sparse& S)
{
    SpmvMat A;
    A.nloc = (int)S.nloc;
    A.mm1 = (int)S.m - 1;
    A.rowptr = S.rowptr.p;
    A.col = S.col.p;
    A.val = S.val.p;
    A.cscptr = S.cscptr.p;
    A.cscrow = S.cscrow.p;
    A.cscval = S.cscval.p;
    A.dA = S.dA.p;
    A.dB = S.dB.p;
    A.chunks = S.chunks.p;
    A.longlines = S.longlines.p;
    A.n_chunks = S.n_chunks;
    A.lines_s = S.lines_s.p;
    A.lines_m = S.lines_m.p;
    A.n_lines_s = S.n_lines_s;
    A.n_lines_m = S.n_lines_m;
    A.chunk_part = S.chunk_part.p;
    A.chunk_cnt = S.chunk_cnt.p;
    A.add_diag_b = (ctx->world == 1 || ctx->rank == 0) ? 1 : 0;
    A.dbg = 0;
    if (const char* e = std::getenv("REGOT_B200_SPMV_DBG")) A.dbg = std::atoi(e);
    return A;
}

void sparse_matvec(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, const regot_sparse& S, int nrhs, const double* va,
                   const double* vb, double* ya, double* yb, int64_t stride_a, int64_t stride_b)
{
    if (nrhs < 1 || nrhs > kMaxRhs) raise(REGOT_E_VALIDATION, "matvec: bad number of right-hand sides");
    SpmvParams p;
    p.A = mat_view(ctx, S);
    p.nrhs = nrhs;
    p.va = va;
    p.vb = vb;
    p.ya = ya;
    p.yb = yb;
    p.sa = stride_a;
    p.sb = stride_b;
    const long items = (long)p.A.n_chunks + p.A.n_lines_m + (p.A.n_lines_s + 3) / 4;
    const int grid = (int)std::max<long>(1, std::min<long>((items + 7) / 8, 8L * ctx->sm_count));
    ProfScope prof(ctx, st, 4);
    k_spmv<<<grid, kSpmvThreads, 0, st>>>(p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
    // column results are partial sums over the row blocks
    if (ctx->world > 1) {
        for (int k = 0; k < nrhs; ++k) allreduce_sum(ctx, comm, yb + (size_t)k * stride_b, (size_t)p.A.mm1, st);
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

// Multi-kernel PCG: the sharded path (NCCL collectives between the kernels).
static int pcg_multikernel(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, SparseWS& ws, const regot_sparse& S, int nrhs,
                           const DVec* const* rhs, DVec* const* sol, double rtol, int max_iter)
{
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
    if (!ws.h_cg) RG_CUDA(cudaMallocHost((void**)&ws.h_cg, sizeof(double) * 4096));
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

// ---- K5, single GPU: the whole solve in ONE persistent cooperative kernel ------------------------
// Single-reduction PCG (Chronopoulos-Gear form): with z = D^{-1} r and w = A z,
//   gamma = r'z, delta = z'w  (ONE grid reduction per iteration)
//   beta = gamma / gamma_old, alpha = gamma / (delta - beta gamma / alpha_old)
//   p = z + beta p, s = w + beta s (= A p), x += alpha p, r -= alpha s
// so an iteration is: mat-vec with fused z'w partials -> grid reduction -> fused vector update
// with r'z partials -> grid barrier.  Reductions are two-stage and ordered (block partials summed
// in block order by every CTA), so all CTAs take identical decisions and the result is bitwise
// reproducible.  delta - beta gamma / alpha_old equals p'Ap: <= 0 means "not positive definite".
constexpr int kPcgThreads = 512;

struct PcgParams {
    SpmvMat A;
    int nrhs, max_iter, n_long;
    int dbg;  // experiments only: 1 skip mat-vec, 2 skip vector update, 4 fixed iteration count
    double tol2;
    const double* rhs_a[kMaxRhs];
    const double* rhs_b[kMaxRhs];
    double *xa, *xb, *ra, *rb, *pa, *pb, *sa_, *sb_, *wa, *wb, *za, *zb;
    long sa, sb;
    double* blockpart;  // 2 buffers x gridDim.x x 2 kMaxRhs
    double* out;        // iters[kMaxRhs], breakdown flag
};

namespace cg = cooperative_groups;

// `extra` more NV-wide entries behind the per-block partials (the long lines' dot contributions)
// take part in the ordered sum
template <int NV>
__device__ __forceinline__ void grid_sum(cg::grid_group& grid, double (&v)[NV], double* scratch, double* bcast,
                                         double* blockpart, int& flip, int extra)
{
    block_sum<NV>(v, scratch);
    double* buf = blockpart + (size_t)flip * (gridDim.x + extra) * NV;
    flip ^= 1;
    if (threadIdx.x == 0)
        for (int k = 0; k < NV; ++k) buf[(size_t)blockIdx.x * NV + k] = v[k];
    grid.sync();
    if (threadIdx.x < 32 * NV) {  // warp k sums component k over the blocks, in block order
        const int k = threadIdx.x >> 5, l = threadIdx.x & 31;
        double s = 0.0;
        for (int b = l; b < (int)gridDim.x + extra; b += 32) s += __ldcg(buf + (size_t)b * NV + k);
        s = warp_sum(s);
        if (l == 0) bcast[k] = s;
    }
    __syncthreads();
    for (int k = 0; k < NV; ++k) v[k] = bcast[k];
    __syncthreads();
}

__global__ void __launch_bounds__(kPcgThreads) k_pcg_persistent(const PcgParams P)
{
    cg::grid_group grid = cg::this_grid();
    __shared__ double scratch[2 * kMaxRhs * (kPcgThreads / 32)];
    __shared__ double bcast[2 * kMaxRhs];
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nthr = gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31, gw = tid >> 5, nw = nthr >> 5;
    const int nloc = P.A.nloc, mfree = P.A.mm1, nrhs = P.nrhs;
    int flip = 0;

    // red[k] = gamma partial (r'z), red[kMaxRhs + k] = delta partial (z'w)
    double red[2 * kMaxRhs] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < nrhs; ++k) {
        for (int i = tid; i < nloc; i += nthr) {
            const double r = P.rhs_a[k][i], z = r / P.A.dA[i];
            P.xa[k * P.sa + i] = 0.0;
            P.ra[k * P.sa + i] = r;
            P.za[k * P.sa + i] = z;
            P.pa[k * P.sa + i] = 0.0;
            P.sa_[k * P.sa + i] = 0.0;
            red[k] += r * z;
        }
        for (int j = tid; j < mfree; j += nthr) {
            const double r = P.rhs_b[k][j], z = r / P.A.dB[j];
            P.xb[k * P.sb + j] = 0.0;
            P.rb[k * P.sb + j] = r;
            P.zb[k * P.sb + j] = z;
            P.pb[k * P.sb + j] = 0.0;
            P.sb_[k * P.sb + j] = 0.0;
            red[k] += r * z;
        }
    }
    grid.sync();  // z complete before the first mat-vec gathers it

    double gamma0[kMaxRhs] = {0.0, 0.0, 0.0}, gamma_old[kMaxRhs] = {1.0, 1.0, 1.0}, alpha_old[kMaxRhs] = {1.0, 1.0, 1.0};
    bool done[kMaxRhs] = {nrhs < 1, nrhs < 2, nrhs < 3};
    int iters[kMaxRhs] = {0, 0, 0};
    bool broke = false;
    for (int it = 0; it <= P.max_iter; ++it) {
        {   // w = A z with delta partials (lane 0 of each warp holds them)
            double zw[kMaxRhs] = {0.0, 0.0, 0.0};
            double* long_pq = P.blockpart + ((size_t)flip * (gridDim.x + P.n_long) + gridDim.x) * 2 * kMaxRhs;
            if (!(P.dbg & 1))
                spmv_warp<true>(P.A, nrhs, P.za, P.zb, P.sa, P.sb, P.wa, P.wb, gw, nw, lane, zw, long_pq);
#pragma unroll
            for (int k = 0; k < kMaxRhs; ++k) red[kMaxRhs + k] = zw[k];
        }
        grid_sum<2 * kMaxRhs>(grid, red, scratch, bcast, P.blockpart, flip, P.n_long);
        double al[kMaxRhs], be[kMaxRhs];
        bool all_done = true;
#pragma unroll
        for (int k = 0; k < kMaxRhs; ++k) {
            const double gamma = red[k], delta = red[kMaxRhs + k];
            al[k] = be[k] = 0.0;
            if (it == 0) {
                gamma0[k] = gamma;
                if (gamma == 0.0) done[k] = true;
            }
            if (!done[k] && gamma <= P.tol2 * gamma0[k]) done[k] = true;
            if (!done[k]) {
                be[k] = (it == 0) ? 0.0 : gamma / gamma_old[k];
                const double denom = delta - be[k] * gamma / alpha_old[k];
                if (!(denom > 0.0)) broke = true;  // p'Ap <= 0 (or NaN): not positive definite
                al[k] = gamma / denom;
                gamma_old[k] = gamma;
                alpha_old[k] = al[k];
                ++iters[k];
            }
            all_done &= done[k];
        }
        if (P.dbg & 4) {
            all_done = false;
            broke = false;
        }
        if (all_done || broke || it == P.max_iter) break;
#pragma unroll
        for (int k = 0; k < kMaxRhs; ++k) red[k] = 0.0;
        for (int k = 0; k < nrhs; ++k) {
            if (done[k] || (P.dbg & 2)) continue;
            const double a = al[k], b = be[k];
            for (int i = tid; i < nloc; i += nthr) {
                const size_t q = (size_t)k * P.sa + i;
                const double pn = P.za[q] + b * P.pa[q];
                const double sn = P.wa[q] + b * P.sa_[q];
                P.pa[q] = pn;
                P.sa_[q] = sn;
                P.xa[q] += a * pn;
                const double r = P.ra[q] - a * sn;
                P.ra[q] = r;
                const double z = r / P.A.dA[i];
                P.za[q] = z;
                red[k] += r * z;
            }
            for (int j = tid; j < mfree; j += nthr) {
                const size_t q = (size_t)k * P.sb + j;
                const double pn = P.zb[q] + b * P.pb[q];
                const double sn = P.wb[q] + b * P.sb_[q];
                P.pb[q] = pn;
                P.sb_[q] = sn;
                P.xb[q] += a * pn;
                const double r = P.rb[q] - a * sn;
                P.rb[q] = r;
                const double z = r / P.A.dB[j];
                P.zb[q] = z;
                red[k] += r * z;
            }
        }
        grid.sync();  // z complete before the next mat-vec gathers it
    }
    if (tid == 0) {
        for (int k = 0; k < kMaxRhs; ++k) P.out[k] = (double)iters[k];
        P.out[kMaxRhs] = broke ? 1.0 : 0.0;
    }
}

static int pcg_persistent(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, const regot_sparse& S, int nrhs,
                          const DVec* const* rhs, DVec* const* sol, double rtol, int max_iter)
{
    const int nloc = (int)S.nloc, mfree = (int)S.m - 1;
    const long sa = nloc, sb = std::max(mfree, 1);
    const size_t per = (size_t)kMaxRhs * (size_t)(sa + sb);
    ws.cg.ensure(6 * per + 16);
    static int blocks_per_sm = 0;
    if (!blocks_per_sm) {
        RG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_pcg_persistent, kPcgThreads, 0));
        if (blocks_per_sm < 1) raise(REGOT_E_CUDA, "pcg: persistent kernel does not fit on an SM");
        blocks_per_sm = std::min(blocks_per_sm, 1);
    }
    const int grid = blocks_per_sm * ctx->sm_count;
    ws.cg_partials.ensure((size_t)2 * (grid + S.n_long) * 2 * kMaxRhs + 8);
    ws.cg_scal.ensure(kScalCount + 2 * kMaxRhs);
    if (!ws.h_cg) RG_CUDA(cudaMallocHost((void**)&ws.h_cg, sizeof(double) * 4096));

    PcgParams P;
    P.A = mat_view(ctx, S);
    P.nrhs = nrhs;
    P.max_iter = max_iter;
    P.n_long = S.n_long;
    P.dbg = 0;
    if (const char* e = std::getenv("REGOT_B200_PCG_DBG")) {
        P.dbg = std::atoi(e);
        if (P.dbg & 4) P.max_iter = 1000;
    }
    P.tol2 = rtol * rtol;
    for (int k = 0; k < kMaxRhs; ++k) {
        P.rhs_a[k] = rhs[k < nrhs ? k : 0]->a.p;
        P.rhs_b[k] = rhs[k < nrhs ? k : 0]->b.p;
    }
    double* base = ws.cg.p;
    P.xa = base;
    P.xb = base + (size_t)kMaxRhs * sa;
    P.ra = base + per;
    P.rb = P.ra + (size_t)kMaxRhs * sa;
    P.pa = base + 2 * per;
    P.pb = P.pa + (size_t)kMaxRhs * sa;
    P.sa_ = base + 3 * per;
    P.sb_ = P.sa_ + (size_t)kMaxRhs * sa;
    P.wa = base + 4 * per;
    P.wb = P.wa + (size_t)kMaxRhs * sa;
    P.za = base + 5 * per;
    P.zb = P.za + (size_t)kMaxRhs * sa;
    P.sa = sa;
    P.sb = sb;
    P.blockpart = ws.cg_partials.p;
    P.out = ws.cg_scal.p;
    void* args[] = {&P};
    {
        ProfScope prof(ctx, st, 5);
        RG_CUDA(cudaLaunchCooperativeKernel((const void*)k_pcg_persistent, dim3(grid), dim3(kPcgThreads), args, 0, st));
    }
    ++ctx->launches;
    RG_CUDA(cudaMemcpyAsync(ws.h_cg, ws.cg_scal.p, sizeof(double) * (kMaxRhs + 1), cudaMemcpyDeviceToHost, st));
    RG_CUDA(cudaStreamSynchronize(st));
    if (ws.h_cg[kMaxRhs] != 0.0) return -1;
    int it = 0;
    for (int k = 0; k < nrhs; ++k) it = std::max(it, (int)ws.h_cg[k]);
    for (int k = 0; k < nrhs; ++k) {
        sol[k]->ensure(S.nloc, S.m);
        RG_CUDA(cudaMemcpyAsync(sol[k]->a.p, P.xa + (size_t)k * sa, sizeof(double) * (size_t)nloc, cudaMemcpyDeviceToDevice, st));
        RG_CUDA(cudaMemcpyAsync(sol[k]->b.p, P.xb + (size_t)k * sb, sizeof(double) * (size_t)mfree, cudaMemcpyDeviceToDevice, st));
        RG_CUDA(cudaMemsetAsync(sol[k]->b.p + mfree, 0, sizeof(double), st));
    }
    return it;
}

int sparse_pcg(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, SparseWS& ws, const regot_sparse& S, int nrhs,
               const DVec* const* rhs, DVec* const* sol, double rtol, int max_iter)
{
    if (nrhs < 1 || nrhs > kMaxRhs) raise(REGOT_E_VALIDATION, "pcg: bad number of right-hand sides");
    if (ctx->world == 1 && !ctx->force_multikernel_pcg) {
        static const bool full_system = std::getenv("REGOT_B200_PCG_FULL") != nullptr;  // A/B experiments only
        if (full_system) return pcg_persistent(ctx, st, ws, S, nrhs, rhs, sol, rtol, max_iter);
        return pcg_schur_persistent(ctx, st, ws, S, nrhs, rhs, sol, rtol, max_iter);
    }
    return pcg_multikernel(ctx, st, comm, ws, S, nrhs, rhs, sol, rtol, max_iter);
}

}  // namespace rg
