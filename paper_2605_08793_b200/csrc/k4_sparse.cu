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

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

namespace rg {

// ---- K3 -----------------------------------------------------------------------------------
__global__ void k_fill_values(int nnz, int nloc, int mm1, double eta, const ExpScale E, double tau, const int* __restrict__ row,
                              const int* __restrict__ col, const int* __restrict__ cscrow, const int* __restrict__ csccol,
                              const double* __restrict__ mval, const double* __restrict__ cscmval, const double* __restrict__ alpha,
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
    }
    // the CSC copy: the same arithmetic on the same operands in CSC order (identical bits), written coalesced -- scattering
    // the CSR values through slot[] was 8-byte writes to random sectors (config D: 0.58 ms per call)
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nnz; q += stride)
        cscval[q] = __ddiv_rn(plan_entry_dev_g((alpha[cscrow[q]] + beta[csccol[q]]) - cscmval[q], E, exp_table), eta);
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
                                        S.cscrow.p, S.csccol.p, S.mval.p, S.cscmval.p, alpha, beta, row_sums, col_sums, ctx->exp_table.p, S.val.p,
                                        S.cscval.p, S.dA.p, S.dB.p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
}

// ---- captured mass of the frozen pattern (pattern reuse, regot_b200_set_pattern_reuse) ---------------
// sum of the pattern's values and of the full row sums over eta, in a fixed order: thread-strided partial sums, a fixed
// shared-memory tree per block, then one block over the per-block partials.  The ratio is the share of the Hessian block's
// mass the pattern still holds at the current point; the solver compares it with the share at the last rebuild.
constexpr int kMassBlocks = 296, kMassThreads = 256;

__global__ void k_captured_mass_partials(int nnz, int nloc, double eta, const double* __restrict__ val,
                                         const double* __restrict__ row_sums, double* __restrict__ partials)
{
    __shared__ double sh[2][kMassThreads];
    const int stride = gridDim.x * blockDim.x;
    double sv = 0.0, sr = 0.0;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nnz; t += stride) sv = __dadd_rn(sv, val[t]);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += stride) sr = __dadd_rn(sr, __ddiv_rn(row_sums[i], eta));
    sh[0][threadIdx.x] = sv;
    sh[1][threadIdx.x] = sr;
    __syncthreads();
    for (int w = kMassThreads / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
            sh[0][threadIdx.x] = __dadd_rn(sh[0][threadIdx.x], sh[0][threadIdx.x + w]);
            sh[1][threadIdx.x] = __dadd_rn(sh[1][threadIdx.x], sh[1][threadIdx.x + w]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = sh[0][0];
        partials[2 * blockIdx.x + 1] = sh[1][0];
    }
}

__global__ void k_captured_mass_final(int blocks, const double* __restrict__ partials, double* __restrict__ out)
{
    if (threadIdx.x < 2) {
        double s = 0.0;
        for (int b = 0; b < blocks; ++b) s = __dadd_rn(s, partials[2 * b + threadIdx.x]);
        out[threadIdx.x] = s;
    }
}

double sparse_captured_mass(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, const regot_sparse& S, DevBuf<double>& scratch,
                            const double* row_sums)
{
    scratch.ensure(2 * kMassBlocks + 8);
    double* out = scratch.p + 2 * kMassBlocks;
    k_captured_mass_partials<<<kMassBlocks, kMassThreads, 0, st>>>((int)S.nnz, (int)S.nloc, ctx->prob.eta, S.val.p, row_sums, scratch.p);
    k_captured_mass_final<<<1, 32, 0, st>>>(kMassBlocks, scratch.p, out);
    RG_CUDA(cudaGetLastError());
    ctx->launches += 2;
    allreduce_sum(ctx, comm, out, 2, st);  // sharded runs: every rank takes the same decision from the same bits
    double h[2] = {0.0, 0.0};
    RG_CUDA(cudaMemcpyAsync(h, out, sizeof(h), cudaMemcpyDeviceToHost, st));
    RG_CUDA(cudaStreamSynchronize(st));
    return h[1] > 0.0 ? h[0] / h[1] : 0.0;
}

// oscillation of the dual variables since the pattern was built: out = {max d_alpha, -min d_alpha, max d_beta, -min d_beta}.
// Every entry of T moved by a factor within exp(+-(osc(d_alpha) + osc(d_beta)) / eta) relative to every other one, so a small
// oscillation bounds how far the top-k ranking can have moved.  One block (the vectors are n + m long).
__global__ void k_dual_drift(int nloc, int m, const double* __restrict__ a, const double* __restrict__ a0,
                             const double* __restrict__ b, const double* __restrict__ b0, double* __restrict__ out)
{
    __shared__ double sh[4][32];
    double v[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    for (int i = threadIdx.x; i < nloc; i += blockDim.x) {
        const double d = a[i] - a0[i];
        v[0] = fmax(v[0], d);
        v[1] = fmax(v[1], -d);
    }
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
        const double d = b[j] - b0[j];
        v[2] = fmax(v[2], d);
        v[3] = fmax(v[3], -d);
    }
    for (int q = 0; q < 4; ++q) {
        for (int o = 16; o > 0; o >>= 1) v[q] = fmax(v[q], __shfl_xor_sync(0xffffffffu, v[q], o));
        if ((threadIdx.x & 31) == 0) sh[q][threadIdx.x >> 5] = v[q];
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        double r = -INFINITY;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, sh[threadIdx.x][w]);
        out[threadIdx.x] = r;
    }
}

double dual_drift(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, const DVec& x, const DVec& x0, DevBuf<double>& scratch)
{
    scratch.ensure(2 * kMassBlocks + 8);
    double* out = scratch.p + 2 * kMassBlocks + 2;
    k_dual_drift<<<1, 1024, 0, st>>>((int)ctx->prob.nloc, (int)ctx->prob.m, x.a.p, x0.a.p, x.b.p, x0.b.p, out);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
    allreduce_max(ctx, comm, out, 4, st);  // alpha is row-sharded; the replicated beta entries are unchanged by the max
    double h[4];
    RG_CUDA(cudaMemcpyAsync(h, out, sizeof(h), cudaMemcpyDeviceToHost, st));
    RG_CUDA(cudaStreamSynchronize(st));
    return (h[0] + h[1]) + (h[2] + h[3]);
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
};

// part of one matrix line (row of B or column of B) against nrhs vectors: kLanes lanes stride
// over [beg, end) with kUnroll independent index/value loads and gathers in flight per lane
// (the mat-vec is latency-bound, not bandwidth-bound: everything lives in L2)
constexpr long kInterleaved4 = -4;  // stride value: right-hand sides interleaved 4 doubles per index

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
        if (sx == kInterleaved4) {
            // the right-hand sides interleaved 4 doubles per index: ONE 32-byte sector per gather (what bounds
            // a scattered gather through L2 is the number of requests, not bytes)
            double2 g01[kUnroll];
            double g2[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const double* q = x + (size_t)c[u] * 4;
                g01[u] = *reinterpret_cast<const double2*>(q);
                g2[u] = q[2];
            }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                acc[0] += a[u] * g01[u].x;
                acc[1] += a[u] * g01[u].y;
                acc[2] += a[u] * g2[u];
            }
        } else {
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
#pragma unroll
                for (int k = 0; k < kMaxRhs; ++k)
                    if (k < nrhs) acc[k] += a[u] * x[(size_t)k * sx + c[u]];
            }
        }
    }
}

// What a finished line's sum s becomes:
//   kEpiFull        y = diag * v_line + s       (A v over rows and columns, K4)
//   kEpiRowsScaled  y_a = s / dA                (rows only: t = D1^-1 B v_b, first half of S v)
//   kEpiColsPlain   y_b = s                     (columns only: u = B' v_a, second half; partial over row blocks)
// The two halves read and write vectors interleaved 4 doubles per index (stride argument kInterleaved4).
enum { kEpiFull = 0, kEpiRowsScaled = 1, kEpiColsPlain = 2 };

template <int kEpi>
__device__ __forceinline__ void line_store(const SpmvMat& A, int line, int k, double s, double diag, double vi,
                                           long sa, long sb, double* ya, double* yb)
{
    if (kEpi == kEpiFull) {
        const double y = diag * vi + s;
        if (line < A.nloc) ya[(size_t)k * sa + line] = y;
        else yb[(size_t)k * sb + (line - A.nloc)] = y;
    } else if (kEpi == kEpiRowsScaled) {
        ya[(size_t)line * 4 + k] = s / diag;  // the Schur halves keep their vectors interleaved x4
    } else {
        yb[(size_t)(line - A.nloc) * 4 + k] = s;
    }
}

// line pointers, diagonal entry and (kEpiFull) the line's own vector entries; issued before the
// gather loop so their latency overlaps it
template <int kEpi>
__device__ __forceinline__ void line_head(const SpmvMat& A, int line, int nrhs, const double* va,
                                          const double* vb, long sa, long sb, int& beg, int& end,
                                          double& diag, double (&vi)[kMaxRhs])
{
    if (line < A.nloc) {
        beg = __ldg(A.rowptr + line);
        end = __ldg(A.rowptr + line + 1);
        diag = (kEpi == kEpiColsPlain) ? 0.0 : __ldg(A.dA + line);
        if (kEpi == kEpiFull) {
#pragma unroll
            for (int k = 0; k < kMaxRhs; ++k)
                if (k < nrhs) vi[k] = va[(size_t)k * sa + line];
        }
    } else {
        const int j = line - A.nloc;
        beg = __ldg(A.cscptr + j);
        end = __ldg(A.cscptr + j + 1);
        diag = (kEpi == kEpiFull && A.add_diag_b) ? __ldg(A.dB + j) : 0.0;
        if (kEpi == kEpiFull) {
#pragma unroll
            for (int k = 0; k < kMaxRhs; ++k)
                if (k < nrhs) vi[k] = vb[(size_t)k * sb + j];
        }
    }
}

// sub-ranges of the three work lists (chunks of long lines, medium lines, short lines); rows come
// first in every list (finish_structure), so a half mat-vec is a range
struct LineRanges {
    int c0, c1, m0, m1, s0, s1;
};

// y = (part of) A v for nrhs vectors.  Lines are binned by length (finish_structure): long lines are
// cut into chunks spread over warps and combined in chunk order by the last warp to arrive; medium
// lines get a warp; short lines get 8 lanes, four lines in flight per warp.  Longest work first.
// Every sum has a fixed order (lane-strided partials, butterfly, chunk order): bitwise reproducible
// for a fixed grid.
template <int kEpi>
__device__ __forceinline__ void spmv_warp(const SpmvMat& A, const LineRanges R, int nrhs, const double* va,
                                          const double* vb, long sa, long sb, double* ya, double* yb, int gw, int nw,
                                          int lane)
{
    // ---- long lines: chunk partials ----
    for (int c = R.c0 + gw; c < R.c1; c += nw) {
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
            line_head<kEpi>(A, line, nrhs, va, vb, sa, sb, b2, e2, diag, vi);
#pragma unroll
            for (int k = 0; k < kMaxRhs; ++k) {
                if (k < nrhs) {
                    double s = 0.0;
                    for (int q = lane; q < cnt; q += 32) s += __ldcg(A.chunk_part + (size_t)(first + q) * kMaxRhs + k);
                    s = warp_sum(s);
                    if (lane == 0) line_store<kEpi>(A, line, k, s, diag, vi[k], sa, sb, ya, yb);
                }
            }
            if (lane == 0) A.chunk_cnt[slot] = 0u;
        }
    }
    // ---- medium lines: one warp each (handed out from the far end so chunk-laden warps get fewer) ----
    for (int q = R.m0 + nw - 1 - gw; q < R.m1; q += nw) {
        const int line = A.lines_m[q];
        int beg, end;
        double diag, vi[kMaxRhs] = {0.0, 0.0, 0.0}, acc[kMaxRhs] = {0.0, 0.0, 0.0};
        line_head<kEpi>(A, line, nrhs, va, vb, sa, sb, beg, end, diag, vi);
        if (line < A.nloc) line_dot<32, 4>(beg, end, lane, A.col, A.val, vb, sb, nrhs, acc);
        else line_dot<32, 4>(beg, end, lane, A.cscrow, A.cscval, va, sa, nrhs, acc);
#pragma unroll
        for (int k = 0; k < kMaxRhs; ++k) {
            if (k < nrhs) {
                const double s = warp_sum(acc[k]);
                if (lane == 0) line_store<kEpi>(A, line, k, s, diag, vi[k], sa, sb, ya, yb);
            }
        }
    }
    // ---- short lines: 8 lanes each, four lines in flight per warp ----
    const int sub = lane >> 3, gl = lane & 7;
    for (int base = R.s0 + gw * 4; base < R.s1; base += nw * 4) {
        const bool valid = base + sub < R.s1;
        int line = 0, beg = 0, end = 0;
        double diag = 0.0, vi[kMaxRhs] = {0.0, 0.0, 0.0}, acc[kMaxRhs] = {0.0, 0.0, 0.0};
        if (valid) {
            line = A.lines_s[base + sub];
            line_head<kEpi>(A, line, nrhs, va, vb, sa, sb, beg, end, diag, vi);
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
                if (valid && gl == 0) line_store<kEpi>(A, line, k, s, diag, vi[k], sa, sb, ya, yb);
            }
        }
    }
}

struct SpmvParams {
    const double* skip = nullptr;  // != null and *skip != 0: nothing to do (an iteration past the end of a PCG solve)
    SpmvMat A;
    LineRanges R;
    int nrhs;
    const double* va;
    const double* vb;
    double* ya;
    double* yb;
    long sa, sb;
};

template <int kEpi>
__global__ void __launch_bounds__(kSpmvThreads, 4) k_spmv(const SpmvParams p)
{
    if (p.skip != nullptr && *p.skip != 0.0) return;
    const int wpb = kSpmvThreads / 32;
    spmv_warp<kEpi>(p.A, p.R, p.nrhs, p.va, p.vb, p.sa, p.sb, p.ya, p.yb, blockIdx.x * wpb + (threadIdx.x >> 5),
                    gridDim.x * wpb, threadIdx.x & 31);
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
    A.add_diag_b = (!ctx->sharded || ctx->rank == 0) ? 1 : 0;
    return A;
}

// one (part of a) mat-vec: kEpiFull over all lines, or one of the two halves of the Schur mat-vec
template <int kEpi>
static void launch_spmv(regot_ctx* ctx, cudaStream_t st, const regot_sparse& S, int nrhs, const double* va,
                        const double* vb, double* ya, double* yb, long sa, long sb, const double* skip = nullptr)
{
    SpmvParams p;
    p.skip = skip;
    p.A = mat_view(ctx, S);
    if (kEpi == kEpiFull) p.R = LineRanges{0, S.n_chunks, 0, S.n_lines_m, 0, S.n_lines_s};
    else if (kEpi == kEpiRowsScaled) p.R = LineRanges{0, S.n_chunks_rows, 0, S.n_lines_m_rows, 0, S.n_lines_s_rows};
    else p.R = LineRanges{S.n_chunks_rows, S.n_chunks, S.n_lines_m_rows, S.n_lines_m, S.n_lines_s_rows, S.n_lines_s};
    p.nrhs = nrhs;
    p.va = va;
    p.vb = vb;
    p.ya = ya;
    p.yb = yb;
    p.sa = sa;
    p.sb = sb;
    const long items = (long)(p.R.c1 - p.R.c0) + (p.R.m1 - p.R.m0) + (p.R.s1 - p.R.s0 + 3) / 4;
    const int grid = (int)std::max<long>(1, std::min<long>((items + 7) / 8, 8L * ctx->sm_count));
    ProfScope prof(ctx, st, 4);
    k_spmv<kEpi><<<grid, kSpmvThreads, 0, st>>>(p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
}

void sparse_matvec(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, const regot_sparse& S, int nrhs, const double* va,
                   const double* vb, double* ya, double* yb, int64_t stride_a, int64_t stride_b)
{
    if (nrhs < 1 || nrhs > kMaxRhs) raise(REGOT_E_VALIDATION, "matvec: bad number of right-hand sides");
    launch_spmv<kEpiFull>(ctx, st, S, nrhs, va, vb, ya, yb, stride_a, stride_b);
    // column results are partial sums over the row blocks
    if (ctx->sharded) {
        for (int k = 0; k < nrhs; ++k) allreduce_sum(ctx, comm, yb + (size_t)k * stride_b, (size_t)S.m - 1, st);
    }
}

// ---- K4, panel form: the half mat-vecs of large patterns --------------------------------------------
// k_spmv gathers its vector through L2: one 32-byte sector per matrix entry (44 B of L2 traffic per 12-byte
// entry; config D: 1.1 GB per half mat-vec, 0.18 ms where the matrix itself streams from HBM in 0.05 ms).  Here the
// gathered vector is cut into P panels of W entries (16 B each: two right-hand sides) that fit in shared memory
// and the lines into Bk blocks per panel of equal work; CTA (p, b) copies panel p into shared memory ONCE
// (coalesced) and processes, for the lines of its block, the entries whose index falls inside the panel -- a
// contiguous piece of the line, since entries are sorted by index -- gathering from shared memory while the
// matrix streams from HBM.  Each (line, panel) piece is summed by one entity in a fixed order (8 lanes, a warp
// or the CTA, by length) into part[p][line]; k_panel_combine adds a line's P partials in panel order and
// applies the epilogue.  No atomics on values: bitwise reproducible.
constexpr int kPanelThreads = 1024;
constexpr int kPanelWarps = kPanelThreads / 32;
constexpr int kPanelMaxW = 12800;       // entries of the gathered vector per panel: 200 KB of shared memory
constexpr int kPanelEllW = 8448;        // ELL stream: narrower panels (132 KB) -- measured best at config D (7168..8352: 0.060 ms, 12800: 0.064)
constexpr int kPanelGroupMax = 256;     // pieces up to this many entries: 8 lanes
constexpr int kPanelWarpMax = 8192;     // up to this many: one warp; longer: the whole CTA
constexpr int kPanelDeferCap = 2048;    // deferred pieces per CTA kept in the shared-memory lists
constexpr int kPanelLineCost = 24;      // work of a piece beyond its entries (pointer loads, reduction), in entries
constexpr int kEllPieces = 8;           // ELL stream: pieces per chunk ...
constexpr int kEllPhases = 4;           // ... and lanes per piece (entry k of a piece belongs to lane group k % 4)
constexpr int kEllBatch = 4;            // rows per batch: a lane's values of a batch are 2 x 16 bytes, its indices 8 bytes
constexpr int kEllItemMax = 2048;        // entries per item: above kPanelGroupMax an item takes a chunk of its own (32 lanes)
constexpr int kEllKeyBits = 12;          // item cap - length fits in 12 bits

struct PanelArgs {
    const double* skip;  // != null and *skip != 0: nothing to do
    int P, Bk, W, nlines, ngather;
    const int* ppt;
    const int* blk;
    const unsigned short* idx;  // per entry: its index minus the first index of its panel (the panel is given by the piece)
    const double* val;  // val or cscval
    const double* x;    // gathered vector, interleaved 4 doubles per index
    double* part;       // P x nlines x 2
    // ELL stream (null eval: pieces are read from the CSR / CSC copy)
    const int* itembase;  // per piece q = p nlines + l: its first item (np + 1 entries)
    const int* nlong;     // per CTA: its long items (one chunk each; they sort first)
    const int* elen;      // per sorted item: entries, ...
    const int* eout;      // ... and where its two sums go (index into part, in pairs)
    const int* chrows;
    const int* choff;
    const unsigned short* eidx;
    const double* eval;
    int ahead;  // rows of the stream between a trip and the rows it prefetches into L2 (0: no prefetch)
#ifdef REGOT_PANEL_TIMING
    int fake;
#endif
};

// first entry of line l whose index is >= p W, for p = 0..P (p = P: the end of the line)
__global__ void k_panel_ptrs(int nlines, int P, int W, const int* __restrict__ ptr, const int* __restrict__ idx,
                             int* __restrict__ ppt, int* __restrict__ cost)
{
    const long total = (long)nlines * (P + 1);
    for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (long)gridDim.x * blockDim.x) {
        const int l = (int)(q / (P + 1)), p = (int)(q - (long)l * (P + 1));
        int lo = ptr[l], hi = ptr[l + 1];
        if (p == 0) hi = lo;
        else if (p < P) {
            const int key = p * W;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (idx[mid] < key) lo = mid + 1;
                else hi = mid;
            }
        } else lo = hi;
        ppt[q] = (p == 0) ? ptr[l] : lo;
    }
    (void)cost;
}
__global__ void k_panel_cost(int nlines, int P, const int* __restrict__ ppt, int* __restrict__ cost)
{
    const long total = (long)nlines * P;
    for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (long)gridDim.x * blockDim.x) {
        const int p = (int)(q / nlines), l = (int)(q - (long)p * nlines);
        const int len = ppt[(size_t)l * (P + 1) + p + 1] - ppt[(size_t)l * (P + 1) + p];
        cost[q] = len > 0 ? len + kPanelLineCost : 1;
    }
}
// 16-bit panel-relative indices (10 bytes per streamed entry instead of 12)
__global__ void k_panel_idx16(int nnz, int W, const int* __restrict__ idx, unsigned short* __restrict__ out)
{
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += gridDim.x * blockDim.x) out[e] = (unsigned short)(idx[e] % W);
}

// block b of panel p starts at the first line whose prefix work reaches b / Bk of the panel's total
__global__ void k_panel_blocks(int nlines, int P, int Bk, const int* __restrict__ scan, int* __restrict__ blk)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= P * (Bk + 1)) return;
    const int p = q / (Bk + 1), b = q - p * (Bk + 1);
    const int* s = scan + (size_t)p * nlines;
    const long base = s[0], tot = (long)scan[(size_t)(p + 1) * nlines] - base;
    int line = nlines;
    if (b < Bk) {
        const long target = base + tot * b / Bk;
        int lo = 0, hi = nlines;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if ((long)s[mid] < target) lo = mid + 1;
            else hi = mid;
        }
        line = lo;
    }
    blk[q] = line;
}

// ---- ELL stream: the pieces of a (panel, block) CTA as one contiguous, coalesced stream ------------------------------
// Reading the pieces where they lie in the CSR / CSC copy costs pointer loads per piece, half-empty trips (a piece of 125
// entries on 8 lanes x 8 in flight) and shuffles per piece; measured 0.085 ms per half at config D = 0.45 of the HBM roof.
// Here the pieces of a CTA up to kPanelGroupMax entries are sorted by length (stable), taken 8 to a chunk, and laid out so
// that a warp reads whole 256-byte rows: entry k of piece j of a chunk sits at row k / 4, lane (k % 4) * 8 + j.  Four
// lanes sum a piece, each its k % 4 class in order, then a fixed two-step butterfly: bitwise reproducible, and independent
// of which warp takes which chunk (chunks are handed out longest first through a counter).  Indices are laid out once per
// pattern; the values are copied into the layout once per solve (k_ell_values).
// items of piece q = p * nlines + l: its segments of up to kEllItemMax entries (an empty piece is one empty item)
__global__ void k_ell_count(int nlines, int P, const int* __restrict__ ppt, int* __restrict__ nseg)
{
    const long total = (long)nlines * P;
    for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q <= total; q += (long)gridDim.x * blockDim.x) {
        int ns = 0;
        if (q < total) {
            const int p = (int)(q / nlines), l = (int)(q - (long)p * nlines);
            const int len = ppt[(size_t)l * (P + 1) + p + 1] - ppt[(size_t)l * (P + 1) + p];
            ns = max(1, (len + kEllItemMax - 1) / kEllItemMax);
        }
        nseg[q] = ns;
    }
}
__global__ void k_ell_fill_u32(long n, unsigned v, unsigned* __restrict__ out)
{
    for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (long)gridDim.x * blockDim.x) out[q] = v;
}
// per line: does any of its pieces consist of several items (then the consumers add those items' sums first)
__global__ void k_ell_multi(int nlines, int P, const int* __restrict__ nseg, unsigned char* __restrict__ multi)
{
    for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nlines; l += gridDim.x * blockDim.x) {
        bool m = false;
        for (int p = 0; p < P; ++p) m = m || nseg[(size_t)p * nlines + l] > 1;
        multi[l] = m ? 1 : 0;
    }
}
__global__ void k_ell_keys(int nlines, int P, int Bk, const int* __restrict__ ppt, const int* __restrict__ blk,
                           const int* __restrict__ itembase, unsigned* __restrict__ key, int* __restrict__ id0, int* __restrict__ item_q)
{
    const long total = (long)nlines * P;
    for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (long)gridDim.x * blockDim.x) {
        const int p = (int)(q / nlines), l = (int)(q - (long)p * nlines);
        const int len = ppt[(size_t)l * (P + 1) + p + 1] - ppt[(size_t)l * (P + 1) + p];
        // the block of line l in panel p: the last b with blk[p][b] <= l (blocks may be empty)
        const int* bl = blk + (size_t)p * (Bk + 1);
        int lo = 0, hi = Bk;  // invariant: bl[lo] <= l, answer in [lo, hi)
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (bl[mid] <= l) lo = mid;
            else hi = mid;
        }
        const unsigned cta = (unsigned)(p * Bk + lo) << kEllKeyBits;
        const int b0 = itembase[q], ns = itembase[q + 1] - b0;
        for (int sg = 0; sg < ns; ++sg) {
            const int seglen = min(kEllItemMax, len - sg * kEllItemMax);
            key[b0 + sg] = cta | (unsigned)(kEllItemMax - seglen);
            id0[b0 + sg] = b0 + sg;
            item_q[b0 + sg] = (int)q;
        }
    }
}
// per sorted item: length, first entry, where its sums go (part[q] for a piece of one item, else part[np + item]); per CTA
// the number of long items (they sort first)
__global__ void k_ell_items(int nlines, int P, const int* __restrict__ ppt, const int* __restrict__ itembase,
                            const unsigned* __restrict__ key, const int* __restrict__ id, const int* __restrict__ item_q,
                            int* __restrict__ elen, int* __restrict__ ebeg, int* __restrict__ eout, int* __restrict__ nlong)
{
    const long np = (long)nlines * P;
    const long total = itembase[np];
    for (long r = (long)blockIdx.x * blockDim.x + threadIdx.x; r < total; r += (long)gridDim.x * blockDim.x) {
        const int it = id[r], q = item_q[it];
        const int p = q / nlines, l = q - p * nlines;
        const int b0 = itembase[q], ns = itembase[q + 1] - b0, sg = it - b0;
        const int beg = ppt[(size_t)l * (P + 1) + p], len = ppt[(size_t)l * (P + 1) + p + 1] - beg;
        const int seglen = min(kEllItemMax, len - sg * kEllItemMax);
        elen[r] = seglen;
        ebeg[r] = beg + sg * kEllItemMax;
        eout[r] = ns == 1 ? q : (int)np + it;
        if (seglen > kPanelGroupMax) atomicAdd(nlong + (key[r] >> kEllKeyBits), 1);
    }
}
// Chunks of CTA (p, b), whose sorted items are [first, first + cnt): the nl long items one per chunk (32 lanes, entry k
// at row k / 32), then the others 8 per chunk (4 lanes each, entry k at row k / 4).  Chunk slots of the CTA start at
// first + cta (an item per slot at worst).  Rows in whole batches of kEllBatch (the loads are vectors over 2 / 4 rows).
struct EllCta {
    int first, cnt, nl, nch, cb;
};
__device__ __forceinline__ EllCta ell_cta(int cta, int nlines, int Bk, const int* __restrict__ blk, const int* __restrict__ itembase,
                                          const int* __restrict__ nlong)
{
    const int p = cta / Bk, b = cta - p * Bk;
    const int l0 = __ldg(blk + (size_t)p * (Bk + 1) + b), l1 = __ldg(blk + (size_t)p * (Bk + 1) + b + 1);
    EllCta c;
    c.first = __ldg(itembase + (size_t)p * nlines + l0);
    c.cnt = __ldg(itembase + (size_t)p * nlines + l1) - c.first;
    c.nl = __ldg(nlong + cta);
    c.nch = c.nl + (c.cnt - c.nl + kEllPieces - 1) / kEllPieces;
    c.cb = c.first + cta;
    return c;
}
__global__ void k_ell_rows(int nlines, int P, int Bk, const int* __restrict__ blk, const int* __restrict__ itembase,
                           const int* __restrict__ nlong, const int* __restrict__ elen, int* __restrict__ chrows)
{
    const EllCta c = ell_cta(blockIdx.x, nlines, Bk, blk, itembase, nlong);
    (void)P;
    for (int ci = threadIdx.x; ci < c.nch; ci += blockDim.x) {
        const bool lng = ci < c.nl;
        const int len = elen[c.first + (lng ? ci : c.nl + (ci - c.nl) * kEllPieces)];
        const int per = (lng ? 32 : kEllPhases) * kEllBatch;
        chrows[c.cb + ci] = (len + per - 1) / per * kEllBatch;
    }
}
// indices and the slot -> entry map of every chunk: one warp per chunk, CTA c of the grid = CTA c of the mat-vec
__global__ void k_ell_fill(int nlines, int P, int Bk, const int* __restrict__ blk, const int* __restrict__ itembase,
                           const int* __restrict__ nlong, const int* __restrict__ elen, const int* __restrict__ ebeg,
                           const int* __restrict__ chrows, const int* __restrict__ choff, const unsigned short* __restrict__ idx16,
                           int* __restrict__ emap, unsigned short* __restrict__ eidx)
{
    const EllCta c = ell_cta(blockIdx.x, nlines, Bk, blk, itembase, nlong);
    (void)P;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int ci = warp; ci < c.nch; ci += nwarps) {
        const int rows = chrows[c.cb + ci];
        const size_t off = (size_t)choff[c.cb + ci] * 32;
        const bool lng = ci < c.nl;
        const int G = lng ? 32 : kEllPhases, g = lng ? lane : lane >> 3;
        const int pos = lng ? ci : c.nl + (ci - c.nl) * kEllPieces + (lane & 7);
        int beg = 0, eff = 0;
        if (pos < c.cnt) {
            eff = elen[c.first + pos];
            beg = ebeg[c.first + pos];
        }
        for (int t = 0; t < rows; ++t) {
            const int k = t * G + g;
            const bool ok = k < eff;
            // values: rows in pairs, a lane's two values adjacent; indices: rows in fours, a lane's four adjacent
            emap[off + (size_t)(t >> 1) * 64 + lane * 2 + (t & 1)] = ok ? beg + k : -1;
            eidx[off + (size_t)(t >> 2) * 128 + lane * 4 + (t & 3)] = ok ? idx16[beg + k] : (unsigned short)0;
        }
    }
}
// the values into the layout, once per solve; the slot count comes from the scan (device memory)
__global__ void k_ell_values(const int* __restrict__ total_rows, const int* __restrict__ emap, const double* __restrict__ val,
                             double* __restrict__ eval)
{
    const long total = (long)(*total_rows) * 32;
    for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (long)gridDim.x * blockDim.x) {
        const int e = emap[q];
        eval[q] = e >= 0 ? __ldg(val + e) : 0.0;
    }
}

// lanes stride over [beg, end) with kLanes lanes and 8 entries in flight per lane; gathers from the staged panel
template <int kLanes>
__device__ __forceinline__ void panel_dot(int beg, int end, int gl, const unsigned short* __restrict__ idx,
                                          const double* __restrict__ val, uint32_t vec, double& a0, double& a1)
{
    for (int t = beg + gl; t < end; t += kLanes * 8) {
        unsigned c[8];
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int tt = t + kLanes * u;
            const bool ok = tt < end;
            c[u] = ok ? (unsigned)__ldg(idx + tt) : 0u;
            v[u] = ok ? __ldg(val + tt) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double2 g = lds_f64x2(vec + c[u] * 16u);
            a0 = __fma_rn(v[u], g.x, a0);
            a1 = __fma_rn(v[u], g.y, a1);
        }
    }
}

__global__ void __launch_bounds__(kPanelThreads, 1) k_spmv_panel(const PanelArgs a)
{
    extern __shared__ __align__(16) unsigned char smem[];
    if (a.skip != nullptr && *a.skip != 0.0) return;
    const int p = blockIdx.x / a.Bk, b = blockIdx.x - p * a.Bk;
    const int col0 = p * a.W, wp = min(a.W, a.ngather - col0);
    const uint32_t vec = smem_u32(smem);
    int* defer_w = reinterpret_cast<int*>(smem + (size_t)a.W * 16);  // pieces for a warp
    int* defer_c = defer_w + kPanelDeferCap;                         // pieces for the CTA
    double* wpart = reinterpret_cast<double*>(defer_c + kPanelDeferCap);  // kPanelWarps x 2
    __shared__ int n_defer_w, n_defer_c, next_chunk;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) n_defer_w = n_defer_c = next_chunk = 0;
#ifdef REGOT_PANEL_TIMING
    __shared__ long long t_warp[kPanelWarps];
    const long long t_0 = clock64();
#endif
    // stage the panel: entries (x[4 j], x[4 j + 1]) of the interleaved vector
    for (int j = tid; j < wp; j += kPanelThreads) {
        const double2 g = __ldcg(reinterpret_cast<const double2*>(a.x + (size_t)(col0 + j) * 4));
        asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(vec + (uint32_t)j * 16u), "d"(g.x), "d"(g.y) : "memory");
    }
    __syncthreads();
#ifdef REGOT_PANEL_TIMING
    const long long t_1 = clock64();
#endif
    const int l0 = a.blk[p * (a.Bk + 1) + b], l1 = a.blk[p * (a.Bk + 1) + b + 1];
    const size_t pstride = (size_t)(a.P + 1);
    double* const part = a.part + (size_t)p * a.nlines * 2;

    if (a.eval != nullptr) {
        // ---- pass 1, ELL stream: chunks of 8 pieces handed out longest first; 4 lanes per piece ----
        const EllCta ec = ell_cta(blockIdx.x, a.nlines, a.Bk, a.blk, a.itembase, a.nlong);
        const int nch = ec.nch, cb = ec.cb;
        // the CTA's stream is contiguous (chunk after chunk); with a.ahead > 0 every trip asks L2 for the 8 rows a.ahead
        // rows further down the stream (measured: no gain -- the stream is not bound by latency; off by default)
        const int end_row = __ldg(a.choff + cb + nch);
        if (a.ahead > 0 && lane < 2) {  // the head of the stream, which no trip asks for
            const int begin_row = __ldg(a.choff + cb);
            for (int r = begin_row + warp * 8; r < min(begin_row + a.ahead, end_row - 8); r += kPanelWarps * 8) {
                if (lane == 0)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.eval + (size_t)r * 32), "r"(8 * 32 * 8) : "memory");
                else
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.eidx + (size_t)r * 32), "r"(8 * 32 * 2) : "memory");
            }
        }
        for (;;) {
            int ci = 0;
            if (lane == 0) ci = atomicAdd(&next_chunk, 1);
            ci = __shfl_sync(0xffffffffu, ci, 0);
            if (ci >= nch) break;
            const int rows = __ldg(a.chrows + cb + ci);
            const int row0 = __ldg(a.choff + cb + ci);
            const bool lng = ci < ec.nl;  // a long item alone on 32 lanes, else 8 items on 4 lanes each
            const int G = lng ? 32 : kEllPhases, g = lng ? lane : lane >> 3;
            const int pos = lng ? ci : ec.nl + (ci - ec.nl) * kEllPieces + (lane & 7);
            const bool valid = pos < ec.cnt;
            int dest = 0, eff = 0;
            if (valid) {
                eff = __ldg(a.elen + ec.first + pos);
                dest = __ldg(a.eout + ec.first + pos);
            }
            const double* vp = a.eval + (size_t)row0 * 32 + lane * 2;          // + (t / 2) * 64: rows t, t + 1
            const unsigned short* ip = a.eidx + (size_t)row0 * 32 + lane * 4;  // + (t / 4) * 128: rows t .. t + 3
            double a0 = 0.0, a1 = 0.0;
            // A batch is 4 rows: per lane two 16-byte loads of values and one 8-byte load of indices (the LSU takes a
            // request per instruction whatever its width: 16 scalar loads per 8 rows kept its queue full -- lg_throttle --
            // at 13 B/clk per SM).  Two batches in registers: one is loaded while the other is consumed.  L1::no_allocate:
            // the stream is read once, and with the panel in shared memory L1 is too small to hold the lines in flight.
            // Vectors wholly past the item's end are not loaded; padding inside a vector is (value 0, index 0).
            struct Batch {
                double2 v01, v23;
                uint2 c;
            };
            auto load4 = [&](int t, Batch& B) {
                B.v01 = B.v23 = make_double2(0.0, 0.0);
                B.c = make_uint2(0u, 0u);
                if (t * G + g < eff) {
                    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(B.c.x), "=r"(B.c.y) : "l"(ip + (size_t)(t >> 2) * 128));
                    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(B.v01.x), "=d"(B.v01.y) : "l"(vp + (size_t)(t >> 1) * 64));
                }
                if ((t + 2) * G + g < eff)
                    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(B.v23.x), "=d"(B.v23.y) : "l"(vp + (size_t)((t >> 1) + 1) * 64));
            };
            auto use1 = [&](unsigned c, double v) {
#ifdef REGOT_PANEL_TIMING
                if (a.fake == 1) c = lane;  // (experiment) conflict-free gather
                if (a.fake == 2) {          // (experiment) the stream alone: no gather
                    a0 = __fma_rn(v, (double)c, a0);
                    return;
                }
#endif
                const double2 gv = lds_f64x2(vec + c * 16u);
                a0 = __fma_rn(v, gv.x, a0);
                a1 = __fma_rn(v, gv.y, a1);
            };
            auto use4 = [&](const Batch& B) {
                use1(B.c.x & 0xffffu, B.v01.x);
                use1(B.c.x >> 16, B.v01.y);
                use1(B.c.y & 0xffffu, B.v23.x);
                use1(B.c.y >> 16, B.v23.y);
            };
            Batch bA, bB;
            load4(0, bA);
            for (int t = 0; t < rows; t += 8) {
                if (a.ahead > 0) {
                    const int prow = row0 + t + a.ahead;
                    if (prow + 8 <= end_row) {
                        // one bulk request per array: 8 rows of values (2 KB) and of indices (512 B)
                        if (lane == 0)
                            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.eval + (size_t)prow * 32), "r"(8 * 32 * 8) : "memory");
                        else if (lane == 1)
                            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.eidx + (size_t)prow * 32), "r"(8 * 32 * 2) : "memory");
                    }
                }
                load4(t + 4, bB);
                use4(bA);
                load4(t + 8, bA);
                use4(bB);
            }
            // short items: lane groups 0 / 2 end with the item's sum of a0, groups 1 / 3 with a1, then the pairs; a long
            // item: the butterfly over the warp, even lanes carrying a0 and odd lanes a1 after the first step (fixed orders)
            double c2;
            if (lng) {
                const bool odd = lane & 1;
                c2 = (odd ? a1 : a0) + shfl_xor_d(odd ? a0 : a1, 1);
                c2 += shfl_xor_d(c2, 2);
                c2 += shfl_xor_d(c2, 4);
                c2 += shfl_xor_d(c2, 8);
                c2 += shfl_xor_d(c2, 16);
            } else {
                const bool odd = g & 1;
                c2 = (odd ? a1 : a0) + shfl_xor_d(odd ? a0 : a1, 8);
                c2 += shfl_xor_d(c2, 16);
            }
            if (valid && g < 2) a.part[(size_t)dest * 2 + g] = c2;  // long: lanes 0 and 1
        }
#ifndef REGOT_PANEL_TIMING
        return;  // every piece went through the stream: no deferred pieces
#endif
    } else {
        // ---- pass 1: four lines per warp, 8 lanes each; longer pieces are deferred ----
        const int sub = lane >> 3, gl = lane & 7;
        // The pointers of a group of lines are loaded two trips ahead and the piece they delimit is prefetched into L2 one
        // trip ahead (with pointers that arrived a trip ago: the prefetch does not wait for a load): the demand loads of the
        // next trip then pay an L2 latency instead of an HBM one.  The kernel is bound by loads in flight, and prefetches
        // hold no registers.
        auto piece = [&](int l, int& pb, int& pe) {
            pb = pe = 0;
            if (l < l1) {
                pb = __ldg(a.ppt + (size_t)l * pstride + p);
                pe = __ldg(a.ppt + (size_t)l * pstride + p + 1);
            }
        };
        int nbeg, nend, n2beg, n2end;
        piece(l0 + warp * 4 + sub, nbeg, nend);
        piece(l0 + warp * 4 + sub + kPanelWarps * 4, n2beg, n2end);
        for (int base = l0 + warp * 4; base < l1; base += kPanelWarps * 4) {
            const int l = base + sub;
            const int beg = nbeg, end = nend;
            nbeg = n2beg;
            nend = n2end;
            piece(l + 2 * kPanelWarps * 4, n2beg, n2end);
            {
                const int plen = min(nend - nbeg, kPanelGroupMax);
                // 16 values or 64 indices per 128-byte line
                for (int t = gl * 16; t < plen; t += 8 * 16) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.val + nbeg + t));
                for (int t = gl * 64; t < plen; t += 8 * 64) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.idx + nbeg + t));
            }
            const int len = end - beg;
            double a0 = 0.0, a1 = 0.0;
            if (len > kPanelGroupMax) {
                if (gl == 0) {
                    const bool cta = len > kPanelWarpMax;
                    const int slot = atomicAdd(cta ? &n_defer_c : &n_defer_w, 1);
                    if (slot < kPanelDeferCap) (cta ? defer_c : defer_w)[slot] = l;
                }
            } else if (len > 0) {
                panel_dot<8>(beg, end, gl, a.idx, a.val, vec, a0, a1);
            }
            // even lanes of a group end with the group's sum of a0, odd lanes with a1 (fixed order)
            const bool odd = lane & 1;
            double c = (odd ? a1 : a0) + shfl_xor_d(odd ? a0 : a1, 1);
            c += shfl_xor_d(c, 2);
            c += shfl_xor_d(c, 4);
            if (l < l1 && len <= kPanelGroupMax && gl < 2) part[(size_t)l * 2 + gl] = c;
        }
    }
#ifdef REGOT_PANEL_TIMING
    if (lane == 0) t_warp[warp] = clock64();
#endif
    __syncthreads();
#ifdef REGOT_PANEL_TIMING
    const long long t_2 = clock64();
#endif
    // ---- pass 2: one warp per deferred piece ----
    const int nw_list = min(n_defer_w, kPanelDeferCap), nc_list = min(n_defer_c, kPanelDeferCap);
    const bool overflow = n_defer_w > kPanelDeferCap || n_defer_c > kPanelDeferCap;
    for (int q = warp; q < nw_list; q += kPanelWarps) {
        const int l = defer_w[q];
        const int beg = __ldg(a.ppt + (size_t)l * pstride + p), end = __ldg(a.ppt + (size_t)l * pstride + p + 1);
        double a0 = 0.0, a1 = 0.0;
        panel_dot<32>(beg, end, lane, a.idx, a.val, vec, a0, a1);
        a0 = warp_sum(a0);
        a1 = warp_sum(a1);
        if (lane == 0) {
            part[(size_t)l * 2] = a0;
            part[(size_t)l * 2 + 1] = a1;
        }
    }
    // ---- pass 3: the whole CTA per very long piece (row 0 / column 0 of Omega*) ----
    for (int q = 0; q < nc_list; ++q) {
        const int l = defer_c[q];
        const int beg = __ldg(a.ppt + (size_t)l * pstride + p), end = __ldg(a.ppt + (size_t)l * pstride + p + 1);
        double a0 = 0.0, a1 = 0.0;
        panel_dot<kPanelThreads>(beg, end, tid, a.idx, a.val, vec, a0, a1);
        a0 = warp_sum(a0);
        a1 = warp_sum(a1);
        if (lane == 0) {
            wpart[warp * 2] = a0;
            wpart[warp * 2 + 1] = a1;
        }
        __syncthreads();
        if (tid < 2) {
            double s = 0.0;
            for (int w = 0; w < kPanelWarps; ++w) s += wpart[w * 2 + tid];
            part[(size_t)l * 2 + tid] = s;
        }
        __syncthreads();
    }
#ifdef REGOT_PANEL_TIMING
    __syncthreads();
    if (tid == 0 && a.ahead == 7777) {
        long long lo = t_warp[0], hi = t_warp[0], sum = 0;
        for (int w = 0; w < kPanelWarps; ++w) {
            lo = min(lo, t_warp[w]);
            hi = max(hi, t_warp[w]);
            sum += t_warp[w] - t_1;
        }
        printf("panel cta %3d p %d b %2d lines %5d stage %6lld pass1 first %6lld mean %6lld last %6lld pass23 %6lld defer %d %d\n", (int)blockIdx.x,
               p, b, l1 - l0, t_1 - t_0, lo - t_1, sum / kPanelWarps, hi - t_1, clock64() - t_2, n_defer_w, n_defer_c);
    }
#endif
    // more deferred pieces than the lists hold (never at the sizes this path is meant for): rescan, one warp each
    if (overflow) {
        for (int l = l0 + warp; l < l1; l += kPanelWarps) {
            const int beg = __ldg(a.ppt + (size_t)l * pstride + p), end = __ldg(a.ppt + (size_t)l * pstride + p + 1);
            if (end - beg <= kPanelGroupMax) continue;
            double a0 = 0.0, a1 = 0.0;
            panel_dot<32>(beg, end, lane, a.idx, a.val, vec, a0, a1);
            a0 = warp_sum(a0);
            a1 = warp_sum(a1);
            if (lane == 0) {
                part[(size_t)l * 2] = a0;
                part[(size_t)l * 2 + 1] = a1;
            }
        }
    }
}

// sums (both right-hand sides) of line l's per-panel partials in panel order; a piece the ELL stream cut into several items
// is summed in item order first (its items' sums sit behind the P x nlines piece slots).  The loads of the common case
// are independent 16-byte loads.
__device__ __forceinline__ double2 panel_line_sum2(const double* __restrict__ part, const int* __restrict__ itembase,
                                                   const unsigned char* __restrict__ multi, int nlines, int P, int l)
{
    const double2* part2 = reinterpret_cast<const double2*>(part);
    // the common case first and unconditionally (its loads do not wait for the flag): every piece of the line is one item
    const bool cut = itembase != nullptr && multi[l] != 0;
    double2 s = make_double2(0.0, 0.0);
#pragma unroll 4
    for (int p = 0; p < P; ++p) {
        const double2 t = part2[(size_t)p * nlines + l];
        s.x += t.x;
        s.y += t.y;
    }
    if (!cut) return s;
    s = make_double2(0.0, 0.0);
    const size_t np = (size_t)nlines * P;
    for (int p = 0; p < P; ++p) {
        const size_t q = (size_t)p * nlines + l;
        const int b0 = itembase[q], ns = itembase[q + 1] - b0;
        double2 t = make_double2(0.0, 0.0);
        if (ns == 1) {
            t = part2[q];
        } else {
            for (int sg = 0; sg < ns; ++sg) {
                const double2 c = part2[np + (size_t)(b0 + sg)];
                t.x += c.x;
                t.y += c.y;
            }
        }
        s.x += t.x;
        s.y += t.y;
    }
    return s;
}

// y_line = sum over panels (panel order) of part[p][line], then the epilogue of the half mat-vec
template <int kEpi>
__global__ void k_panel_combine(int nlines, int P, const double* __restrict__ part, const int* __restrict__ itembase,
                                const unsigned char* __restrict__ multi, const double* __restrict__ diag, double* __restrict__ y,
                                const double* skip)
{
    if (skip != nullptr && *skip != 0.0) return;
    for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nlines; l += gridDim.x * blockDim.x) {
        double2 sm = panel_line_sum2(part, itembase, multi, nlines, P, l);
        if (kEpi == kEpiRowsScaled) {
            const double d = diag[l];
            sm.x = sm.x / d;
            sm.y = sm.y / d;
        }
        *reinterpret_cast<double2*>(y + (size_t)l * 4) = sm;
    }
}

static constexpr int panel_smem(int W, bool ell = false) { return W * 16 + (ell ? 0 : 2 * kPanelDeferCap * 4 + kPanelWarps * 2 * 8); }

// (re)build the plan of one half for the current pattern; everything stays on the device
static void build_panel_plan(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, const regot_sparse& S, bool rows)
{
    PanelPlan& Q = rows ? S.panel_rows : S.panel_cols;
    if (Q.stamp == S.structure_stamp && Q.P > 0) return;
    const int nloc = (int)S.nloc, mfree = std::max((int)S.m - 1, 0);
    Q.nlines = rows ? nloc : mfree;
    Q.ngather = rows ? mfree : nloc;
    const int wmax = ctx->panel_width > 0 ? std::min(ctx->panel_width, kPanelMaxW) : (ctx->panel_ell ? kPanelEllW : kPanelMaxW);
    Q.P = std::max(1, (Q.ngather + wmax - 1) / wmax);
    if (Q.P > ctx->sm_count) raise(REGOT_E_UNSUPPORTED, "panel mat-vec: the gathered vector needs more panels than there are SMs");
    Q.W = ((Q.ngather + Q.P - 1) / Q.P + 31) / 32 * 32;
    Q.Bk = std::max(1, ctx->sm_count / Q.P);
    const size_t np = (size_t)Q.P * (size_t)Q.nlines;
    Q.ppt.ensure((size_t)Q.nlines * (Q.P + 1) + 1);
    Q.cost.ensure(np + 1);
    Q.scan.ensure(np + 1);
    Q.blk.ensure((size_t)Q.P * (Q.Bk + 1));
    Q.part.ensure(np * 2 + 2);
    Q.idx16.ensure((size_t)S.nnz + 8);
    const int* ptr = rows ? S.rowptr.p : S.cscptr.p;
    const int* idx = rows ? S.col.p : S.cscrow.p;
    k_panel_idx16<<<(int)std::max<long>(1, std::min<long>(((long)S.nnz + 255) / 256, 8L * ctx->sm_count)), 256, 0, st>>>((int)S.nnz, Q.W, idx,
                                                                                                                    Q.idx16.p);
    const int g1 = (int)std::max<long>(1, std::min<long>(((long)Q.nlines * (Q.P + 1) + 255) / 256, 8L * ctx->sm_count));
    k_panel_ptrs<<<g1, 256, 0, st>>>(Q.nlines, Q.P, Q.W, ptr, idx, Q.ppt.p, Q.cost.p);
    k_panel_cost<<<g1, 256, 0, st>>>(Q.nlines, Q.P, Q.ppt.p, Q.cost.p);
    RG_CUDA(cudaMemsetAsync(Q.cost.p + np, 0, sizeof(int), st));
    size_t bytes = 0;
    RG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, Q.cost.p, Q.scan.p, (int)(np + 1), st));
    ws.cub_tmp.ensure(bytes);
    RG_CUDA(cub::DeviceScan::ExclusiveSum(ws.cub_tmp.p, bytes, Q.cost.p, Q.scan.p, (int)(np + 1), st));
    const int nb = Q.P * (Q.Bk + 1);
    k_panel_blocks<<<(nb + 127) / 128, 128, 0, st>>>(Q.nlines, Q.P, Q.Bk, Q.scan.p, Q.blk.p);
    RG_CUDA(cudaGetLastError());
    ctx->launches += 5;
    if (ctx->panel_ell) {
        // ELL stream: every piece cut into items of up to kPanelGroupMax entries, the items of a CTA sorted by length
        // (stable), chunk tables, indices.  Item and slot counts stay on the device; the buffers take their bounds.
        const int ncta = Q.P * Q.Bk;
        Q.item_cap = np + (size_t)S.nnz / kEllItemMax + 1;
        Q.nchunk_slots = (int)Q.item_cap + ncta + 1;
        // slots: the entries, the sorted short chunks' slack (16 x 256 per CTA), up to a batch of rows of padding per chunk
        const size_t max_chunks = Q.item_cap / kEllPieces + (size_t)ncta + (size_t)S.nnz / (kPanelGroupMax + 1) + 1;
        Q.ell_cap = (size_t)S.nnz + (size_t)ncta * 2 * kEllPieces * kPanelGroupMax + max_chunks * 32 * kEllBatch + 64;
        Q.nseg.ensure(np + 2);
        Q.itembase.ensure(np + 2);
        Q.ekey.ensure(Q.item_cap);
        Q.ekey2.ensure(Q.item_cap);
        Q.eid0.ensure(Q.item_cap);
        Q.eid.ensure(Q.item_cap);
        Q.item_q.ensure(Q.item_cap);
        Q.elen.ensure(Q.item_cap);
        Q.ebeg.ensure(Q.item_cap);
        Q.eout.ensure(Q.item_cap);
        Q.nlong.ensure((size_t)ncta + 1);
        Q.multi.ensure((size_t)Q.nlines + 1);
        Q.chrows.ensure((size_t)Q.nchunk_slots + 1);
        Q.choff.ensure((size_t)Q.nchunk_slots + 1);
        Q.emap.ensure(Q.ell_cap);
        Q.eidx.ensure(Q.ell_cap);
        Q.eval.ensure(Q.ell_cap);
        Q.part.ensure((np + Q.item_cap) * 2 + 2);
        // the piece slots of cut pieces are never written but are read (and discarded) by the consumers' common-case loads
        RG_CUDA(cudaMemsetAsync(Q.part.p, 0, sizeof(double) * ((np + Q.item_cap) * 2 + 2), st));
        const int gi = (int)std::max<long>(1, std::min<long>(((long)np + 255) / 256, 8L * ctx->sm_count));
        const int gk = (int)std::max<long>(1, std::min<long>(((long)Q.item_cap + 255) / 256, 8L * ctx->sm_count));
        int cta_bits = 1;
        while ((1 << cta_bits) < ncta) ++cta_bits;
        const int key_bits = kEllKeyBits + cta_bits + 1;  // the top bit marks the unused tail of the item arrays
        size_t sbytes = 0;
        k_ell_count<<<gi, 256, 0, st>>>(Q.nlines, Q.P, Q.ppt.p, Q.nseg.p);
        RG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, sbytes, Q.nseg.p, Q.itembase.p, (int)np + 1, st));
        ws.cub_tmp.ensure(sbytes);
        RG_CUDA(cub::DeviceScan::ExclusiveSum(ws.cub_tmp.p, sbytes, Q.nseg.p, Q.itembase.p, (int)np + 1, st));
        k_ell_fill_u32<<<gk, 256, 0, st>>>((long)Q.item_cap, 1u << (kEllKeyBits + cta_bits), Q.ekey.p);
        RG_CUDA(cudaMemsetAsync(Q.eid0.p, 0, sizeof(int) * Q.item_cap, st));  // the unused tail is sorted along (to the end)
        k_ell_keys<<<gi, 256, 0, st>>>(Q.nlines, Q.P, Q.Bk, Q.ppt.p, Q.blk.p, Q.itembase.p, Q.ekey.p, Q.eid0.p, Q.item_q.p);
        RG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sbytes, Q.ekey.p, Q.ekey2.p, Q.eid0.p, Q.eid.p, (int)Q.item_cap, 0, key_bits, st));
        ws.cub_tmp.ensure(sbytes);
        RG_CUDA(cub::DeviceRadixSort::SortPairs(ws.cub_tmp.p, sbytes, Q.ekey.p, Q.ekey2.p, Q.eid0.p, Q.eid.p, (int)Q.item_cap, 0, key_bits, st));
        RG_CUDA(cudaMemsetAsync(Q.chrows.p, 0, sizeof(int) * ((size_t)Q.nchunk_slots + 1), st));
        RG_CUDA(cudaMemsetAsync(Q.nlong.p, 0, sizeof(int) * ((size_t)ncta + 1), st));
        k_ell_items<<<gk, 256, 0, st>>>(Q.nlines, Q.P, Q.ppt.p, Q.itembase.p, Q.ekey2.p, Q.eid.p, Q.item_q.p, Q.elen.p, Q.ebeg.p, Q.eout.p,
                                        Q.nlong.p);
        k_ell_rows<<<ncta, 256, 0, st>>>(Q.nlines, Q.P, Q.Bk, Q.blk.p, Q.itembase.p, Q.nlong.p, Q.elen.p, Q.chrows.p);
        k_ell_multi<<<(Q.nlines + 255) / 256, 256, 0, st>>>(Q.nlines, Q.P, Q.nseg.p, Q.multi.p);
        RG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, sbytes, Q.chrows.p, Q.choff.p, Q.nchunk_slots + 1, st));
        ws.cub_tmp.ensure(sbytes);
        RG_CUDA(cub::DeviceScan::ExclusiveSum(ws.cub_tmp.p, sbytes, Q.chrows.p, Q.choff.p, Q.nchunk_slots + 1, st));
        k_ell_fill<<<ncta, 1024, 0, st>>>(Q.nlines, Q.P, Q.Bk, Q.blk.p, Q.itembase.p, Q.nlong.p, Q.elen.p, Q.ebeg.p, Q.chrows.p,
                                          Q.choff.p, Q.idx16.p, Q.emap.p, Q.eidx.p);
        RG_CUDA(cudaGetLastError());
        ctx->launches += 10;
    }
    Q.stamp = S.structure_stamp;
}

// the current values of the half's matrix copy into the ELL stream (once per solve: the values change between solves)
static void panel_refresh_values(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, const regot_sparse& S, bool rows)
{
    if (!ctx->panel_ell) return;
    build_panel_plan(ctx, st, ws, S, rows);
    PanelPlan& Q = rows ? S.panel_rows : S.panel_cols;
    k_ell_values<<<8 * ctx->sm_count, 256, 0, st>>>(Q.choff.p + Q.nchunk_slots, Q.emap.p, rows ? S.val.p : S.cscval.p, Q.eval.p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
}

// one half mat-vec in panel form: y (interleaved x4) = epilogue(B x) or epilogue(B' x) for two right-hand sides
template <int kEpi>
static void launch_spmv_panel(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, const regot_sparse& S, const double* x, double* y,
                              const double* skip = nullptr, bool combine = true)
{
    constexpr bool rows = kEpi == kEpiRowsScaled;
    build_panel_plan(ctx, st, ws, S, rows);
    const PanelPlan& Q = rows ? S.panel_rows : S.panel_cols;
    static bool attr_set = false;
    if (!attr_set) {
        RG_CUDA(cudaFuncSetAttribute(k_spmv_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, panel_smem(kPanelMaxW)));
        attr_set = true;
    }
    PanelArgs a;
    a.skip = skip;
    a.P = Q.P;
    a.Bk = Q.Bk;
    a.W = Q.W;
    a.nlines = Q.nlines;
    a.ngather = Q.ngather;
    a.ppt = Q.ppt.p;
    a.blk = Q.blk.p;
    a.idx = Q.idx16.p;
    a.val = rows ? S.val.p : S.cscval.p;
    a.x = x;
    a.part = Q.part.p;
    a.itembase = Q.itembase.p;
    a.nlong = Q.nlong.p;
    a.elen = Q.elen.p;
    a.eout = Q.eout.p;
    a.chrows = Q.chrows.p;
    a.choff = Q.choff.p;
    a.eidx = Q.eidx.p;
    a.eval = ctx->panel_ell ? Q.eval.p : nullptr;
    a.ahead = ctx->panel_ahead;
#ifdef REGOT_PANEL_TIMING
    static long dbg_count = 0;
    if (ctx->panel_ahead == 7777 || ctx->panel_ahead == 7778) a.ahead = (++dbg_count % 400) < 2 ? 7777 : 0;
    static const bool fake = std::getenv("REGOT_PANEL_FAKE") != nullptr;
    a.fake = fake ? std::atoi(std::getenv("REGOT_PANEL_FAKE")) : 0;
#endif
    {
        ProfScope prof(ctx, st, 4);
        k_spmv_panel<<<Q.P * Q.Bk, kPanelThreads, panel_smem(Q.W, ctx->panel_ell != 0), st>>>(a);
        if (combine) {  // else the consumer adds the per-panel partials itself (one kernel and one pass over the vector less)
            const int g = (int)std::max<long>(1, std::min<long>(((long)Q.nlines + 127) / 128, 8L * ctx->sm_count));
            k_panel_combine<kEpi><<<g, 128, 0, st>>>(Q.nlines, Q.P, Q.part.p, ctx->panel_ell ? Q.itembase.p : nullptr, Q.multi.p, rows ? S.dA.p : nullptr,
                                                     y, skip);
        }
    }
    RG_CUDA(cudaGetLastError());
    ctx->launches += combine ? 2 : 1;
}

static bool use_panel_spmv(const regot_ctx* ctx, const regot_sparse& S, int nrhs)
{
    if (nrhs > 2 || ctx->panel_spmv == 0 || S.nnz == 0 || S.m < 2) return false;
    if (ctx->panel_spmv > 0) return true;
    return S.nnz >= (1 << 19);  // below that the gather-through-L2 kernel is not bandwidth-bound
}

// ---- K5, multi-kernel form: Jacobi-PCG on the Schur complement of the alpha block ------------------
// Same algorithm as the persistent kernel (k5_pcg.cu) -- S x_b = r_b - B' D1^-1 r_a, S = D2 - B' D1^-1 B,
// x_a = D1^-1 (r_a - B x_b) -- as a sequence of kernels: the path for problems whose iterated vector does
// not fit in shared memory (the two half mat-vecs run at 32 warps / SM, which is what a latency-bound
// gather wants at that size) and for row-sharded runs: alpha-space quantities and the rows of B are
// local, beta-space vectors are replicated, so the only collective per iteration is ONE allreduce of
// the m-1 partial sums B' t (every rank then takes identical decisions from identical dot products).
// Single-reduction recurrences (Chronopoulos-Gear), as in the persistent kernels: z = D2^-1 r, w = S z,
// gamma = r'z, delta = z'w; beta = gamma / gamma_old, alpha = gamma / (delta - beta gamma / alpha_old);
// p = z + beta p, s = w + beta s, x += alpha p, r -= alpha s.  One iteration = rows half (t = D1^-1 B z) | columns
// half (u = B' t, all-reduced over row blocks) | k_schur_w (w = D2 z - u, the two dot products; the last CTA to finish
// turns them into alpha, beta and the convergence flags) | k_schur_step (the five vector updates).  Every kernel
// returns at once when the all-done flag is set, so the host enqueues iterations in bursts and looks at the flags
// only between bursts: an iteration past convergence costs five empty launches, not a pass over the matrix.
// scalars (device), per system k: gamma_old, alpha_old, gamma0 (the FULL system's r' D^-1 r: the meaning of rtol is
// unchanged), alpha, beta, done, iterations, g0a / g0b (the two halves of gamma0), then the global flags
constexpr int kScalGammaOld = 0 * kMaxRhs;
constexpr int kScalAlphaOld = 1 * kMaxRhs;
constexpr int kScalGamma0 = 2 * kMaxRhs;
constexpr int kScalAlpha = 3 * kMaxRhs;
constexpr int kScalBeta = 4 * kMaxRhs;
constexpr int kScalDone = 5 * kMaxRhs;   // 0 / 1
constexpr int kScalIters = 6 * kMaxRhs;  // iterations taken by each system
constexpr int kScalG0a = 7 * kMaxRhs;    // alpha-block part of gamma0 (summed over ranks)
constexpr int kScalG0b = 8 * kMaxRhs;    // beta-block part of gamma0
constexpr int kScalDots = 9 * kMaxRhs;   // 2 kMaxRhs: gamma, delta of the current iteration
constexpr int kScalBreak = 11 * kMaxRhs;      // breakdown flag
constexpr int kScalAllDone = 11 * kMaxRhs + 1;  // every system done, or breakdown, or the iteration limit: nothing left to do
constexpr int kScalIt = 11 * kMaxRhs + 2;       // iterations started
constexpr int kScalStepIt = 11 * kMaxRhs + 3;   // the iteration whose alpha / beta are waiting for their step (0: none)
constexpr int kScalCount = 11 * kMaxRhs + 4;
constexpr int kCgThreads = 256;

struct CgVecs {
    int nloc, mfree, nrhs, max_iter, n_parts;
    double tol2;
    // all interleaved 4 doubles per index (entry 3 is padding)
    double *ta;                           // alpha space: t = D1^-1 (...)
    double *ub, *xb, *rb, *pb, *sb, *zb;  // beta space: u = B' t, x, r, p, s = S p, z = D2^-1 r
    const int* part_itembase;             // ELL stream: first item of every (panel, column) piece; else null
    const unsigned char* part_multi;      // ELL stream: per column, whether any of its pieces has several items
    const double* part;                   // panel mat-vec on one GPU: u = sum of n_parts per-panel partials (mfree x 2 each); else null
    const double *dA, *dB;
    const double* mB;  // Jacobi preconditioner of the Schur complement (its diagonal)
    double* scal;
    double* partials;
    unsigned int* ticket;
};

// block partials -> global partials; the last CTA to arrive sums them in CTA order into out[0..NV) and returns true
template <int NV>
__device__ __forceinline__ bool two_stage_sum(double (&acc)[NV], double* scratch, double* partials, unsigned int* ticket, double* out)
{
    block_sum<NV>(acc, scratch);
    if (threadIdx.x == 0)
        for (int k = 0; k < NV; ++k) partials[(size_t)blockIdx.x * NV + k] = acc[k];
    __shared__ bool is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!is_last) return false;
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
    __syncthreads();
    return true;
}

// t = D1^-1 r_a and the alpha-block part of r' D^-1 r
__global__ void __launch_bounds__(kCgThreads) k_schur_init_a(const CgVecs v, const double* const* rhs_a)
{
    __shared__ double scratch[kMaxRhs * (kCgThreads / 32)];
    double acc[kMaxRhs] = {0.0, 0.0, 0.0};
    const int stride = gridDim.x * blockDim.x;
    for (int k = 0; k < v.nrhs; ++k)
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < v.nloc; i += stride) {
            const double r = rhs_a[k][i], t = r / v.dA[i];
            v.ta[(size_t)i * 4 + k] = t;
            acc[k] += r * t;
        }
    two_stage_sum<kMaxRhs>(acc, scratch, v.partials, v.ticket, v.scal + kScalG0a);
}

// u of system k at column j: the all-reduced vector, or (panel mat-vec on one GPU) the sum of the per-panel partials
__device__ __forceinline__ double schur_u(const CgVecs& v, int j, int k)
{
    if (v.part == nullptr || k >= 2) return v.ub[(size_t)j * 4 + k];
    const double2 u2 = panel_line_sum2(v.part, v.part_itembase, v.part_multi, v.mfree, v.n_parts, j);
    return k ? u2.y : u2.x;
}

// set-up: c = r_b - u (u = B' t summed over ranks): r = c, z = D2^-1 c, x = p = s = 0; gamma = r'z; beta part of
// gamma0; the last CTA decides which systems need iterations at all
__global__ void __launch_bounds__(kCgThreads) k_schur_init_b(const CgVecs v, const double* const* rhs_b)
{
    __shared__ double scratch[2 * kMaxRhs * (kCgThreads / 32)];
    double acc[2 * kMaxRhs] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    const int stride = gridDim.x * blockDim.x;
    for (int k = 0; k < v.nrhs; ++k)
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < v.mfree; j += stride) {
            const double d = v.dB[j], rb = rhs_b[k][j];
            const double c = rb - schur_u(v, j, k), z = c / v.mB[j];
            const size_t o = (size_t)j * 4 + k;
            v.rb[o] = c;
            v.zb[o] = z;
            v.xb[o] = 0.0;
            v.pb[o] = 0.0;
            v.sb[o] = 0.0;
            acc[k] += c * z;
            acc[kMaxRhs + k] += rb * (rb / v.mB[j]);  // the stopping rule's norm: the preconditioner's
        }
    __shared__ double out6[2 * kMaxRhs];
    if (!two_stage_sum<2 * kMaxRhs>(acc, scratch, v.partials, v.ticket, out6)) return;
    if (threadIdx.x == 0) {
        bool all = true;
        for (int k = 0; k < kMaxRhs; ++k) {
            const double gamma = out6[k], gamma0 = v.scal[kScalG0a + k] + out6[kMaxRhs + k];
            v.scal[kScalG0b + k] = out6[kMaxRhs + k];
            v.scal[kScalGamma0 + k] = gamma0;
            v.scal[kScalGammaOld + k] = 1.0;
            v.scal[kScalAlphaOld + k] = 1.0;
            const bool done = k >= v.nrhs || gamma0 == 0.0 || !(gamma > v.tol2 * gamma0);
            v.scal[kScalDone + k] = done ? 1.0 : 0.0;
            all = all && done;
        }
        v.scal[kScalAllDone] = all ? 1.0 : 0.0;
    }
}

// w = D2 z - u, gamma = r'z, delta = z'w; the last CTA turns the dot products into this iteration's alpha and beta
// and the flags (a system is done when gamma <= tol^2 gamma0; p'Sp <= 0 is a breakdown: not positive definite)
__global__ void __launch_bounds__(kCgThreads) k_schur_w(const CgVecs v)
{
    if (v.scal[kScalAllDone] != 0.0) return;
    __shared__ double scratch[2 * kMaxRhs * (kCgThreads / 32)];
    double acc[2 * kMaxRhs] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    const int stride = gridDim.x * blockDim.x;
    bool live[kMaxRhs];
    for (int k = 0; k < kMaxRhs; ++k) live[k] = k < v.nrhs && v.scal[kScalDone + k] == 0.0;
    // one column per thread and trip, all systems at once: 16-byte loads, the per-panel partials of both systems in one
    // go; every accumulator still adds its columns in ascending order
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < v.mfree; j += stride) {
        const size_t o = (size_t)j * 4;
        double u[kMaxRhs], z[kMaxRhs], r[kMaxRhs];
        if (v.part != nullptr) {
            const double2 u2 = panel_line_sum2(v.part, v.part_itembase, v.part_multi, v.mfree, v.n_parts, j);
            u[0] = u2.x;
            u[1] = u2.y;
            u[2] = live[2] ? v.ub[o + 2] : 0.0;
        } else {
            const double2 u2 = *reinterpret_cast<const double2*>(v.ub + o);
            u[0] = u2.x;
            u[1] = u2.y;
            u[2] = live[2] ? v.ub[o + 2] : 0.0;
        }
        const double2 z2 = *reinterpret_cast<const double2*>(v.zb + o), r2 = *reinterpret_cast<const double2*>(v.rb + o);
        z[0] = z2.x;
        z[1] = z2.y;
        z[2] = live[2] ? v.zb[o + 2] : 0.0;
        r[0] = r2.x;
        r[1] = r2.y;
        r[2] = live[2] ? v.rb[o + 2] : 0.0;
        const double d = v.dB[j];
#pragma unroll
        for (int k = 0; k < kMaxRhs; ++k) {
            if (!live[k]) continue;
            const double w = d * z[k] - u[k];
            v.ub[o + k] = w;  // u is not needed any more: w takes its place
            acc[k] += r[k] * z[k];
            acc[kMaxRhs + k] += z[k] * w;
        }
    }
    if (!two_stage_sum<2 * kMaxRhs>(acc, scratch, v.partials, v.ticket, v.scal + kScalDots)) return;
    if (threadIdx.x == 0) {
        const int it = (int)v.scal[kScalIt];
        bool all = true, broke = false;
        for (int k = 0; k < v.nrhs; ++k) {
            v.scal[kScalAlpha + k] = v.scal[kScalBeta + k] = 0.0;
            if (v.scal[kScalDone + k] != 0.0) continue;
            const double gamma = v.scal[kScalDots + k], delta = v.scal[kScalDots + kMaxRhs + k];
            if (it > 0 && !(gamma > v.tol2 * v.scal[kScalGamma0 + k])) {
                v.scal[kScalDone + k] = 1.0;
                continue;
            }
            const double beta = it == 0 ? 0.0 : gamma / v.scal[kScalGammaOld + k];
            const double denom = delta - beta * gamma / v.scal[kScalAlphaOld + k];  // = p'Sp
            if (!(denom > 0.0)) broke = true;
            const double alpha = gamma / denom;
            v.scal[kScalAlpha + k] = alpha;
            v.scal[kScalBeta + k] = beta;
            v.scal[kScalGammaOld + k] = gamma;
            v.scal[kScalAlphaOld + k] = alpha;
            v.scal[kScalIters + k] += 1.0;
            all = false;
        }
        v.scal[kScalIt] = (double)(it + 1);
        if (broke) v.scal[kScalBreak] = 1.0;
        if (all || broke || it + 1 >= v.max_iter) v.scal[kScalAllDone] = 1.0;
        // the step below runs for the systems that got an alpha in this very iteration, unless it broke down
        v.scal[kScalStepIt] = (all || broke) ? 0.0 : (double)(it + 1);
    }
}

// p = z + beta p, s = w + beta s, x += alpha p, r -= alpha s, z = D2^-1 r (a finished system is frozen)
__global__ void __launch_bounds__(kCgThreads) k_schur_step(const CgVecs v, int iteration)
{
    if (v.scal[kScalStepIt] != (double)iteration) return;  // this iteration was skipped (the solve had ended) or broke down
    const int stride = gridDim.x * blockDim.x;
    double al[kMaxRhs], be[kMaxRhs];
    bool live[kMaxRhs];
    for (int k = 0; k < kMaxRhs; ++k) {
        al[k] = k < v.nrhs ? v.scal[kScalAlpha + k] : 0.0;
        be[k] = k < v.nrhs ? v.scal[kScalBeta + k] : 0.0;
        live[k] = k < v.nrhs && v.scal[kScalDone + k] == 0.0 && al[k] != 0.0;
    }
    // one column per thread and trip: systems 0 and 1 as 16-byte vectors, system 2 (stand-alone compute_direction) scalar
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < v.mfree; j += stride) {
        const size_t o = (size_t)j * 4;
        const double mj = v.mB[j];
        if (live[0] || live[1]) {
            double2 z = *reinterpret_cast<const double2*>(v.zb + o), pp = *reinterpret_cast<const double2*>(v.pb + o);
            double2 w = *reinterpret_cast<const double2*>(v.ub + o), ss = *reinterpret_cast<const double2*>(v.sb + o);
            double2 r = *reinterpret_cast<const double2*>(v.rb + o), x = *reinterpret_cast<const double2*>(v.xb + o);
            if (live[0]) {
                pp.x = z.x + be[0] * pp.x;
                ss.x = w.x + be[0] * ss.x;
                x.x += al[0] * pp.x;
                r.x = r.x - al[0] * ss.x;
                z.x = r.x / mj;
            }
            if (live[1]) {
                pp.y = z.y + be[1] * pp.y;
                ss.y = w.y + be[1] * ss.y;
                x.y += al[1] * pp.y;
                r.y = r.y - al[1] * ss.y;
                z.y = r.y / mj;
            }
            *reinterpret_cast<double2*>(v.pb + o) = pp;
            *reinterpret_cast<double2*>(v.sb + o) = ss;
            *reinterpret_cast<double2*>(v.xb + o) = x;
            *reinterpret_cast<double2*>(v.rb + o) = r;
            *reinterpret_cast<double2*>(v.zb + o) = z;
        }
        if (live[2]) {
            const size_t q = o + 2;
            const double pn = v.zb[q] + be[2] * v.pb[q], sn = v.ub[q] + be[2] * v.sb[q];
            const double rn = v.rb[q] - al[2] * sn;
            v.pb[q] = pn;
            v.sb[q] = sn;
            v.xb[q] += al[2] * pn;
            v.rb[q] = rn;
            v.zb[q] = rn / mj;
        }
    }
}

// x_a = D1^-1 r_a - t (t = D1^-1 B x_b); x_b out, gauge entry zeroed
__global__ void __launch_bounds__(kCgThreads) k_schur_final(const CgVecs v, const double* const* rhs_a, double* const* sol_a,
                                                            double* const* sol_b)
{
    const int stride = gridDim.x * blockDim.x;
    for (int k = 0; k < v.nrhs; ++k) {
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < v.nloc; i += stride)
            sol_a[k][i] = rhs_a[k][i] / v.dA[i] - v.ta[(size_t)i * 4 + k];
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= v.mfree; j += stride)
            sol_b[k][j] = j < v.mfree ? v.xb[(size_t)j * 4 + k] : 0.0;
    }
}

static int pcg_schur_multikernel(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, SparseWS& ws, const regot_sparse& S,
                                 int nrhs, const DVec* const* rhs, DVec* const* sol, double rtol, int max_iter)
{
    const int nloc = (int)S.nloc, mfree = std::max((int)S.m - 1, 0);
    const size_t la = 4 * (size_t)std::max(nloc, 1), lb = 4 * (size_t)std::max(mfree, 1);
    // layout of ws.cg: t | u (then w) | x | r | p | s | z, interleaved x4
    ws.cg.ensure(la + 6 * lb + 16);
    ws.cg_scal.ensure(kScalCount + 8 * kMaxRhs);
    ws.cg_partials.ensure((size_t)(2 * ctx->sm_count + 8) * 2 * kMaxRhs);
    if (!ws.cg_ticket.p) {
        ws.cg_ticket.ensure(1);
        RG_CUDA(cudaMemsetAsync(ws.cg_ticket.p, 0, sizeof(unsigned int), st));
    }
    if (!ws.h_cg) RG_CUDA(cudaMallocHost((void**)&ws.h_cg, sizeof(double) * 4096));
    RG_CUDA(cudaMemsetAsync(ws.cg_scal.p, 0, sizeof(double) * (kScalCount + 8 * kMaxRhs), st));

    const bool panel = use_panel_spmv(ctx, S, nrhs);
    CgVecs v;
    v.nloc = nloc;
    v.mfree = mfree;
    v.nrhs = nrhs;
    v.max_iter = max_iter;
    v.tol2 = rtol * rtol;
    double* base = ws.cg.p;
    v.ta = base;
    v.ub = base + la;
    v.xb = v.ub + lb;
    v.rb = v.xb + lb;
    v.pb = v.rb + lb;
    v.sb = v.pb + lb;
    v.zb = v.sb + lb;
    // the padding entries are gathered (and multiplied into an unused accumulator): keep them finite
    RG_CUDA(cudaMemsetAsync(base, 0, sizeof(double) * (la + 6 * lb), st));
    v.dA = S.dA.p;
    v.dB = S.dB.p;
    v.mB = S.dS.p;
    v.scal = ws.cg_scal.p;
    v.partials = ws.cg_partials.p;
    v.ticket = ws.cg_ticket.p;
    v.part = nullptr;
    v.part_itembase = nullptr;
    v.part_multi = nullptr;
    v.n_parts = 0;

    // pointer tables (rhs_a | rhs_b | sol_a | sol_b) live behind the scalars on the device
    for (int k = 0; k < nrhs; ++k) sol[k]->ensure(S.nloc, S.m);
    const void* h_ptrs[4 * kMaxRhs];
    for (int k = 0; k < kMaxRhs; ++k) {
        const int kk = k < nrhs ? k : 0;
        h_ptrs[k] = rhs[kk]->a.p;
        h_ptrs[kMaxRhs + k] = rhs[kk]->b.p;
        h_ptrs[2 * kMaxRhs + k] = sol[kk]->a.p;
        h_ptrs[3 * kMaxRhs + k] = sol[kk]->b.p;
    }
    void** d_ptrs = reinterpret_cast<void**>(ws.cg_scal.p + kScalCount);
    RG_CUDA(cudaMemcpyAsync((void*)d_ptrs, h_ptrs, sizeof(h_ptrs), cudaMemcpyHostToDevice, st));
    const double* const* d_rhs_a = reinterpret_cast<const double* const*>(d_ptrs);
    const double* const* d_rhs_b = reinterpret_cast<const double* const*>(d_ptrs + kMaxRhs);
    double* const* d_sol_a = reinterpret_cast<double* const*>(d_ptrs + 2 * kMaxRhs);
    double* const* d_sol_b = reinterpret_cast<double* const*>(d_ptrs + 3 * kMaxRhs);

    const int grid_a = (int)std::max<long>(1, std::min<long>((nloc + kCgThreads - 1) / kCgThreads, 2L * ctx->sm_count));
    const int grid_b = (int)std::max<long>(1, std::min<long>((mfree + kCgThreads - 1) / kCgThreads, 2L * ctx->sm_count));
    const double* skip = ws.cg_scal.p + kScalAllDone;
    // t = D1^-1 B x for a beta-space vector x
    auto half_rows = [&](const double* xb, const double* skip_flag) {
        if (panel) launch_spmv_panel<kEpiRowsScaled>(ctx, st, ws, S, xb, v.ta, skip_flag, true);
        else launch_spmv<kEpiRowsScaled>(ctx, st, S, nrhs, nullptr, xb, v.ta, nullptr, kInterleaved4, kInterleaved4, skip_flag);
    };
    // u = B' t, summed over the row blocks; on one GPU the panel form leaves its per-panel partials for the consumer
    auto half_cols = [&](const double* skip_flag) {
        if (panel) launch_spmv_panel<kEpiColsPlain>(ctx, st, ws, S, v.ta, v.ub, skip_flag, ctx->sharded);
        else launch_spmv<kEpiColsPlain>(ctx, st, S, nrhs, v.ta, nullptr, nullptr, v.ub, kInterleaved4, kInterleaved4, skip_flag);
        if (ctx->sharded) allreduce_sum(ctx, comm, v.ub, 4 * (size_t)mfree, st);
    };
    if (panel) {
        panel_refresh_values(ctx, st, ws, S, true);
        panel_refresh_values(ctx, st, ws, S, false);
    }
    if (panel && !ctx->sharded) {
        build_panel_plan(ctx, st, ws, S, false);
        v.part = S.panel_cols.part.p;
        v.part_itembase = ctx->panel_ell ? S.panel_cols.itembase.p : nullptr;
        v.part_multi = S.panel_cols.multi.p;
        v.n_parts = S.panel_cols.P;
    }

    k_schur_init_a<<<grid_a, kCgThreads, 0, st>>>(v, d_rhs_a);
    RG_CUDA(cudaGetLastError());
    if (ctx->sharded) allreduce_sum(ctx, comm, ws.cg_scal.p + kScalG0a, kMaxRhs, st);
    half_cols(nullptr);
    k_schur_init_b<<<grid_b, kCgThreads, 0, st>>>(v, d_rhs_b);
    RG_CUDA(cudaGetLastError());
    ctx->launches += 2;

    bool finished = false, broke = false;
    auto poll = [&]() {
        RG_CUDA(cudaMemcpyAsync(ws.h_cg, ws.cg_scal.p, sizeof(double) * kScalCount, cudaMemcpyDeviceToHost, st));
        RG_CUDA(cudaStreamSynchronize(st));
        broke = ws.h_cg[kScalBreak] != 0.0;
        finished = ws.h_cg[kScalAllDone] != 0.0;
    };
    poll();  // a right-hand side that is already solved takes no iteration
    // sharded runs enqueue a collective per iteration, which no rank may skip on its own: there the flags are identical on
    // every rank (replicated beta-space arithmetic), so skipping is consistent, but the collective itself is always issued
    int burst = 8;
    for (int it = 0; it < max_iter && !finished && !broke;) {
        const int n = std::min(burst, max_iter - it);
        for (int b = 0; b < n; ++b, ++it) {
            half_rows(v.zb, skip);  // t = D1^-1 B z
            half_cols(skip);        // u = B' t
            k_schur_w<<<grid_b, kCgThreads, 0, st>>>(v);
            k_schur_step<<<grid_b, kCgThreads, 0, st>>>(v, it + 1);
            RG_CUDA(cudaGetLastError());
            ctx->launches += 2;
        }
        poll();
        burst = std::min(32, burst * 2);  // long solves look at the flags less often
    }
    if (broke) return -1;
    int iters = 0;  // report the slowest system's exact count
    for (int k = 0; k < nrhs; ++k) iters = std::max(iters, (int)ws.h_cg[kScalIters + k]);
    half_rows(v.xb, nullptr);  // t = D1^-1 B x_b
    k_schur_final<<<std::max(grid_a, grid_b), kCgThreads, 0, st>>>(v, d_rhs_a, d_sol_a, d_sol_b);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
    return iters;
}

// ---- the Jacobi preconditioner: the diagonal of the Schur complement itself -----------------------------------------
// S = D2 - B' D1^-1 B.  D2 alone is a poor stand-in for diag(S) once the plan concentrates: the pattern then carries most
// of a column's mass, B_ij^2 / D1_i nearly cancels D2_j, and diag(S)_j / D2_j ranges over three orders of magnitude
// (measured on Gaussian-mixture clouds: 7e-4 .. 0.95), which is exactly the scaling Jacobi is there to remove: 129 -> 56
// and 165 -> 43 PCG iterations on a 700 x 700 instance, config D 4919 -> see DESIGN.md.  One pass over the CSC copy per
// solve (the values change between solves); sharded runs add the ranks' partial column sums.  A difference lost to
// rounding (below 1e-10 D2_j: the pattern carries the whole column) falls back to that floor: any positive diagonal
// is a valid preconditioner.  The stopping rule measures the right-hand side in the same norm as the residual
// (gamma0 = r_a' D1^-1 r_a + r_b' diag(S)^-1 r_b): keeping D2 there made the test stricter than rtol says and cost one or
// two iterations per solve at the paper's sizes.
__device__ __forceinline__ double schur_diag_guard(double d2, double s)
{
    const double x = d2 - s, lo = 1e-10 * d2;
    return x > lo ? x : lo;
}
constexpr int kDiagThreads = 256, kDiagWarps = kDiagThreads / 32;
constexpr int kDiagLong = 4096;  // columns above this many entries are left to k_schur_diag_long (column 0 of Omega* is full)
constexpr int kDiagLongThreads = 256;
// sum over e = first, first + step, ... < end of cscval[e]^2 / dA[cscrow[e]], eight entries in flight: the indices and values
// of a batch are loaded first, then the gathered diagonal entries, then the arithmetic (a plain loop waits for every
// dependent pair of loads in turn: 35 us for the 1,600 entries of a full column on one warp)
__device__ __forceinline__ double schur_diag_strided(const int* __restrict__ cscrow, const double* __restrict__ cscval,
                                                     const double* __restrict__ dA, int first, int end, int step)
{
    double s = 0.0;
    for (int e0 = first; e0 < end; e0 += 8 * step) {
        int r[8];
        double v[8], d[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * step;
            const bool ok = e < end;
            r[u] = ok ? __ldg(cscrow + e) : -1;
            v[u] = ok ? __ldg(cscval + e) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) d[u] = r[u] >= 0 ? __ldg(dA + r[u]) : 1.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u] * (v[u] / d[u]);
    }
    return s;
}
// a warp per column (lanes strided, butterfly: a fixed order); long columns are listed for the kernel below
__global__ void __launch_bounds__(kDiagThreads) k_schur_diag(int mfree, const int* __restrict__ cscptr, const int* __restrict__ cscrow,
                                                             const double* __restrict__ cscval, const double* __restrict__ dA,
                                                             const double* __restrict__ dB, double* __restrict__ out, int finalize,
                                                             int* __restrict__ long_list, int* __restrict__ n_long)
{
    const int lane = threadIdx.x & 31, nw = (gridDim.x * blockDim.x) >> 5;
    for (int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < mfree; j += nw) {
        const int beg = __ldg(cscptr + j), end = __ldg(cscptr + j + 1);
        if (end - beg > kDiagLong) {
            if (lane == 0) long_list[atomicAdd(n_long, 1)] = j;  // the order of the list does not matter
            continue;
        }
        double s = schur_diag_strided(cscrow, cscval, dA, beg + lane, end, 32);
        s = warp_sum(s);
        if (lane == 0) out[j] = finalize ? schur_diag_guard(__ldg(dB + j), s) : s;
    }
}
// a CTA per long column: threads strided, butterfly per warp, warps in order
__global__ void __launch_bounds__(kDiagLongThreads) k_schur_diag_long(const int* __restrict__ cscptr, const int* __restrict__ cscrow,
                                                                      const double* __restrict__ cscval, const double* __restrict__ dA,
                                                                      const double* __restrict__ dB, double* __restrict__ out,
                                                                      int finalize, const int* __restrict__ long_list,
                                                                      const int* __restrict__ n_long)
{
    __shared__ double wsum[kDiagLongThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, n = *n_long;
    for (int q = blockIdx.x; q < n; q += gridDim.x) {
        const int j = long_list[q], beg = __ldg(cscptr + j), end = __ldg(cscptr + j + 1);
        double s = schur_diag_strided(cscrow, cscval, dA, beg + tid, end, kDiagLongThreads);
        s = warp_sum(s);
        if (lane == 0) wsum[warp] = s;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < kDiagLongThreads / 32; ++w) t += wsum[w];
            out[j] = finalize ? schur_diag_guard(__ldg(dB + j), t) : t;
        }
        __syncthreads();
    }
}
__global__ void k_schur_diag_fin(int mfree, const double* __restrict__ dB, double* __restrict__ io)
{
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < mfree; j += gridDim.x * blockDim.x) io[j] = schur_diag_guard(dB[j], io[j]);
}
static void compute_schur_diag(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, const regot_sparse& S)
{
    const int mfree = std::max((int)S.m - 1, 0);
    S.dS.ensure((size_t)std::max(mfree, 1));
    if (mfree == 0) return;
    if (!ctx->schur_diag) {
        RG_CUDA(cudaMemcpyAsync(S.dS.p, S.dB.p, sizeof(double) * (size_t)mfree, cudaMemcpyDeviceToDevice, st));
        return;
    }
    const int grid = (int)std::max<long>(1, std::min<long>(((long)mfree + kDiagWarps - 1) / kDiagWarps, 64L * ctx->sm_count));
    S.diag_long.ensure((size_t)mfree + 1);  // entry 0: the count; then the list
    const int fin = ctx->sharded ? 0 : 1;
    // a column has at most nloc entries: with nloc <= kDiagLong no column is long, and the list, its reset and the second
    // kernel are not needed (the paper's sizes: one launch per solve)
    const bool may_be_long = S.nloc > kDiagLong;
    if (may_be_long) RG_CUDA(cudaMemsetAsync(S.diag_long.p, 0, sizeof(int), st));
    k_schur_diag<<<grid, kDiagThreads, 0, st>>>(mfree, S.cscptr.p, S.cscrow.p, S.cscval.p, S.dA.p, S.dB.p, S.dS.p, fin, S.diag_long.p + 1,
                                               S.diag_long.p);
    if (may_be_long)
        k_schur_diag_long<<<8 * ctx->sm_count, kDiagLongThreads, 0, st>>>(S.cscptr.p, S.cscrow.p, S.cscval.p, S.dA.p, S.dB.p, S.dS.p, fin,
                                                                         S.diag_long.p + 1, S.diag_long.p);
    RG_CUDA(cudaGetLastError());
    ctx->launches += may_be_long ? 2 : 1;
    if (ctx->sharded) {
        allreduce_sum(ctx, comm, S.dS.p, (size_t)mfree, st);
        k_schur_diag_fin<<<(mfree + 255) / 256, 256, 0, st>>>(mfree, S.dB.p, S.dS.p);
        RG_CUDA(cudaGetLastError());
        ++ctx->launches;
    }
}

int sparse_pcg(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, SparseWS& ws, const regot_sparse& S, int nrhs,
               const DVec* const* rhs, DVec* const* sol, double rtol, int max_iter)
{
    if (nrhs < 1 || nrhs > kMaxRhs) raise(REGOT_E_VALIDATION, "pcg: bad number of right-hand sides");
    compute_schur_diag(ctx, st, comm, S);
    // one GPU: the block-resident kernel when every block of the pattern fits in shared memory, else the persistent
    // kernel that streams the matrix (iterated vectors in shared memory), else kernel by kernel
    if (!ctx->sharded && !ctx->force_multikernel_pcg && S.blocks.fits)
        return pcg_schur_blocks(ctx, st, ws, S, nrhs, rhs, sol, rtol, max_iter);
    if (!ctx->sharded && !ctx->force_multikernel_pcg && S.pcg.fits)
        return pcg_schur_persistent(ctx, st, ws, S, nrhs, rhs, sol, rtol, max_iter);
    return pcg_schur_multikernel(ctx, st, comm, ws, S, nrhs, rhs, sol, rtol, max_iter);
}

}  // namespace rg
