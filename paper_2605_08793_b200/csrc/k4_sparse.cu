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
    A.add_diag_b = (ctx->world == 1 || ctx->rank == 0) ? 1 : 0;
    return A;
}

// one (part of a) mat-vec: kEpiFull over all lines, or one of the two halves of the Schur mat-vec
template <int kEpi>
static void launch_spmv(regot_ctx* ctx, cudaStream_t st, const regot_sparse& S, int nrhs, const double* va,
                        const double* vb, double* ya, double* yb, long sa, long sb)
{
    SpmvParams p;
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
    if (ctx->world > 1) {
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
constexpr int kPanelGroupMax = 256;     // pieces up to this many entries: 8 lanes
constexpr int kPanelWarpMax = 8192;     // up to this many: one warp; longer: the whole CTA
constexpr int kPanelDeferCap = 2048;    // deferred pieces per CTA kept in the shared-memory lists
constexpr int kPanelLineCost = 24;      // work of a piece beyond its entries (pointer loads, reduction), in entries

struct PanelArgs {
    int P, Bk, W, nlines, ngather;
    const int* ppt;
    const int* blk;
    const int* idx;     // col (row phase) or cscrow (column phase)
    const double* val;  // val or cscval
    const double* x;    // gathered vector, interleaved 4 doubles per index
    double* part;       // P x nlines x 2
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

// lanes stride over [beg, end) with kLanes lanes and 8 entries in flight per lane; gathers from the staged panel
template <int kLanes>
__device__ __forceinline__ void panel_dot(int beg, int end, int gl, const int* __restrict__ idx, const double* __restrict__ val,
                                          uint32_t vec, int col0, double& a0, double& a1)
{
    for (int t = beg + gl; t < end; t += kLanes * 8) {
        int c[8];
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int tt = t + kLanes * u;
            const bool ok = tt < end;
            c[u] = ok ? __ldg(idx + tt) : col0;
            v[u] = ok ? __ldg(val + tt) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double2 g = lds_f64x2(vec + (uint32_t)(c[u] - col0) * 16u);
            a0 = __fma_rn(v[u], g.x, a0);
            a1 = __fma_rn(v[u], g.y, a1);
        }
    }
}

__global__ void __launch_bounds__(kPanelThreads, 1) k_spmv_panel(const PanelArgs a)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int p = blockIdx.x / a.Bk, b = blockIdx.x - p * a.Bk;
    const int col0 = p * a.W, wp = min(a.W, a.ngather - col0);
    const uint32_t vec = smem_u32(smem);
    int* defer_w = reinterpret_cast<int*>(smem + (size_t)a.W * 16);  // pieces for a warp
    int* defer_c = defer_w + kPanelDeferCap;                         // pieces for the CTA
    double* wpart = reinterpret_cast<double*>(defer_c + kPanelDeferCap);  // kPanelWarps x 2
    __shared__ int n_defer_w, n_defer_c;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) n_defer_w = n_defer_c = 0;
    // stage the panel: entries (x[4 j], x[4 j + 1]) of the interleaved vector
    for (int j = tid; j < wp; j += kPanelThreads) {
        const double2 g = __ldcg(reinterpret_cast<const double2*>(a.x + (size_t)(col0 + j) * 4));
        asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(vec + (uint32_t)j * 16u), "d"(g.x), "d"(g.y) : "memory");
    }
    __syncthreads();
    const int l0 = a.blk[p * (a.Bk + 1) + b], l1 = a.blk[p * (a.Bk + 1) + b + 1];
    const size_t pstride = (size_t)(a.P + 1);
    double* const part = a.part + (size_t)p * a.nlines * 2;

    // ---- pass 1: four lines per warp, 8 lanes each; longer pieces are deferred ----
    const int sub = lane >> 3, gl = lane & 7;
    for (int base = l0 + warp * 4; base < l1; base += kPanelWarps * 4) {
        const int l = base + sub;
        int beg = 0, end = 0;
        if (l < l1) {
            beg = __ldg(a.ppt + (size_t)l * pstride + p);
            end = __ldg(a.ppt + (size_t)l * pstride + p + 1);
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
            panel_dot<8>(beg, end, gl, a.idx, a.val, vec, col0, a0, a1);
        }
        // even lanes of a group end with the group's sum of a0, odd lanes with a1 (fixed order)
        const bool odd = lane & 1;
        double c = (odd ? a1 : a0) + shfl_xor_d(odd ? a0 : a1, 1);
        c += shfl_xor_d(c, 2);
        c += shfl_xor_d(c, 4);
        if (l < l1 && len <= kPanelGroupMax && gl < 2) part[(size_t)l * 2 + gl] = c;
    }
    __syncthreads();
    // ---- pass 2: one warp per deferred piece ----
    const int nw_list = min(n_defer_w, kPanelDeferCap), nc_list = min(n_defer_c, kPanelDeferCap);
    const bool overflow = n_defer_w > kPanelDeferCap || n_defer_c > kPanelDeferCap;
    for (int q = warp; q < nw_list; q += kPanelWarps) {
        const int l = defer_w[q];
        const int beg = __ldg(a.ppt + (size_t)l * pstride + p), end = __ldg(a.ppt + (size_t)l * pstride + p + 1);
        double a0 = 0.0, a1 = 0.0;
        panel_dot<32>(beg, end, lane, a.idx, a.val, vec, col0, a0, a1);
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
        panel_dot<kPanelThreads>(beg, end, tid, a.idx, a.val, vec, col0, a0, a1);
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
    // more deferred pieces than the lists hold (never at the sizes this path is meant for): rescan, one warp each
    if (overflow) {
        for (int l = l0 + warp; l < l1; l += kPanelWarps) {
            const int beg = __ldg(a.ppt + (size_t)l * pstride + p), end = __ldg(a.ppt + (size_t)l * pstride + p + 1);
            if (end - beg <= kPanelGroupMax) continue;
            double a0 = 0.0, a1 = 0.0;
            panel_dot<32>(beg, end, lane, a.idx, a.val, vec, col0, a0, a1);
            a0 = warp_sum(a0);
            a1 = warp_sum(a1);
            if (lane == 0) {
                part[(size_t)l * 2] = a0;
                part[(size_t)l * 2 + 1] = a1;
            }
        }
    }
}

// y_line = sum over panels (panel order) of part[p][line], then the epilogue of the half mat-vec
template <int kEpi>
__global__ void k_panel_combine(int nlines, int P, const double* __restrict__ part, const double* __restrict__ diag,
                                double* __restrict__ y)
{
    const int total = nlines * 2;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < total; q += gridDim.x * blockDim.x) {
        const int l = q >> 1, k = q & 1;
        double s = 0.0;
        for (int p = 0; p < P; ++p) s += part[((size_t)p * nlines + l) * 2 + k];
        y[(size_t)l * 4 + k] = (kEpi == kEpiRowsScaled) ? s / diag[l] : s;
    }
}

static constexpr int panel_smem(int W) { return W * 16 + 2 * kPanelDeferCap * 4 + kPanelWarps * 2 * 8; }

// (re)build the plan of one half for the current pattern; everything stays on the device
static void build_panel_plan(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, const regot_sparse& S, bool rows)
{
    PanelPlan& Q = rows ? S.panel_rows : S.panel_cols;
    if (Q.stamp == S.structure_stamp && Q.P > 0) return;
    const int nloc = (int)S.nloc, mfree = std::max((int)S.m - 1, 0);
    Q.nlines = rows ? nloc : mfree;
    Q.ngather = rows ? mfree : nloc;
    const int wmax = ctx->panel_width > 0 ? std::min(ctx->panel_width, kPanelMaxW) : kPanelMaxW;
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
    const int* ptr = rows ? S.rowptr.p : S.cscptr.p;
    const int* idx = rows ? S.col.p : S.cscrow.p;
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
    Q.stamp = S.structure_stamp;
}

// one half mat-vec in panel form: y (interleaved x4) = epilogue(B x) or epilogue(B' x) for two right-hand sides
template <int kEpi>
static void launch_spmv_panel(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, const regot_sparse& S, const double* x, double* y)
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
    a.P = Q.P;
    a.Bk = Q.Bk;
    a.W = Q.W;
    a.nlines = Q.nlines;
    a.ngather = Q.ngather;
    a.ppt = Q.ppt.p;
    a.blk = Q.blk.p;
    a.idx = rows ? S.col.p : S.cscrow.p;
    a.val = rows ? S.val.p : S.cscval.p;
    a.x = x;
    a.part = Q.part.p;
    {
        ProfScope prof(ctx, st, 4);
        k_spmv_panel<<<Q.P * Q.Bk, kPanelThreads, panel_smem(Q.W), st>>>(a);
        const int g = (int)std::max<long>(1, std::min<long>(((long)Q.nlines * 2 + 255) / 256, 4L * ctx->sm_count));
        k_panel_combine<kEpi><<<g, 256, 0, st>>>(Q.nlines, Q.P, Q.part.p, rows ? S.dA.p : nullptr, y);
    }
    RG_CUDA(cudaGetLastError());
    ctx->launches += 2;
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
// scalars (device), per rhs k: rz[2][k] (double-buffered by iteration parity), pAp[k], rz0[k] (the FULL
// system's r' D^-1 r: the meaning of rtol is unchanged), done[k], breakdown flag, iterations[k], g0a[k]
constexpr int kScalRz = 0;                   // 2 * kMaxRhs
constexpr int kScalPap = 2 * kMaxRhs;        // kMaxRhs
constexpr int kScalRz0 = 3 * kMaxRhs;        // kMaxRhs
constexpr int kScalDone = 4 * kMaxRhs;       // kMaxRhs (0/1)
constexpr int kScalBreak = 5 * kMaxRhs;      // 1: breakdown flag
constexpr int kScalIters = 5 * kMaxRhs + 1;  // kMaxRhs: iterations taken by each system
constexpr int kScalG0a = 6 * kMaxRhs + 1;    // kMaxRhs: alpha-block part of rz0 (summed over ranks)
constexpr int kScalG0b = 7 * kMaxRhs + 1;    // kMaxRhs: beta-block part of rz0
constexpr int kScalCount = 8 * kMaxRhs + 4;
constexpr int kCgThreads = 256;

struct CgVecs {
    int nloc, mfree, nrhs;
    // all interleaved 4 doubles per index (entry 3 is padding)
    double *ta;                      // alpha space: t = D1^-1 (...)
    double *ub, *xb, *rb, *pb, *qb;  // beta space: u = B' t, x, r, p, q = S p
    const double *dA, *dB;
    double* scal;
    double* partials;
    unsigned int* ticket;
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
    two_stage_store<kMaxRhs>(acc, scratch, v.partials, v.ticket, v.scal + kScalG0a);
}

// c = r_b - u (u = B' t summed over ranks): r = c, z = D2^-1 c, p = z, x = 0; rz = r'z; beta part of rz0
__global__ void __launch_bounds__(kCgThreads) k_schur_init_b(const CgVecs v, const double* const* rhs_b)
{
    __shared__ double scratch[2 * kMaxRhs * (kCgThreads / 32)];
    double acc[2 * kMaxRhs] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    const int stride = gridDim.x * blockDim.x;
    for (int k = 0; k < v.nrhs; ++k)
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < v.mfree; j += stride) {
            const double d = v.dB[j], rb = rhs_b[k][j];
            const double c = rb - v.ub[(size_t)j * 4 + k], z = c / d;
            v.rb[(size_t)j * 4 + k] = c;
            v.pb[(size_t)j * 4 + k] = z;
            v.xb[(size_t)j * 4 + k] = 0.0;
            acc[k] += c * z;
            acc[kMaxRhs + k] += rb * (rb / d);
        }
    // rz[0][k] and g0b[k] are not adjacent: two stores through a small staging area
    __shared__ double out6[2 * kMaxRhs];
    block_sum<2 * kMaxRhs>(acc, scratch);
    if (threadIdx.x == 0)
        for (int k = 0; k < 2 * kMaxRhs; ++k) v.partials[(size_t)blockIdx.x * 2 * kMaxRhs + k] = acc[k];
    __shared__ bool is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = (atomicAdd(v.ticket, 1u) == gridDim.x - 1);
    __syncthreads();
    if (is_last) {
        __threadfence();
        if (threadIdx.x < 32) {
            for (int k = 0; k < 2 * kMaxRhs; ++k) {
                double s = 0.0;
                for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) s += v.partials[(size_t)b * 2 * kMaxRhs + k];
                s = warp_sum(s);
                if (threadIdx.x == 0) out6[k] = s;
            }
            if (threadIdx.x == 0) {
                for (int k = 0; k < kMaxRhs; ++k) {
                    v.scal[kScalRz + k] = out6[k];
                    v.scal[kScalG0b + k] = out6[kMaxRhs + k];
                }
                *v.ticket = 0u;
            }
        }
    }
}

// q = D2 p - u, pAp[k] = p_k . q_k
__global__ void __launch_bounds__(kCgThreads) k_schur_q(const CgVecs v)
{
    __shared__ double scratch[kMaxRhs * (kCgThreads / 32)];
    double acc[kMaxRhs] = {0.0, 0.0, 0.0};
    const int stride = gridDim.x * blockDim.x;
    for (int k = 0; k < v.nrhs; ++k)
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < v.mfree; j += stride) {
            const double p = v.pb[(size_t)j * 4 + k];
            const double q = v.dB[j] * p - v.ub[(size_t)j * 4 + k];
            v.qb[(size_t)j * 4 + k] = q;
            acc[k] += p * q;
        }
    two_stage_store<kMaxRhs>(acc, scratch, v.partials, v.ticket, v.scal + kScalPap);
}

// x += a p, r -= a q, rz_new = r . D2^-1 r ; a = rz / pAp (0 once the system is done)
__global__ void __launch_bounds__(kCgThreads) k_schur_update(const CgVecs v, int parity)
{
    __shared__ double scratch[kMaxRhs * (kCgThreads / 32)];
    double acc[kMaxRhs] = {0.0, 0.0, 0.0};
    const int stride = gridDim.x * blockDim.x;
    for (int k = 0; k < v.nrhs; ++k) {
        const double pap = v.scal[kScalPap + k];
        const bool live = v.scal[kScalDone + k] == 0.0 && pap > 0.0;
        const double a = live ? v.scal[kScalRz + parity * kMaxRhs + k] / pap : 0.0;
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < v.mfree; j += stride) {
            v.xb[(size_t)j * 4 + k] += a * v.pb[(size_t)j * 4 + k];
            const double r = v.rb[(size_t)j * 4 + k] - a * v.qb[(size_t)j * 4 + k];
            v.rb[(size_t)j * 4 + k] = r;
            acc[k] += r * (r / v.dB[j]);
        }
    }
    two_stage_store<kMaxRhs>(acc, scratch, v.partials, v.ticket, v.scal + kScalRz + (parity ^ 1) * kMaxRhs);
}

// p = z + b p with b = rz_new / rz
__global__ void __launch_bounds__(kCgThreads) k_schur_direction(const CgVecs v, int parity)
{
    const int stride = gridDim.x * blockDim.x;
    for (int k = 0; k < v.nrhs; ++k) {
        const double rz = v.scal[kScalRz + parity * kMaxRhs + k];
        const double rzn = v.scal[kScalRz + (parity ^ 1) * kMaxRhs + k];
        const bool done = v.scal[kScalDone + k] != 0.0;
        const double b = (!done && rz > 0.0) ? rzn / rz : 0.0;
        if (!done)
            for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < v.mfree; j += stride)
                v.pb[(size_t)j * 4 + k] = v.rb[(size_t)j * 4 + k] / v.dB[j] + b * v.pb[(size_t)j * 4 + k];
    }
}

// single thread: bookkeeping between iterations (runs after k_schur_update)
__global__ void k_cg_flags(double* scal, int nrhs, int parity, double tol2, int first)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int k = 0; k < nrhs; ++k) {
        if (first) {
            const double rz0 = scal[kScalG0a + k] + scal[kScalG0b + k];
            scal[kScalRz0 + k] = rz0;
            scal[kScalDone + k] = (rz0 == 0.0 || !(scal[kScalRz + k] > tol2 * rz0)) ? 1.0 : 0.0;
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
        if (!(rzn > tol2 * scal[kScalRz0 + k])) scal[kScalDone + k] = 1.0;
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
    // layout of ws.cg: t | u | x | r | p | q, interleaved x4
    ws.cg.ensure(la + 5 * lb + 16);
    ws.cg_scal.ensure(kScalCount + 8 * kMaxRhs);
    ws.cg_partials.ensure((size_t)(2 * ctx->sm_count + 8) * 2 * kMaxRhs);
    if (!ws.cg_ticket.p) {
        ws.cg_ticket.ensure(1);
        RG_CUDA(cudaMemsetAsync(ws.cg_ticket.p, 0, sizeof(unsigned int), st));
    }
    if (!ws.h_cg) RG_CUDA(cudaMallocHost((void**)&ws.h_cg, sizeof(double) * 4096));
    RG_CUDA(cudaMemsetAsync(ws.cg_scal.p, 0, sizeof(double) * (kScalCount + 8 * kMaxRhs), st));

    CgVecs v;
    v.nloc = nloc;
    v.mfree = mfree;
    v.nrhs = nrhs;
    double* base = ws.cg.p;
    v.ta = base;
    v.ub = base + la;
    v.xb = v.ub + lb;
    v.rb = v.xb + lb;
    v.pb = v.rb + lb;
    v.qb = v.pb + lb;
    // the padding entries are gathered (and multiplied into an unused accumulator): keep them finite
    RG_CUDA(cudaMemsetAsync(base, 0, sizeof(double) * (la + 5 * lb), st));
    v.dA = S.dA.p;
    v.dB = S.dB.p;
    v.scal = ws.cg_scal.p;
    v.partials = ws.cg_partials.p;
    v.ticket = ws.cg_ticket.p;

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
    const double tol2 = rtol * rtol;
    const bool panel = use_panel_spmv(ctx, S, nrhs);
    // t = D1^-1 B x for a beta-space vector x
    auto half_rows = [&](const double* xb) {
        if (panel) launch_spmv_panel<kEpiRowsScaled>(ctx, st, ws, S, xb, v.ta);
        else launch_spmv<kEpiRowsScaled>(ctx, st, S, nrhs, nullptr, xb, v.ta, nullptr, kInterleaved4, kInterleaved4);
    };
    // u = B' t, summed over the row blocks
    auto half_cols = [&]() {
        if (panel) launch_spmv_panel<kEpiColsPlain>(ctx, st, ws, S, v.ta, v.ub);
        else launch_spmv<kEpiColsPlain>(ctx, st, S, nrhs, v.ta, nullptr, nullptr, v.ub, kInterleaved4, kInterleaved4);
        if (ctx->world > 1) allreduce_sum(ctx, comm, v.ub, 4 * (size_t)mfree, st);
    };

    k_schur_init_a<<<grid_a, kCgThreads, 0, st>>>(v, d_rhs_a);
    RG_CUDA(cudaGetLastError());
    if (ctx->world > 1) allreduce_sum(ctx, comm, ws.cg_scal.p + kScalG0a, kMaxRhs, st);
    half_cols();
    k_schur_init_b<<<grid_b, kCgThreads, 0, st>>>(v, d_rhs_b);
    k_cg_flags<<<1, 32, 0, st>>>(ws.cg_scal.p, nrhs, 0, tol2, 1);
    RG_CUDA(cudaGetLastError());
    ctx->launches += 3;

    const int check_every = 8;
    int it = 0, parity = 0;
    bool finished = false, broke = false;
    auto poll = [&]() {
        RG_CUDA(cudaMemcpyAsync(ws.h_cg, ws.cg_scal.p, sizeof(double) * kScalCount, cudaMemcpyDeviceToHost, st));
        RG_CUDA(cudaStreamSynchronize(st));
        broke = ws.h_cg[kScalBreak] != 0.0;
        finished = true;
        for (int k = 0; k < nrhs; ++k) finished &= ws.h_cg[kScalDone + k] != 0.0;
    };
    poll();  // a right-hand side that is already solved takes no iteration
    while (it < max_iter && !finished && !broke) {
        const int burst = std::min(check_every, max_iter - it);
        for (int b = 0; b < burst; ++b, ++it) {
            half_rows(v.pb);                                                                         // t = D1^-1 B p
            half_cols();                                                                            // u = B' t
            k_schur_q<<<grid_b, kCgThreads, 0, st>>>(v);
            k_schur_update<<<grid_b, kCgThreads, 0, st>>>(v, parity);
            k_cg_flags<<<1, 32, 0, st>>>(ws.cg_scal.p, nrhs, parity, tol2, 0);
            k_schur_direction<<<grid_b, kCgThreads, 0, st>>>(v, parity);
            RG_CUDA(cudaGetLastError());
            ctx->launches += 4;
            parity ^= 1;
        }
        poll();
    }
    if (broke) return -1;
    it = 0;  // report the slowest system's exact count, not the burst-rounded loop count
    for (int k = 0; k < nrhs; ++k) it = std::max(it, (int)ws.h_cg[kScalIters + k]);
    half_rows(v.xb);  // t = D1^-1 B x_b
    k_schur_final<<<std::max(grid_a, grid_b), kCgThreads, 0, st>>>(v, d_rhs_a, d_sol_a, d_sol_b);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
    return it;
}

int sparse_pcg(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, SparseWS& ws, const regot_sparse& S, int nrhs,
               const DVec* const* rhs, DVec* const* sol, double rtol, int max_iter)
{
    if (nrhs < 1 || nrhs > kMaxRhs) raise(REGOT_E_VALIDATION, "pcg: bad number of right-hand sides");
    // one GPU: the block-resident kernel when every block of the pattern fits in shared memory, else the persistent
    // kernel that streams the matrix (iterated vectors in shared memory), else kernel by kernel
    if (ctx->world == 1 && !ctx->force_multikernel_pcg && S.blocks.fits)
        return pcg_schur_blocks(ctx, st, ws, S, nrhs, rhs, sol, rtol, max_iter);
    if (ctx->world == 1 && !ctx->force_multikernel_pcg && S.pcg.fits)
        return pcg_schur_persistent(ctx, st, ws, S, nrhs, rhs, sol, rtol, max_iter);
    return pcg_schur_multikernel(ctx, st, comm, ws, S, nrhs, rhs, sol, rtol, max_iter);
}

}  // namespace rg
