// sparse.hpp -- device representation of A = H_Omega + tau I (sparsity.h:97-195)
// and the scratch of the top-k selection.
//
// A = [ diag(dA)   B      ]    B = T_Omega / eta, nloc x (m-1), stored twice:
//     [ B'         diag(dB) ]   CSR (row-major == the reference's lexicographic
//                               coordinate order) for B v, CSC for B' v.
// The reference's CSC-of-both-triangles layout (sparsity.h:249-289) is produced
// on export only.
#pragma once

#include <functional>
#include "ctx.hpp"

namespace rg {
// Work schedule of the persistent Schur-complement PCG kernel (k5_pcg.cu), built on the host per
// pattern: rows and columns of B cut into warp-sized items (4 short lines / 1 medium line / 1 chunk
// of a long line), dealt to the grid's warps longest-first.  items: kPcgItemInts ints each
// {kind, nE, chunk, slot, first, cnt, -, -, line[4], beg[4], len[4], -...}; wptr: per phase
// (rows, columns) nw + 1 offsets into items.  The kernel keeps the gathered vector in shared memory;
// fits == false (vector too long) sends the solve down the kernel-by-kernel path instead.
constexpr int kPcgWarpsPerCta = 16;
constexpr int kPcgItemInts = 24;
constexpr int kPcgSmemBudget = 227 * 1024;     // dynamic shared memory of the persistent kernel
constexpr int kPcgVecSmemMax = 168 * 1024;     // largest gathered vector (16 B / entry) staged in shared memory
constexpr long kPcgMaxEntriesL2Gather = 4000000;  // one phase gathering through L2: only up to this many entries of B
struct PcgSchedule {
    DevBuf<int> items, wptr;
    mutable DevBuf<double> chunk_part;
    mutable DevBuf<unsigned int> chunk_cnt;
    int grid = 0;  // CTAs the schedule was dealt over: all SMs, or one cluster for a small system
    int nw = 0, n_long = 0, n_long_rows = 0, n_chunks = 0;  // long lines: the row phase's come first
    bool fits = false;                // the persistent kernel takes this pattern (else: kernel by kernel)
    bool stage_rows = false, stage_cols = false;  // which phase's gathered vector is staged in shared memory
    int vec_bytes = 0, desc_cap = 0;  // shared-memory carve-up: vector buffer, descriptors per warp
};
}  // namespace rg

namespace rg {
// Plan of the panel mat-vec (k4_sparse.cu, k_spmv_panel): the gathered vector of one Schur half is cut into P
// panels of W entries that fit in shared memory, the lines (rows or columns of B) of each panel into Bk blocks
// of equal work; CTA (p, b) stages panel p once and processes the pieces of its lines that fall inside it.
struct PanelPlan {
    int P = 0, Bk = 0, W = 0, nlines = 0, ngather = 0;
    unsigned long stamp = 0;  // structure_stamp of the pattern this plan was built for
    DevBuf<int> ppt;          // nlines x (P + 1): first entry of line l at or beyond panel p
    DevBuf<int> blk;          // P x (Bk + 1): line boundaries of the blocks
    DevBuf<unsigned short> idx16;  // per entry of the half's matrix copy: index relative to its panel
    DevBuf<int> cost, scan;   // P x nlines (+1): work per piece and its exclusive prefix sum
    DevBuf<double> part;      // P x nlines x 2: per-panel partial sums of every line (ELL stream: then the sums of the items of cut pieces)
    // ELL stream of the pieces (k4_sparse.cu): every piece cut into items of up to kEllItemMax entries, the items of a
    // CTA sorted by length; a long item is a chunk (entry k at row k / 32, lane k % 32), the others go 8 to a chunk (entry k
    // of item j at row k / 4, lane (k % 4) * 8 + j)
    DevBuf<int> nseg, itembase;     // per piece q = p nlines + l: its items, and their exclusive prefix sum (np + 1)
    DevBuf<unsigned> ekey, ekey2;   // sort keys: (CTA, cap - length)
    DevBuf<int> eid0, eid;          // item ids before / after the sort
    DevBuf<int> item_q;             // piece of every item
    DevBuf<int> nlong;              // per CTA: items above kPanelGroupMax entries (a chunk each)
    DevBuf<unsigned char> multi;    // per line: any piece of several items
    DevBuf<int> elen, ebeg, eout;   // per sorted item: entries, first entry, where its sums go (pairs of part)
    DevBuf<int> chrows, choff;      // per chunk slot: rows of 32 entries, first row
    DevBuf<int> emap;               // per ELL slot: the entry of the matrix copy it holds, or -1
    DevBuf<unsigned short> eidx;    // per ELL slot: panel-relative index
    DevBuf<double> eval;            // per ELL slot: value (rewritten once per solve)
    size_t item_cap = 0;
    int nchunk_slots = 0;
    size_t ell_cap = 0;             // slots allocated
};
}  // namespace rg

namespace rg {
// Plan of the block-resident Schur-complement PCG kernel (k6_pcg_blocks.cu), built on the device per pattern: B
// cut into P x Q blocks (rows dealt round-robin to block rows, columns to block columns), every block laid out
// for one CTA's shared memory -- its rows and its columns as 32-line chunks sorted by length -- in two arenas.
constexpr int kPcgBlocksHdrInts = 16;
constexpr int kPcgBlocksMaxHeavy = 256;  // lines of a block too long for one thread, per copy
struct PcgBlocksPlan {
    bool fits = false;     // every block fits in shared memory: the solve takes this kernel
    bool pending = false;  // built, summary not read yet
    int P = 0, Q = 0, R = 0, C = 0, SR = 0, SC = 0, Lr = 0, Lc = 0, smem = 0;
    int cluster = 0;  // the CTAs of a block row form a thread-block cluster (exchanges in distributed shared memory)
    unsigned long stamp = 0;
    DevBuf<int> cnt, vpos;  // G x (R + C): line lengths per block; sorted position of every line
    DevBuf<int> hdr;        // G x kPcgBlocksHdrInts sizes and arena offsets, then the 4-int summary
    DevBuf<unsigned short> a16;  // per block: column index of every row-copy slot, line tables, row index and value reference of every column-copy slot
    DevBuf<int> a32;             // per block (fixed stride): chunk and heavy-line tables
    DevBuf<int> asrc;            // per block: CSR position of every row-copy slot (-1: padding)
    DevBuf<unsigned short> rowslot;  // row-copy slot of every CSR entry (scratch of the construction)
};
}  // namespace rg

struct regot_sparse {
    regot_ctx* ctx = nullptr;  // owner; never dereferenced on the free path (the context may be gone by then)
    int device = 0;
    int64_t n = 0, m = 0, nloc = 0, row_begin = 0;
    int64_t nnz = 0;  // |Omega| restricted to this rank's rows
    double tau = 0.0;
    // CSR of B over local rows; `row` is the local row of each entry
    rg::DevBuf<int> rowptr, col, row;
    rg::DevBuf<double> val, mval;  // values and the gathered costs M_ij (so value refreshes never touch M)
    // CSC of B (columns 0..m-2), rows ascending inside a column
    rg::DevBuf<int> cscptr, cscrow;
    rg::DevBuf<int> csccol;                // column of every CSC entry
    rg::DevBuf<double> cscmval;            // gathered costs in CSC order (the CSC values are computed in place)
    rg::DevBuf<double> cscval;
    rg::DevBuf<double> dA, dB;  // diagonal: row_sums/eta + tau, col_sums/eta + tau
    // lines (rows / columns of B) too long for one warp -- always row 0 and column 0 of
    // Omega* at scale -- cut into chunks: chunks = {line, beg, end, slot} x n_chunks,
    // longlines = {first chunk, count} x n_long; chunk_part / chunk_cnt are mat-vec scratch
    rg::DevBuf<int> chunks, longlines;
    mutable rg::DevBuf<double> chunk_part;
    mutable rg::DevBuf<unsigned int> chunk_cnt;
    int n_chunks = 0, n_long = 0;
    int n_chunks_rows = 0, n_lines_s_rows = 0, n_lines_m_rows = 0;  // rows come first in chunks / lines_s / lines_m
    // the other lines, binned by length so the mat-vec can give each line a fitting number of
    // lanes: short (<= kShortLine entries, 8 lanes) and medium (<= kLongLine, one warp)
    rg::DevBuf<int> lines_s, lines_m;
    int n_lines_s = 0, n_lines_m = 0;
    rg::PcgSchedule pcg;  // single-GPU direction solve (k5_pcg.cu)
    unsigned long structure_stamp = 0;         // bumped by finish_structure: derived plans know when they are stale
    mutable rg::DevBuf<int> diag_long;  // compute_schur_diag: count and list of the columns a whole CTA sums
    mutable rg::DevBuf<double> dS;  // diagonal of the Schur complement D2 - B' D1^-1 B: the Jacobi preconditioner of the PCG (per solve)
    mutable rg::PanelPlan panel_rows, panel_cols;  // kernel-by-kernel direction solve of large / sharded problems
    rg::PcgBlocksPlan blocks;                      // block-resident direction solve (k6_pcg_blocks.cu)
};

namespace rg {
constexpr int kShortLine = 64;  // <= this: 8 lanes per line, four lines per warp
constexpr int kLongLine = 512;  // > this: chunked across warps
constexpr int kChunkLen = 256;
}  // namespace rg

namespace rg {

struct SparseWS {
    // top-k selection scratch
    DevBuf<unsigned long long> hist;  // 4096 coarse bins | 8192 refine bins
    DevBuf<int> cnt, pre, rowtot, candptr;
    DevBuf<unsigned long long> cand_key;
    DevBuf<int> cand_col, cand_row, keep, tie, scan_a, scan_b;
    DevBuf<double> cand_m;
    DevBuf<unsigned char> cub_tmp;
    DevBuf<int> sort_k0, sort_k1, sort_v0, sort_v1;
    unsigned long long* h_hist = nullptr;  // pinned
    int* h_small = nullptr;                // pinned
    // PCG scratch
    DevBuf<double> cg;  // vectors
    DevBuf<double> cg_scal;
    DevBuf<double> cg_partials;
    DevBuf<unsigned int> cg_ticket;
    DevBuf<unsigned int> cg_barrier;
    DevBuf<unsigned long long> cg_xchg;  // persistent PCG: grid-barrier counter + flagged words of the partial-sum exchange
    // called by finish_structure once the pointer arrays are on their way to the host: GPU work that does not
    // depend on the pattern (the solver's candidate chain) is enqueued here and runs while the host builds the lists
    std::function<void()> after_pointer_download;
    cudaEvent_t ev_ptrs = nullptr;
    PinnedBuf<int> h_ptrs;   // rowptr | cscptr of the current pattern (device -> host)
    PinnedBuf<int> h_lines;  // line lists and the PCG schedule (host -> device)
    double* h_cg = nullptr;  // pinned
    HostMailbox cg_mbox;     // iteration counts / breakdown flag of the persistent PCG kernel
    int* h_blocks = nullptr;                 // pinned: summary of the block plan under construction
    DevBuf<unsigned long long> blocks_xchg;  // block-resident PCG: flagged words of its five exchanges
    unsigned int blocks_round = 0;           // next unused round number of those words
    ~SparseWS()
    {
        if (h_hist) cudaFreeHost(h_hist);
        if (h_small) cudaFreeHost(h_small);
        if (h_cg) cudaFreeHost(h_cg);
        if (h_blocks) cudaFreeHost(h_blocks);
    }
};

// Source of plan entries for the selection sweeps.
enum TopkSource { kFromDual = 0, kFromDenseT = 1 };

// k2_topk.cu -- select_topk (sparsity.h:44-91) + the structural half of assemble
// (sparsity.h:226-289) on the device.  In kFromDual mode T is formed on the fly
// from (alpha, beta) and the resident cost matrix; in kFromDenseT mode the
// "cost matrix" resident in ctx IS the dense plan (the parity entry point).
// Fills S's structure arrays (rowptr/col/row/mval, CSC, slot, long rows).
void topk_build_pattern(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, TopkSource src, const double* alpha,
                        const double* beta, int64_t k, regot_sparse& S);
// assemble at a caller-given pattern (host coords, sorted unique, global rows)
void pattern_from_coords(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, const int32_t* coords, int64_t ncoords,
                         regot_sparse& S);
// builds CSC + slot map + long row/col lists from rowptr/col/row (called by both of the above)
void finish_structure(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, regot_sparse& S);

// k4_sparse.cu -- fill_transport_values (sparsity.h:202-220): K3
void sparse_fill_values(regot_ctx* ctx, cudaStream_t st, regot_sparse& S, const double* alpha, const double* beta,
                        double tau, const double* row_sums, const double* col_sums);
// share of the Hessian block's mass (sum of all row sums over eta) held by the pattern's values as they stand; synchronises
// `st`; summed over the ranks when sharded (pattern reuse, regot_b200_set_pattern_reuse)
double sparse_captured_mass(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, const regot_sparse& S, DevBuf<double>& scratch,
                            const double* row_sums);
// osc(alpha - alpha0) + osc(beta - beta0) over the whole problem (max over the ranks when sharded); synchronises `st`
double dual_drift(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, const DVec& x, const DVec& x0, DevBuf<double>& scratch);
// y = A v on free vectors (K4); nrhs systems stored back to back with strides
void sparse_matvec(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, const regot_sparse& S, int nrhs, const double* va,
                   const double* vb, double* ya, double* yb, int64_t stride_a, int64_t stride_b);
// Jacobi-PCG (K5): solves A x_k = rhs_k for k < nrhs simultaneously.  Returns
// iterations, or -1 on breakdown (p'Ap <= 0: "not positive definite").
// k5_pcg.cu -- the single-GPU path of sparse_pcg: Schur-complement PCG in one persistent kernel
// rowptr_host / cscptr_host: nloc + 1 / m entries; staging: pinned scratch the uploads are issued from
// (asynchronously on st; the caller synchronises before the staging is reused)
void build_pcg_schedule(regot_ctx* ctx, cudaStream_t st, regot_sparse& S, const int* rowptr_host, const int* cscptr_host,
                        PinnedBuf<int>& staging, size_t staging_used);
int pcg_schur_persistent(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, const regot_sparse& S, int nrhs,
                         const DVec* const* rhs, DVec* const* sol, double rtol, int max_iter);
// k6_pcg_blocks.cu -- the block-resident form: plan construction (enqueued on st; finish_* after the caller's
// synchronisation reads the summary) and the solve
void build_pcg_blocks_plan(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, regot_sparse& S, const int* csc2csr, bool allow_cluster = true);
void finish_pcg_blocks_plan(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, regot_sparse& S, const int* csc2csr);
int pcg_schur_blocks(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, const regot_sparse& S, int nrhs, const DVec* const* rhs,
                     DVec* const* sol, double rtol, int max_iter);
int sparse_pcg(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, SparseWS& ws, const regot_sparse& S, int nrhs,
               const DVec* const* rhs, DVec* const* sol, double rtol, int max_iter);

}  // namespace rg
