// k6_pcg_blocks.cu -- K5 on one GPU, block-resident form: the direction solve of small and mid-size
// patterns with the matrix held in shared memory for the whole solve.
//
// Replaces numeric_factorize + solve (sparse_chol.h:330-427) inside compute_direction (splr.h:128-167),
// like k5_pcg.cu: Jacobi-preconditioned CG on the Schur complement of the alpha block,
//     S x_b = r_b - B' D1^-1 r_a,   S = D2 - B' D1^-1 B,   x_a = D1^-1 (r_a - B x_b),
// two right-hand sides carried through every pass (interleaved 2 doubles per index), single-reduction
// recurrences (Chronopoulos-Gear).  What differs is where things live.  k_pcg_schur streams the matrix
// from L2 twice per iteration and has every CTA copy the whole iterated vector into shared memory at the
// start of each phase (config B: 24 MB + 47 MB through L2 per iteration, ~25 dependent L2 latencies,
// 25 us).  Here B is cut into P x Q blocks (P, Q coprime, P Q <= number of SMs): rows are dealt to block
// rows round-robin (row i -> block row i mod P, local row i / P), columns likewise (j mod Q, j / Q), so
// banded and clustered patterns spread evenly and a full row / column of Omega* is split over Q / P
// blocks by construction.  CTA (p, q) keeps block (p, q) in shared memory for the whole solve -- once as
// rows (local column index + value per entry) and once as columns (local row index + a 16-bit reference
// into the row copy's values) -- and needs only the q-th slice of a beta-space vector and the p-th slice
// of an alpha-space vector.  Lines of a block are sorted by length and processed one per thread in
// 32-line chunks stored entry-major (no shuffles, no bank conflicts on the matrix); lines longer than a
// threshold are processed by a warp each.
//
// One CG iteration is four exchanges through L2, none of them a barrier:
//   z slices (owners -> block column) | row phase | partial sums (block row -> owners), t = D1^-1 sum |
//   t slices (owners -> block row) | column phase | partial sums (block column -> owners) together with
//   the partial dot products (everybody -> everybody) | owners update p, s, x, r, z of their slice.
// Every exchanged double travels as two 64-bit words that each carry 32 bits of the value and the 32-bit
// round number, so the consumer polls the data itself: no fence, no flag, no atomic (an aligned 8-byte
// store is single-copy atomic).  A word is rewritten only after every reader has consumed it (the chain
// of dependencies around one iteration guarantees it, see the comment at k_pcg_blocks).  delta = z'Sz is
// formed as sum(D2 z^2) - sum over blocks of z_q . (B_pq' t_p), so the dot products ride on the same
// exchange as the column partial sums.  Every sum has a fixed order (entries of a line in index order,
// blocks in block order, CTAs in CTA order): results are bitwise reproducible.
#include "common.cuh"
#include "ctx.hpp"
#include "sparse.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace rg {

constexpr int kB2Threads = 512;
constexpr int kB2Warps = kB2Threads / 32;
constexpr int kB2MaxL = 64;        // longest line processed by one thread
constexpr int kB2MaxChunks = 1024;  // 32-line chunks per block and copy
constexpr int kB2Slack = 2048;     // bytes of shared memory behind the arrays (predicated over-reads stay in bounds)
enum {
    kH_NV_R = 0, kH_NCH_R, kH_NSL_R, kH_NHV_R, kH_NHE_R,  // row copy: light lines, chunks, chunk slots, heavy lines, heavy entries
    kH_NV_C, kH_NCH_C, kH_NSL_C, kH_NHV_C, kH_NHE_C,      // column copy
    kH_OFF16, kH_OFFSRC, kH_SMEM, kH_BAD
};
static_assert(kH_BAD < kPcgBlocksHdrInts, "header too small");

typedef unsigned long long u64;
typedef unsigned short u16;

__host__ __device__ __forceinline__ int pad8(int n) { return (n + 7) & ~7; }

// where the pieces of one block sit inside its region of the 16-bit arena (units: u16)
struct Lay16 {
    int ell_r, lov_r, ell_c, ref_c, lov_c, size;
};
__host__ __device__ __forceinline__ Lay16 lay16(const int* h)
{
    Lay16 L;
    L.ell_r = 0;
    L.lov_r = pad8(h[kH_NSL_R] + h[kH_NHE_R]);
    L.ell_c = L.lov_r + pad8(h[kH_NV_R]);
    L.ref_c = L.ell_c + pad8(h[kH_NSL_C] + h[kH_NHE_C]);
    L.lov_c = L.ref_c + pad8(h[kH_NSL_C] + h[kH_NHE_C]);
    L.size = L.lov_c + pad8(h[kH_NV_C]);
    return L;
}
// tables of one block in the 32-bit arena (fixed stride per block): chunk (base, width) pairs and heavy
// (line, start, length) triples of the row copy, then of the column copy
struct Lay32 {
    int chunk_r, heavy_r, chunk_c, heavy_c, stride;
};
__host__ __device__ __forceinline__ Lay32 lay32(int R, int C)
{
    Lay32 L;
    L.chunk_r = 0;
    L.heavy_r = 2 * (R / 32 + 2);
    L.chunk_c = L.heavy_r + 3 * kPcgBlocksMaxHeavy;
    L.heavy_c = L.chunk_c + 2 * (C / 32 + 2);
    L.stride = (L.heavy_c + 3 * kPcgBlocksMaxHeavy + 3) & ~3;
    return L;
}

// dynamic shared memory of the solve kernel for one block (the carve-up at the top of k_pcg_blocks)
__host__ __device__ __forceinline__ long b2_smem_need(const int* h, int R, int C, int SR, int SC, int P, int Q)
{
    const int nval = h[kH_NSL_R] + h[kH_NHE_R];
    const int segcap_r = h[kH_NHE_R] / 128 + h[kH_NHV_R], segcap_c = h[kH_NHE_C] / 128 + h[kH_NHV_C];
    const int tables = 2 * h[kH_NCH_R] + 3 * h[kH_NHV_R] + 2 * h[kH_NCH_C] + 3 * h[kH_NHV_C];
    const int derived = h[kH_NV_R] + h[kH_NV_C] + 2 * (h[kH_NHV_R] + h[kH_NHV_C]) + 2 + segcap_r + segcap_c + 4;
    return (long)(((nval + 1) * 8 + 15) & ~15) + 16L * C + 16L * R + 16L * (segcap_r > segcap_c ? segcap_r : segcap_c) + 2L * lay16(h).size +
           (long)(((tables + derived) * 4 + 15) & ~15) + 8L * (6 * 2 * SC + SC + SR) + 8L * (Q * 2 * SR > P * 2 * SC ? Q * 2 * SR : P * 2 * SC) + 8L * (8 * P * Q) + 8L * (16 + 8 * kB2Warps) + 256 + kB2Slack;
}

// ---- plan construction (device; once per pattern) -----------------------------------------------------
// line lengths per block: cnt_r[b][local row], cnt_c[b][local column]
__global__ void k_b2_count(int nnz, int P, int Q, int R, int C, const int* __restrict__ row, const int* __restrict__ col,
                           int* __restrict__ cnt_r, int* __restrict__ cnt_c)
{
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += gridDim.x * blockDim.x) {
        const int i = row[e], j = col[e];
        const int b = (i % P) * Q + (j % Q);
        atomicAdd(cnt_r + (size_t)b * R + i / P, 1);
        atomicAdd(cnt_c + (size_t)b * C + j / Q, 1);
    }
}

// One CTA per block: light lines (<= L entries) sorted by decreasing length (a counting sort; the order
// inside a bucket is arrival order, which moves a line to another thread but never changes a sum), cut
// into chunks of 32; chunk c is as wide as its first line.  Heavy lines get a slot in the heavy table.
// vpos[line] = sorted position, or 0x40000000 | heavy slot.
__global__ void __launch_bounds__(256) k_b2_layout(int P, int Q, int R, int C, int nloc, int mfree, int Lr, int Lc,
                                                   const int* __restrict__ cnt_r, const int* __restrict__ cnt_c,
                                                   int* __restrict__ vpos_r, int* __restrict__ vpos_c, int* __restrict__ a32,
                                                   int* __restrict__ hdr)
{
    __shared__ int hist[kB2MaxL + 2], startd[kB2MaxL + 2], cursor[kB2MaxL + 2], width[kB2MaxChunks];
    __shared__ int n_heavy, n_heavy_ent, bad;
    const int b = blockIdx.x, p = b / Q, q = b % Q, tid = threadIdx.x;
    const Lay32 T = lay32(R, C);
    int* tbl = a32 + (size_t)b * T.stride;
    int* h = hdr + (size_t)b * kPcgBlocksHdrInts;
    if (tid == 0) bad = 0;
    for (int copy = 0; copy < 2; ++copy) {
        const int nlines = copy == 0 ? (nloc - p + P - 1) / P : (mfree - q + Q - 1) / Q;
        const int L = copy == 0 ? Lr : Lc;
        const int* cnt = copy == 0 ? cnt_r + (size_t)b * R : cnt_c + (size_t)b * C;
        int* vpos = copy == 0 ? vpos_r + (size_t)b * R : vpos_c + (size_t)b * C;
        int* chunk = tbl + (copy == 0 ? T.chunk_r : T.chunk_c);
        int* heavy = tbl + (copy == 0 ? T.heavy_r : T.heavy_c);
        for (int k = tid; k <= L; k += blockDim.x) hist[k] = 0;
        if (tid == 0) n_heavy = n_heavy_ent = 0;
        __syncthreads();
        // histogram of the light lines; heavy lines in index order (warp 0: ballot rank, scan of the lengths)
        for (int l = tid; l < nlines; l += blockDim.x) {
            const int len = cnt[l];
            if (len <= L) atomicAdd(&hist[len], 1);
        }
        if (tid < 32) {
            int nh = 0, ne = 0;
            for (int l0 = 0; l0 < nlines; l0 += 32) {
                const int l = l0 + tid, len = l < nlines ? cnt[l] : 0;
                const bool hv = len > L;
                const unsigned m = __ballot_sync(0xffffffffu, hv);
                int incl = hv ? len : 0;  // inclusive scan of the heavy lengths over the tile
                for (int o = 1; o < 32; o <<= 1) {
                    const int up = __shfl_up_sync(0xffffffffu, incl, o);
                    if (tid >= o) incl += up;
                }
                if (hv) {
                    const int slot = nh + __popc(m & ((1u << tid) - 1u));
                    if (slot < kPcgBlocksMaxHeavy) {
                        heavy[3 * slot] = l;
                        heavy[3 * slot + 1] = ne + incl - len;
                        heavy[3 * slot + 2] = len;
                    }
                    vpos[l] = 0x40000000 | slot;
                }
                nh += __popc(m);
                ne += __shfl_sync(0xffffffffu, incl, 31);
            }
            if (tid == 0) {
                n_heavy = nh;
                n_heavy_ent = ne;
            }
        }
        __syncthreads();
        if (tid == 0) {
            int acc = 0;
            for (int len = L; len >= 0; --len) {
                startd[len] = cursor[len] = acc;
                acc += hist[len];
            }
            startd[L + 1] = acc;  // = number of light lines
        }
        __syncthreads();
        const int nv = startd[L + 1], nch = (nv + 31) / 32;
        // stable positions: lines of one length keep their index order (warp w ranks the lengths w, w + 8, ... by ballot),
        // so the layout -- and with it the order in which a thread meets its lines -- is the same in every run
        {
            const int wl = tid & 31, ww = tid >> 5, nwarp = blockDim.x >> 5;
            for (int l0 = 0; l0 < nlines; l0 += 32) {
                const int l = l0 + wl, len = l < nlines ? cnt[l] : -1;
                for (int bk = ww; bk <= L; bk += nwarp) {
                    const unsigned m = __ballot_sync(0xffffffffu, len == bk);
                    if (m == 0u) continue;
                    const int base = cursor[bk];
                    __syncwarp();
                    if (len == bk) vpos[l] = base + __popc(m & ((1u << wl) - 1u));
                    if (wl == 0) cursor[bk] = base + __popc(m);
                    __syncwarp();
                }
            }
        }
        for (int c = tid; c < nch && c < kB2MaxChunks; c += blockDim.x) {
            int w = 0;  // length of the line at sorted position 32 c
            for (int len = L; len >= 0; --len)
                if (startd[len] <= 32 * c && 32 * c < startd[len] + hist[len]) w = len;
            width[c] = w;
        }
        __syncthreads();
        if (tid == 0) {
            int base = 0;
            for (int c = 0; c < nch && c < kB2MaxChunks; ++c) {
                chunk[2 * c] = base;
                chunk[2 * c + 1] = width[c];
                base += 32 * width[c];
            }
            if (nch > kB2MaxChunks || n_heavy > kPcgBlocksMaxHeavy || base + n_heavy_ent > 65000) bad = 1;
            const int o = copy == 0 ? kH_NV_R : kH_NV_C;
            h[o] = nv;
            h[o + 1] = nch;
            h[o + 2] = base;
            h[o + 3] = min(n_heavy, kPcgBlocksMaxHeavy);
            h[o + 4] = n_heavy_ent;
        }
        __syncthreads();
    }
    if (tid == 0) h[kH_BAD] = bad;
}

// arena offsets of every block (one CTA), shared-memory need of the solve kernel per block, and the summary
// the host reads: {largest need, any block unusable, total u16 units, total source entries}
__global__ void k_b2_offsets(int P, int Q, int R, int C, int SR, int SC, int* __restrict__ hdr, int* __restrict__ summary)
{
    if (threadIdx.x != 0) return;
    const int G = P * Q;
    long off16 = 0, offsrc = 0;
    int worst = 0, bad = 0;
    for (int b = 0; b < G; ++b) {
        int* h = hdr + (size_t)b * kPcgBlocksHdrInts;
        const Lay16 L = lay16(h);
        h[kH_OFF16] = (int)off16;
        h[kH_OFFSRC] = (int)offsrc;
        const int nval = h[kH_NSL_R] + h[kH_NHE_R];
        off16 += L.size;
        offsrc += (nval + 3) & ~3;
        const long need = b2_smem_need(h, R, C, SR, SC, P, Q);
        h[kH_SMEM] = need < (1L << 30) ? (int)need : (1 << 30);
        worst = max(worst, h[kH_SMEM]);
        bad |= h[kH_BAD];
    }
    summary[0] = worst;
    summary[1] = bad || off16 > 0x7fffffffL;
    summary[2] = (int)off16;
    summary[3] = (int)offsrc;
}

// defaults of every slot (padding: index 0, no source, reference to the zero value) and the sorted-position ->
// line tables
__global__ void __launch_bounds__(256) k_b2_fill(int P, int Q, int R, int C, int nloc, int mfree, const int* __restrict__ hdr,
                                                 const int* __restrict__ vpos_r, const int* __restrict__ vpos_c,
                                                 u16* __restrict__ a16, int* __restrict__ asrc)
{
    const int b = blockIdx.x, p = b / Q, q = b % Q, tid = threadIdx.x;
    const int* h = hdr + (size_t)b * kPcgBlocksHdrInts;
    const Lay16 L = lay16(h);
    u16* w = a16 + h[kH_OFF16];
    const int nval = h[kH_NSL_R] + h[kH_NHE_R], ncol = h[kH_NSL_C] + h[kH_NHE_C];
    for (int s = tid; s < L.size; s += blockDim.x) w[s] = 0;
    __syncthreads();
    for (int s = tid; s < ncol; s += blockDim.x) w[L.ref_c + s] = (u16)nval;  // val[nval] == 0
    int* src = asrc + h[kH_OFFSRC];
    for (int s = tid; s < ((nval + 3) & ~3); s += blockDim.x) src[s] = -1;
    const int Rp = (nloc - p + P - 1) / P, Cq = (mfree - q + Q - 1) / Q;
    for (int l = tid; l < Rp; l += blockDim.x) {
        const int v = vpos_r[(size_t)b * R + l];
        if (!(v & 0x40000000)) w[L.lov_r + v] = (u16)l;
    }
    for (int l = tid; l < Cq; l += blockDim.x) {
        const int v = vpos_c[(size_t)b * C + l];
        if (!(v & 0x40000000)) w[L.lov_c + v] = (u16)l;
    }
}

// One warp per line of the CSR (kRows) or CSC of B: every entry goes to its slot of its block.  The rank of an
// entry among the entries of its line that fall into the same block is its position in index order (the order
// of the per-thread sums), found 32 entries at a time with match_any.
template <bool kRows>
__global__ void __launch_bounds__(256) k_b2_scatter(int nlines, int P, int Q, int R, int C, const int* __restrict__ ptr,
                                                    const int* __restrict__ idx, const int* __restrict__ csc2csr,
                                                    const int* __restrict__ hdr, const int* __restrict__ vpos,
                                                    const int* __restrict__ a32, u16* __restrict__ a16, int* __restrict__ asrc,
                                                    u16* __restrict__ rowslot)
{
    __shared__ int seen[8][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const Lay32 T = lay32(R, C);
    const int nother = kRows ? Q : P;
    for (int line = blockIdx.x * 8 + wib; line < nlines; line += gridDim.x * 8) {
        seen[wib][lane] = 0;
        __syncwarp();
        const int mine = kRows ? line % P : line % Q, lline = kRows ? line / P : line / Q;
        const int beg = ptr[line], end = ptr[line + 1];
        for (int e0 = beg; e0 < end; e0 += 32) {
            const int e = e0 + lane;
            const bool ok = e < end;
            const int x = ok ? idx[e] : 0;
            const int other = ok ? x % nother : nother + lane;  // inactive lanes match nobody
            const unsigned same = __match_any_sync(0xffffffffu, other);
            const int before = __popc(same & ((1u << lane) - 1u));
            const int base = ok ? seen[wib][other] : 0;
            __syncwarp();
            if (ok && before == 0) seen[wib][other] = base + __popc(same);
            __syncwarp();
            if (!ok) continue;
            const int rank = base + before;
            const int b = kRows ? mine * Q + other : other * Q + mine;
            const int* h = hdr + (size_t)b * kPcgBlocksHdrInts;
            const int* tbl = a32 + (size_t)b * T.stride;
            const int v = vpos[(size_t)b * (kRows ? R : C) + lline];
            int slot;
            if (v & 0x40000000) {
                const int hs = v & 0x3fffffff;
                slot = h[kRows ? kH_NSL_R : kH_NSL_C] + tbl[(kRows ? T.heavy_r : T.heavy_c) + 3 * min(hs, kPcgBlocksMaxHeavy - 1) + 1] + rank;
            } else {
                slot = tbl[(kRows ? T.chunk_r : T.chunk_c) + 2 * min(v >> 5, kB2MaxChunks - 1)] + 32 * rank + (v & 31);
            }
            if (h[kH_BAD]) continue;  // the plan is dropped by the host; stay inside the arenas
            const Lay16 L = lay16(h);
            u16* w = a16 + h[kH_OFF16];
            if (kRows) {
                w[L.ell_r + slot] = (u16)(x / Q);
                asrc[h[kH_OFFSRC] + slot] = e;
                rowslot[e] = (u16)slot;
            } else {
                w[L.ell_c + slot] = (u16)(x / P);
                w[L.ref_c + slot] = rowslot[csc2csr[e]];
            }
        }
        __syncwarp();
    }
}

// ---- the solve ------------------------------------------------------------------------------------------
// The loop body has to stay well inside the 32 KB instruction cache of an SM: with 16 warps per CTA and every
// section of an iteration executed once, a body that spills out of it fetches its instructions from L2 line by
// line (measured on the first version of this kernel, 64 KB of SASS: 7 k clk for a 300-instruction section).
// Hence the polling loops, the mat-vec phase and the divisions are single out-of-line copies.
struct BlocksParams {
    int nloc, mfree, nrhs, max_iter, fixed_iters;
    int P, Q, R, C, SR, SC;
    double tol2;
    const int* hdr;
    const u16* a16;
    const int* a32;
    const int* asrc;
    const double* val;  // CSR values of B (regot_sparse::val)
    const double* dA;
    const double* dB;
    const double* rhs_a[2];
    const double* rhs_b[2];
    double* sol_a[2];
    double* sol_b[2];
    u64 *x1, *x2, *x3, *x4, *x5;  // flagged words of the five exchanges
    unsigned int round0;          // round number of this launch's first exchange
    double* out;                  // iters[2], -, breakdown flag
    double* mbox;
    unsigned long long mseq;
};

__device__ __forceinline__ void fw_post(u64* slot, double v, unsigned int round)
{
    const u64 b = (u64)__double_as_longlong(v), f = (u64)round << 32;
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(slot), "l"((b & 0xffffffffull) | f), "l"((b >> 32) | f) : "memory");
}
__device__ __forceinline__ bool fw_try(const u64* slot, unsigned int round, double& v)
{
    u64 lo, hi;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(slot) : "memory");
    v = __longlong_as_double((long long)((lo & 0xffffffffull) | (hi << 32)));
    return (unsigned int)(lo >> 32) == round && (unsigned int)(hi >> 32) == round;
}
// Flagged doubles -> shared memory, all threads of the CTA, 4 loads in flight per thread.  Element (o, r), o <
// n_outer, r < n_inner, is awaited at src + 2 (o src_stride + r) and lands in dst[o n_inner + r].
__device__ __noinline__ void fw_gather(const u64* src, double* dst, int n_inner, int n_outer, int src_stride, unsigned int round)
{
    const int n = n_inner * n_outer;
    for (int i0 = threadIdx.x; i0 < n; i0 += kB2Threads * 4) {
        double v[4];
        const u64* at[4];
        unsigned pend = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = i0 + u * kB2Threads;
            at[u] = src;
            if (i < n) {
                const int o = i / n_inner;
                at[u] = src + 2 * ((size_t)o * src_stride + (i - o * n_inner));
                pend |= 1u << u;
            }
        }
        const unsigned valid = pend;
        while (pend) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if ((pend >> u) & 1u)
                    if (fw_try(at[u], round, v[u])) pend &= ~(1u << u);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if ((valid >> u) & 1u) dst[i0 + u * kB2Threads] = v[u];
    }
}

constexpr int kB2Seg = 128;  // entries of a heavy line one warp sums at a time

struct BlockCopy {  // one copy (rows or columns) of the CTA's block in shared memory
    const u16* ell;     // entry -> local index into the gathered slice
    const u16* ref;     // column copy: entry -> position in `val` (row copy: null, the entry's own position)
    const u16* lov;     // sorted position -> local line
    const int* off;     // sorted position -> word offset of the line's two sums in the exchange
    const int* chunk;   // (first slot, width) per 32-line chunk
    const int* heavy;   // (line, first entry, length) per heavy line
    const int* hoff;    // heavy line -> word offset in the exchange
    const int* hfirst;  // heavy line -> its first segment
    const int* hseg;    // segment -> heavy line
    int nv, nch, nsl, nhv, nseg;
};

// One mat-vec phase over the CTA's block: lines are the block's rows and `vec` the z (or x) slice of the block
// column, or lines are its columns and `vec` the t slice of the block row.  Work items: segments of heavy lines
// first, then the 32-line chunks by decreasing width.  Each finished line's two sums are posted as flagged words where the owner of the
// line's slice expects them; with zvec != null (column phase) z . (B' t) is accumulated per system into dc[0..1]
// of this thread.
__device__ __noinline__ void block_phase(const BlockCopy* Bp, const double* __restrict__ val, int zero_slot,
                                         const double2* __restrict__ vec, const double2* __restrict__ zvec, u64* xbase,
                                         unsigned int round, double2* hpart, double* dc)
{
    const BlockCopy B = *Bp;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int total = B.nseg + B.nch;
    double dc0 = 0.0, dc1 = 0.0;
    // items by decreasing cost, dealt over the warps in a snake: static, so every thread meets its lines in the same
    // order in every run (the dot-product partials are summed in that order)
    for (int r0 = 0;; ++r0) {
        const int item = r0 * kB2Warps + ((r0 & 1) ? kB2Warps - 1 - warp : warp);
        if (r0 * kB2Warps >= total) break;
        if (item >= total) continue;
        double a0 = 0.0, a1 = 0.0;
        if (item < B.nseg) {
            const int h = B.hseg[item], sidx = item - B.hfirst[h];
            const int beg = B.nsl + B.heavy[3 * h + 1] + sidx * kB2Seg, len = min(kB2Seg, B.heavy[3 * h + 2] - sidx * kB2Seg);
            for (int t = lane; t < len; t += 32) {
                const int s = beg + t;
                const double v = val[B.ref ? (int)B.ref[s] : s];
                const double2 g = vec[B.ell[s]];
                a0 = __fma_rn(v, g.x, a0);
                a1 = __fma_rn(v, g.y, a1);
            }
            a0 = warp_sum(a0);
            a1 = warp_sum(a1);
            if (lane == 0) hpart[item] = make_double2(a0, a1);
            continue;
        }
        const int c = item - B.nseg;
        const int base = B.chunk[2 * c] + lane, w = B.chunk[2 * c + 1];
#pragma unroll 1
        for (int k0 = 0; k0 < w; k0 += 4) {
            int ix[4], vi[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int s = base + 32 * (k0 + u);
                const bool ok = k0 + u < w;
                const int raw = B.ell[s];
                ix[u] = ok ? raw : 0;
                const int rr = B.ref ? (int)B.ref[s] : s;
                vi[u] = ok ? rr : zero_slot;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double v = val[vi[u]];
                const double2 g = vec[ix[u]];
                a0 = __fma_rn(v, g.x, a0);
                a1 = __fma_rn(v, g.y, a1);
            }
        }
        const int vpos = 32 * c + lane;
        if (vpos < B.nv) {
            u64* w2 = xbase + B.off[vpos];
            fw_post(w2, a0, round);
            fw_post(w2 + 2, a1, round);
            if (zvec) {
                const double2 z = zvec[B.lov[vpos]];
                dc0 = __fma_rn(z.x, a0, dc0);
                dc1 = __fma_rn(z.y, a1, dc1);
            }
        }
    }
    if (B.nhv > 0) {  // uniform over the CTA
        __syncthreads();
        for (int h = threadIdx.x; h < B.nhv; h += kB2Threads) {
            double a0 = 0.0, a1 = 0.0;
            for (int sg = B.hfirst[h]; sg < B.hfirst[h + 1]; ++sg) {
                a0 += hpart[sg].x;
                a1 += hpart[sg].y;
            }
            u64* w2 = xbase + B.hoff[h];
            fw_post(w2, a0, round);
            fw_post(w2 + 2, a1, round);
            if (zvec) {
                const double2 z = zvec[B.heavy[3 * h]];
                dc0 = __fma_rn(z.x, a0, dc0);
                dc1 = __fma_rn(z.y, a1, dc1);
            }
        }
    }
    dc[0] = dc0;
    dc[1] = dc1;
}

// Sum of 8 per-thread values over the CTA in a fixed order (transposing butterfly in the warp, then the 16 warps in
// a 4-step butterfly): thread 16 k (k < 8) returns the total of v[k]; 13 shuffles instead of 80.
__device__ __forceinline__ double block_sum8(const double (&v)[8], double* scratch /* 8 x kB2Warps */)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double c = warp_sum8_transpose(v, lane);
    if ((lane & 3) == 0) scratch[warp_sum8_index(lane) * kB2Warps + warp] = c;
    __syncthreads();
    double d = 0.0;
    if (threadIdx.x < 8 * kB2Warps) {
        d = scratch[threadIdx.x];
        d += shfl_xor_d(d, 8);
        d += shfl_xor_d(d, 4);
        d += shfl_xor_d(d, 2);
        d += shfl_xor_d(d, 1);
    }
    return d;
}
static_assert(kB2Warps == 16, "block_sum8 folds 16 warps per component");
static_assert(2 * sizeof(BlockCopy) <= 256, "descriptor area of the shared-memory plan");

// Why a single buffer per exchange is enough (a word is awaited by exact round number, so a writer must
// not get a round ahead of a reader): round r + 1 writes of X4 follow the owner's update, which needs every
// CTA's X5 post of round r, which every CTA makes after it has read X4, X1 (owners) and X2 of round r;
// X1 / X2 of round r + 1 follow the CTA's own read of X4 (r + 1), i.e. every owner's update; X3 (r + 1)
// likewise; X5 (r + 1) follows the CTA's row phase of round r + 1, whose t slice needs z slices of round
// r + 1 from owners in every block column, i.e. everybody's update, i.e. everybody's read of X5 (r).
__global__ void __launch_bounds__(kB2Threads, 1) k_pcg_blocks(const __grid_constant__ BlocksParams A)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int P = A.P, Q = A.Q, G = P * Q, b = blockIdx.x, p = b / Q, q = b % Q;
    const int Rp = (A.nloc - p + P - 1) / P, Cq = (A.mfree - q + Q - 1) / Q;
    const int SR = A.SR, SC = A.SC, nrhs = A.nrhs;
    const int* h = A.hdr + (size_t)b * kPcgBlocksHdrInts;
    const Lay16 L16 = lay16(h);
    const Lay32 T = lay32(A.R, A.C);
    const int nval = h[kH_NSL_R] + h[kH_NHE_R];
    BlockCopy Br, Bc;
    Br.nv = h[kH_NV_R];
    Br.nch = h[kH_NCH_R];
    Br.nsl = h[kH_NSL_R];
    Br.nhv = h[kH_NHV_R];
    Bc.nv = h[kH_NV_C];
    Bc.nch = h[kH_NCH_C];
    Bc.nsl = h[kH_NSL_C];
    Bc.nhv = h[kH_NHV_C];
    const int segcap_r = h[kH_NHE_R] / kB2Seg + Br.nhv, segcap_c = h[kH_NHE_C] / kB2Seg + Bc.nhv;

    // ---- shared-memory carve-up (b2_smem_need) ----
    unsigned char* sp = smem;
    double* val = reinterpret_cast<double*>(sp);
    sp += ((nval + 1) * 8 + 15) & ~15;
    double2* vecz = reinterpret_cast<double2*>(sp);
    sp += 16 * (size_t)A.C;
    double2* vect = reinterpret_cast<double2*>(sp);
    sp += 16 * (size_t)A.R;
    double2* hpart = reinterpret_cast<double2*>(sp);
    sp += 16 * (size_t)max(segcap_r, segcap_c);
    u16* s16 = reinterpret_cast<u16*>(sp);
    sp += 2 * (size_t)L16.size;
    int* s32 = reinterpret_cast<int*>(sp);
    const int n_tables = 2 * Br.nch + 3 * Br.nhv + 2 * Bc.nch + 3 * Bc.nhv;
    const int n_derived = Br.nv + Bc.nv + 2 * (Br.nhv + Bc.nhv) + 2 + segcap_r + segcap_c + 4;
    sp += ((n_tables + n_derived) * 4 + 15) & ~15;
    double* own = reinterpret_cast<double*>(sp);  // z p s x r w of the owned column slice (x2), 1/dB of it, 1/dA of the owned row slice
    sp += 8 * (size_t)(6 * 2 * SC + SC + SR);
    double* xbuf = reinterpret_cast<double*>(sp);  // partial sums collected by the owner: Q x 2 SR or P x 2 SC
    sp += 8 * (size_t)max(Q * 2 * SR, P * 2 * SC);
    double* stage = reinterpret_cast<double*>(sp);  // 8 G: everybody's partial dot products
    sp += 8 * (size_t)(8 * G);
    double* bcast = reinterpret_cast<double*>(sp);  // 8 totals, my own 4 partials, then block_sum scratch
    double* scratch = bcast + 16;
    BlockCopy* s_copy = reinterpret_cast<BlockCopy*>(scratch + 8 * kB2Warps);  // the two copies' descriptors, read by block_phase
    double *oz = own, *op = own + 2 * SC, *os = own + 4 * SC, *ox = own + 6 * SC, *orr = own + 8 * SC, *ow = own + 10 * SC,
           *oib = own + 12 * SC, *oia = own + 13 * SC;
    int* tb = s32;
    Br.chunk = tb;
    tb += 2 * Br.nch;
    Br.heavy = tb;
    tb += 3 * Br.nhv;
    Bc.chunk = tb;
    tb += 2 * Bc.nch;
    Bc.heavy = tb;
    tb += 3 * Bc.nhv;
    int *off_r = tb, *off_c = off_r + Br.nv, *hoff_r = off_c + Bc.nv, *hoff_c = hoff_r + Br.nhv, *hfirst_r = hoff_c + Bc.nhv,
        *hfirst_c = hfirst_r + Br.nhv + 1, *hseg_r = hfirst_c + Bc.nhv + 1, *hseg_c = hseg_r + segcap_r;
    Br.ell = s16 + L16.ell_r;
    Br.ref = nullptr;
    Br.lov = s16 + L16.lov_r;
    Br.off = off_r;
    Br.hoff = hoff_r;
    Br.hfirst = hfirst_r;
    Br.hseg = hseg_r;
    Bc.ell = s16 + L16.ell_c;
    Bc.ref = s16 + L16.ref_c;
    Bc.lov = s16 + L16.lov_c;
    Bc.off = off_c;
    Bc.hoff = hoff_c;
    Bc.hfirst = hfirst_c;
    Bc.hseg = hseg_c;

    // ---- the block: structure from the arenas, values from the CSR of B ----
    {
        const u16* g16 = A.a16 + h[kH_OFF16];
        for (int s = tid; s < L16.size / 8; s += kB2Threads)
            reinterpret_cast<uint4*>(s16)[s] = __ldg(reinterpret_cast<const uint4*>(g16) + s);
        const int* g32 = A.a32 + (size_t)b * T.stride;
        int o = 0;
        const int part_off[4] = {T.chunk_r, T.heavy_r, T.chunk_c, T.heavy_c};
        const int part_len[4] = {2 * Br.nch, 3 * Br.nhv, 2 * Bc.nch, 3 * Bc.nhv};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            for (int s = tid; s < part_len[k]; s += kB2Threads) s32[o + s] = __ldg(g32 + part_off[k] + s);
            o += part_len[k];
        }
        const int* src = A.asrc + h[kH_OFFSRC];
        for (int s = tid; s < nval; s += kB2Threads) {
            const int e = __ldg(src + s);
            val[s] = e >= 0 ? __ldg(A.val + e) : 0.0;
        }
        if (tid == 0) val[nval] = 0.0;
    }
    __syncthreads();
    // where each line's sums go: rows -> [owner = line / SR][source q][line % SR][2], columns likewise with P, SC
    for (int v = tid; v < Br.nv; v += kB2Threads) {
        const int line = Br.lov[v], o = line / SR;
        off_r[v] = ((o * Q + q) * SR + (line - o * SR)) * 4;
    }
    for (int v = tid; v < Bc.nv; v += kB2Threads) {
        const int line = Bc.lov[v], o = line / SC;
        off_c[v] = ((o * P + p) * SC + (line - o * SC)) * 4;
    }
    for (int hh = tid; hh < Br.nhv; hh += kB2Threads) {
        const int line = Br.heavy[3 * hh], o = line / SR;
        hoff_r[hh] = ((o * Q + q) * SR + (line - o * SR)) * 4;
    }
    for (int hh = tid; hh < Bc.nhv; hh += kB2Threads) {
        const int line = Bc.heavy[3 * hh], o = line / SC;
        hoff_c[hh] = ((o * P + p) * SC + (line - o * SC)) * 4;
    }
    if (tid < 2) {  // segments of the heavy lines: thread 0 the rows', thread 1 the columns'
        const BlockCopy& B = tid == 0 ? Br : Bc;
        int* hf = tid == 0 ? hfirst_r : hfirst_c;
        int* hs = tid == 0 ? hseg_r : hseg_c;
        int n = 0;
        for (int hh = 0; hh < B.nhv; ++hh) {
            hf[hh] = n;
            const int cnt = (B.heavy[3 * hh + 2] + kB2Seg - 1) / kB2Seg;
            for (int k = 0; k < cnt; ++k) hs[n++] = hh;
        }
        hf[B.nhv] = n;
    }
    __syncthreads();
    if (tid == 0) {
        Br.nseg = hfirst_r[Br.nhv];
        Bc.nseg = hfirst_c[Bc.nhv];
        s_copy[0] = Br;
        s_copy[1] = Bc;
    }

    // owned slices: local rows [r_lo, r_hi) of block row p, local columns [c_lo, c_hi) of block column q
    const int r_lo = min(q * SR, Rp), r_hi = min(r_lo + SR, Rp), c_lo = min(p * SC, Cq), c_hi = min(c_lo + SC, Cq);
    const int n_own_r = r_hi - r_lo, n_own_c = c_hi - c_lo;
    u64* const x1_mine = A.x1 + (size_t)(p * Q) * Q * SR * 4;          // block row p: [owner][source q][SR][2] doubles
    u64* const x1_own = x1_mine + (size_t)q * Q * SR * 4;               // what I sum as owner q
    u64* const x2_row = A.x2 + (size_t)p * A.R * 4;                     // t of block row p: [R][2]
    u64* const x3_mine = A.x3 + (size_t)(q * P) * P * SC * 4;          // block column q: [owner][source p][SC][2]
    u64* const x3_own = x3_mine + (size_t)p * P * SC * 4;
    u64* const x4_col = A.x4 + (size_t)q * A.C * 4;                     // z of block column q: [C][2]

    // ---- t = D1^-1 r_a on my block row; the alpha part of r' D^-1 r over my row slice ----
    double part[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // gamma[2], sum dB z^2 [2], z.(B't) [2], r'D^-1 r [2]
    for (int li = tid; li < Rp; li += kB2Threads) {
        const int gi = p + li * P;
        const double inv = 1.0 / __ldg(A.dA + gi);
        const double r0 = __ldg(A.rhs_a[0] + gi), r1 = nrhs > 1 ? __ldg(A.rhs_a[1] + gi) : 0.0;
        const double t0 = r0 * inv, t1 = r1 * inv;
        if (li >= r_lo && li < r_hi) {
            part[6] += r0 * t0;
            part[7] += r1 * t1;
            oia[li - r_lo] = inv;
        }
        vect[li] = make_double2(t0, t1);
    }
    for (int c = tid; c < n_own_c; c += kB2Threads) oib[c] = 1.0 / __ldg(A.dB + q + (c_lo + c) * Q);
    __syncthreads();

#ifdef REGOT_PCG_TIMING  // per-section cycle counts per CTA (experiments only)
    long long tsec[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tprev = clock64();
#define B2_TICK(i)                         \
    {                                      \
        __syncthreads();                   \
        const long long now__ = clock64(); \
        tsec[i] += now__ - tprev;          \
        tprev = now__;                     \
    }
#else
#define B2_TICK(i)
#endif
    double gamma[2] = {0.0, 0.0}, gamma0[2] = {0.0, 0.0}, gamma_old[2] = {1.0, 1.0}, alpha_old[2] = {1.0, 1.0};
    bool done[2] = {false, false}, broke = false;
    int iters[2] = {0, 0}, it = 0;
    bool init = true;
    unsigned int round = A.round0;
#pragma unroll 1
    for (;; ++round) {
        if (!init) {
            // owners publish z of their column slice; everybody collects its block column's
            for (int item = tid; item < 2 * n_own_c; item += kB2Threads) fw_post(x4_col + ((size_t)c_lo * 2 + item) * 2, oz[item], round);
            fw_gather(x4_col, reinterpret_cast<double*>(vecz), 2 * Cq, 1, 0, round);
            __syncthreads();
            B2_TICK(0)
            block_phase(&s_copy[0], val, nval, vecz, nullptr, x1_mine, round, hpart, bcast + 12);
            B2_TICK(1)
            // owner: the Q partials of my rows, summed in block order; t = D1^-1 sum goes to the block row
            fw_gather(x1_own, xbuf, 2 * n_own_r, Q, 2 * SR, round);
            __syncthreads();
            for (int item = tid; item < 2 * n_own_r; item += kB2Threads) {
                double s = 0.0;
                for (int src = 0; src < Q; ++src) s += xbuf[src * 2 * n_own_r + item];
                fw_post(x2_row + ((size_t)r_lo * 2 + item) * 2, s * oia[item >> 1], round);
            }
            B2_TICK(2)
            fw_gather(x2_row, reinterpret_cast<double*>(vect), 2 * Rp, 1, 0, round);
            __syncthreads();
            B2_TICK(3)
        }
        // column phase: partial B' t of my block; z . (B' t) rides along
        block_phase(&s_copy[1], val, nval, vect, vecz, x3_mine, round, hpart, part + 4);
        if (init) part[4] = part[5] = 0.0;
        B2_TICK(4)
        // owner: u = sum of the P partials of my columns, then the new r/z (set-up) or w = D2 z - u
        fw_gather(x3_own, xbuf, 2 * n_own_c, P, 2 * SC, round);
        __syncthreads();
        for (int item = tid; item < 2 * n_own_c; item += kB2Threads) {
            const int c = item >> 1, k = item & 1;
            double u = 0.0;
            for (int src = 0; src < P; ++src) u += xbuf[src * 2 * n_own_c + item];
            const double inv = oib[c], d = __ldg(A.dB + q + (c_lo + c) * Q);
            if (init) {
                const double rb = k < nrhs ? __ldg((k ? A.rhs_b[1] : A.rhs_b[0]) + q + (c_lo + c) * Q) : 0.0;
                const double r = rb - u, z = r * inv;  // Schur right-hand side
                orr[item] = r;
                oz[item] = z;
                ox[item] = 0.0;
                op[item] = 0.0;
                os[item] = 0.0;
                const double g0 = rb * (rb * inv);
                if (k) {
                    part[1] += r * z;
                    part[3] += d * z * z;
                    part[7] += g0;
                } else {
                    part[0] += r * z;
                    part[2] += d * z * z;
                    part[6] += g0;
                }
            } else {
                ow[item] = d * oz[item] - u;
            }
        }
        B2_TICK(5)
        // everybody's partial dot products, summed in CTA order
        {
            const double mine = block_sum8(part, scratch);
            if (tid < 8 * kB2Warps && (tid & (kB2Warps - 1)) == 0) {
                fw_post(A.x5 + ((size_t)b * 8 + tid / kB2Warps) * 2, mine, round);
                if (tid < 4 * kB2Warps) bcast[8 + tid / kB2Warps] = mine;  // my partials of gamma and sum dB z^2 stay valid until my next update
            }
        }
        fw_gather(A.x5, stage, 8 * G, 1, 0, round);
        __syncthreads();
        if (warp < 8) {
            double s = 0.0;
            for (int c = lane; c < G; c += 32) s += stage[c * 8 + warp];
            s = warp_sum(s);
            if (lane == 0) bcast[warp] = s;
        }
        __syncthreads();
        double tot[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            tot[k] = bcast[k];
            part[k] = 0.0;
        }
        B2_TICK(6)

        if (init) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                gamma[k] = tot[k];
                gamma0[k] = tot[6 + k];
                done[k] = (k >= nrhs) || gamma0[k] == 0.0 || !(gamma[k] > A.tol2 * gamma0[k]);
                if (A.fixed_iters > 0 && k < nrhs) done[k] = false;
            }
            if (tid == 0) {
#pragma unroll
                for (int k = 0; k < 4; ++k) part[k] = bcast[8 + k];
            }
            init = false;
        } else {
            double al[2], be[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                al[k] = be[k] = 0.0;
                if (done[k]) continue;
                gamma[k] = tot[k];
                if (it > 0 && !(gamma[k] > A.tol2 * gamma0[k]) && A.fixed_iters == 0) {
                    done[k] = true;
                    continue;
                }
                const double delta = tot[2 + k] - tot[4 + k];  // z'D2 z - z'B'D1^-1 B z
                be[k] = (it == 0) ? 0.0 : gamma[k] / gamma_old[k];
                const double denom = delta - be[k] * gamma[k] / alpha_old[k];  // = p'Sp
                if (!(denom > 0.0) && A.fixed_iters == 0) broke = true;        // not positive definite (or NaN)
                al[k] = gamma[k] / denom;
                gamma_old[k] = gamma[k];
                alpha_old[k] = al[k];
                ++iters[k];
            }
            ++it;
            if (!broke && !(done[0] && done[1])) {
                // p = z + beta p, s = w + beta s, x += alpha p, r -= alpha s, z = D2^-1 r on the owned slice
                for (int item = tid; item < 2 * n_own_c; item += kB2Threads) {
                    const int k = item & 1;
                    if (k ? done[1] : done[0]) continue;  // a finished system is frozen; its partials are not used any more
                    const double bek = k ? be[1] : be[0], alk = k ? al[1] : al[0];
                    const double inv = oib[item >> 1], d = __ldg(A.dB + q + (c_lo + (item >> 1)) * Q);
                    const double pn = oz[item] + bek * op[item], sn = ow[item] + bek * os[item];
                    const double xn = ox[item] + alk * pn, rn = orr[item] - alk * sn, zn = rn * inv;
                    op[item] = pn;
                    os[item] = sn;
                    ox[item] = xn;
                    orr[item] = rn;
                    oz[item] = zn;
                    if (k) {
                        part[1] += rn * zn;
                        part[3] += d * zn * zn;
                    } else {
                        part[0] += rn * zn;
                        part[2] += d * zn * zn;
                    }
                }
            }
        }
        B2_TICK(7)
        bool all_done = done[0] && done[1];
        if (A.fixed_iters > 0) all_done = it >= A.fixed_iters;
        if (all_done || broke || it >= A.max_iter) break;
    }
#ifdef REGOT_PCG_TIMING
    if (tid == 0)
        for (int k = 0; k < 8; ++k) A.out[4 + (size_t)b * 8 + k] = (double)tsec[k];
#endif
#undef B2_TICK
    // ---- back-substitution: owners publish x, one more row phase, x_a = D1^-1 (r_a - B x_b) on the owned rows ----
    ++round;
    for (int item = tid; item < 2 * n_own_c; item += kB2Threads) {
        const int k = item & 1;
        fw_post(x4_col + ((size_t)c_lo * 2 + item) * 2, ox[item], round);
        if (k < nrhs) (k ? A.sol_b[1] : A.sol_b[0])[q + (c_lo + (item >> 1)) * Q] = ox[item];
    }
    fw_gather(x4_col, reinterpret_cast<double*>(vecz), 2 * Cq, 1, 0, round);
    __syncthreads();
    block_phase(&s_copy[0], val, nval, vecz, nullptr, x1_mine, round, hpart, bcast + 12);
    fw_gather(x1_own, xbuf, 2 * n_own_r, Q, 2 * SR, round);
    __syncthreads();
    for (int item = tid; item < 2 * n_own_r; item += kB2Threads) {
        const int k = item & 1, gi = p + (r_lo + (item >> 1)) * P;
        double s = 0.0;
        for (int src = 0; src < Q; ++src) s += xbuf[src * 2 * n_own_r + item];
        if (k < nrhs) (k ? A.sol_a[1] : A.sol_a[0])[gi] = (__ldg((k ? A.rhs_a[1] : A.rhs_a[0]) + gi) - s) / __ldg(A.dA + gi);
    }
    if (b == 0 && tid == 0) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            if (k < nrhs) A.sol_b[k][A.mfree] = 0.0;
            A.out[k] = (double)iters[k];
        }
        A.out[3] = broke ? 1.0 : 0.0;
        // the host may go on as soon as the flags are there; everything it launches next is ordered behind the grid
        if (A.mbox) {
            const double post[4] = {(double)iters[0], (double)iters[1], 0.0, broke ? 1.0 : 0.0};
            mailbox_post(A.mbox, post, 4, A.mseq);
        }
    }
}

// ---- host ---------------------------------------------------------------------------------------------------
static int gcd_int(int a, int b) { return b ? gcd_int(b, a % b) : a; }

// largest coprime P x Q <= sm_count with 8 <= Q <= 16 (block rows exchange among Q CTAs, block columns among P)
static void pick_grid(const regot_ctx* ctx, int& P, int& Q)
{
    if (ctx->pcg_blocks_p > 0 && ctx->pcg_blocks_q > 0) {
        P = ctx->pcg_blocks_p;
        Q = ctx->pcg_blocks_q;
        return;
    }
    int best = 0;
    P = Q = 1;
    for (int q = 8; q <= 16; ++q) {
        int p = ctx->sm_count / q;
        while (p > 1 && gcd_int(p, q) != 1) --p;
        if (p * q >= best && p >= 1) {
            best = p * q;
            P = p;
            Q = q;
        }
    }
}

// Build the block plan of the current pattern; everything is enqueued on st, the summary lands in pinned memory
// (valid after the caller's next synchronisation with st).  csc2csr[t] = CSR position of CSC entry t.
void build_pcg_blocks_plan(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, regot_sparse& S, const int* csc2csr)
{
    PcgBlocksPlan& Q2 = S.blocks;
    Q2.fits = false;
    Q2.pending = false;
    const int nloc = (int)S.nloc, mfree = std::max((int)S.m - 1, 0), nnz = (int)S.nnz;
    if (ctx->pcg_blocks == 0 || ctx->world != 1 || nnz < 1 || nloc < 64 || mfree < 64) return;
    // far too large for shared memory: do not even try (12 B per entry and copy at the very least)
    if ((long)nnz * 12 > (long)ctx->sm_count * kPcgSmemBudget) return;
    int P, Q;
    pick_grid(ctx, P, Q);
    if (P * Q > ctx->sm_count || gcd_int(P, Q) != 1) raise(REGOT_E_VALIDATION, "pcg blocks: grid must be coprime and fit the device");
    const int G = P * Q, R = (nloc + P - 1) / P, C = (mfree + Q - 1) / Q;
    if (R > 32000 || C > 32000) return;
    Q2.P = P;
    Q2.Q = Q;
    Q2.R = R;
    Q2.C = C;
    Q2.SR = (R + Q - 1) / Q;
    Q2.SC = (C + P - 1) / P;
    auto thr = [](long avg) {
        int L = 16;
        while (L < kB2MaxL && L < 4 * avg) L *= 2;
        return L;
    };
    Q2.Lr = thr((long)nnz / std::max(1L, (long)G * R) + 1);
    Q2.Lc = thr((long)nnz / std::max(1L, (long)G * C) + 1);
    const Lay32 T = lay32(R, C);
    Q2.cnt.ensure((size_t)G * (R + C));
    Q2.vpos.ensure((size_t)G * (R + C));
    Q2.hdr.ensure((size_t)G * kPcgBlocksHdrInts + 8);
    Q2.a32.ensure((size_t)G * T.stride);
    // upper bounds of the arenas: every entry once per copy plus padding (< 32 slots per distinct length and copy)
    const size_t pad_slots = (size_t)G * 32 * (kB2MaxL + 2);
    Q2.a16.ensure(3 * (size_t)nnz + 3 * pad_slots + (size_t)G * (R + C + 64));
    Q2.asrc.ensure((size_t)nnz + pad_slots + (size_t)G * 8);
    Q2.rowslot.ensure((size_t)nnz + 1);
    int* cnt_r = Q2.cnt.p;
    int* cnt_c = Q2.cnt.p + (size_t)G * R;
    int* vpos_r = Q2.vpos.p;
    int* vpos_c = Q2.vpos.p + (size_t)G * R;
    int* summary = Q2.hdr.p + (size_t)G * kPcgBlocksHdrInts;
    RG_CUDA(cudaMemsetAsync(Q2.cnt.p, 0, sizeof(int) * (size_t)G * (R + C), st));
    const int g1 = (int)std::max<long>(1, std::min<long>(((long)nnz + 255) / 256, 8L * ctx->sm_count));
    k_b2_count<<<g1, 256, 0, st>>>(nnz, P, Q, R, C, S.row.p, S.col.p, cnt_r, cnt_c);
    k_b2_layout<<<G, 256, 0, st>>>(P, Q, R, C, nloc, mfree, Q2.Lr, Q2.Lc, cnt_r, cnt_c, vpos_r, vpos_c, Q2.a32.p, Q2.hdr.p);
    k_b2_offsets<<<1, 32, 0, st>>>(P, Q, R, C, Q2.SR, Q2.SC, Q2.hdr.p, summary);
    k_b2_fill<<<G, 256, 0, st>>>(P, Q, R, C, nloc, mfree, Q2.hdr.p, vpos_r, vpos_c, Q2.a16.p, Q2.asrc.p);
    const int gr = (int)std::max<long>(1, std::min<long>(((long)nloc + 7) / 8, 16L * ctx->sm_count));
    const int gc = (int)std::max<long>(1, std::min<long>(((long)mfree + 7) / 8, 16L * ctx->sm_count));
    k_b2_scatter<true><<<gr, 256, 0, st>>>(nloc, P, Q, R, C, S.rowptr.p, S.col.p, nullptr, Q2.hdr.p, vpos_r, Q2.a32.p, Q2.a16.p,
                                           Q2.asrc.p, Q2.rowslot.p);
    k_b2_scatter<false><<<gc, 256, 0, st>>>(mfree, P, Q, R, C, S.cscptr.p, S.cscrow.p, csc2csr, Q2.hdr.p, vpos_c, Q2.a32.p,
                                            Q2.a16.p, Q2.asrc.p, Q2.rowslot.p);
    RG_CUDA(cudaGetLastError());
    ctx->launches += 6;
    if (!ws.h_blocks) RG_CUDA(cudaMallocHost((void**)&ws.h_blocks, sizeof(int) * 8));
    RG_CUDA(cudaMemcpyAsync(ws.h_blocks, summary, sizeof(int) * 4, cudaMemcpyDeviceToHost, st));
    Q2.pending = true;
    Q2.stamp = S.structure_stamp;
}

// after the stream has been synchronised: does the plan fit?
void finish_pcg_blocks_plan(regot_ctx* ctx, SparseWS& ws, regot_sparse& S)
{
    PcgBlocksPlan& Q2 = S.blocks;
    if (!Q2.pending) return;
    Q2.pending = false;
    Q2.smem = ws.h_blocks[0];
    Q2.fits = ws.h_blocks[1] == 0 && Q2.smem <= kPcgSmemBudget;
    static const bool show = std::getenv("REGOT_B200_PCG_BLOCKS_INFO") != nullptr;
    if (show)
        std::fprintf(stderr, "pcg blocks: %d x %d blocks, slices %d x %d, L %d/%d, smem %d B, %s\n", Q2.P, Q2.Q, Q2.R, Q2.C, Q2.Lr, Q2.Lc,
                     Q2.smem, Q2.fits ? "fits" : "does not fit");
    (void)ctx;
}

static int pcg_blocks_launch(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, const regot_sparse& S, int nrhs,
                             const DVec* const* rhs, DVec* const* sol, double rtol, int max_iter)
{
    const PcgBlocksPlan& Q2 = S.blocks;
    const int nloc = (int)S.nloc, mfree = std::max((int)S.m - 1, 0), G = Q2.P * Q2.Q;
    static bool attr_set = false;
    if (!attr_set) {
        RG_CUDA(cudaFuncSetAttribute(k_pcg_blocks, cudaFuncAttributeMaxDynamicSharedMemorySize, kPcgSmemBudget));
        attr_set = true;
    }
    BlocksParams A;
    std::memset(&A, 0, sizeof(A));
    A.nloc = nloc;
    A.mfree = mfree;
    A.nrhs = nrhs;
    A.max_iter = max_iter;
    A.fixed_iters = 0;
    if (const char* e = std::getenv("REGOT_B200_PCG_FIXED_ITERS")) A.fixed_iters = std::atoi(e);
    A.P = Q2.P;
    A.Q = Q2.Q;
    A.R = Q2.R;
    A.C = Q2.C;
    A.SR = Q2.SR;
    A.SC = Q2.SC;
    A.tol2 = rtol * rtol;
    A.hdr = Q2.hdr.p;
    A.a16 = Q2.a16.p;
    A.a32 = Q2.a32.p;
    A.asrc = Q2.asrc.p;
    A.val = S.val.p;
    A.dA = S.dA.p;
    A.dB = S.dB.p;
    for (int k = 0; k < 2; ++k) {
        const int kk = k < nrhs ? k : 0;
        A.rhs_a[k] = rhs[kk]->a.p;
        A.rhs_b[k] = rhs[kk]->b.p;
        sol[kk]->ensure(S.nloc, S.m);
        A.sol_a[k] = sol[kk]->a.p;
        A.sol_b[k] = sol[kk]->b.p;
    }
    // the five exchanges, in words
    const size_t n1 = (size_t)G * Q2.Q * Q2.SR * 4, n2 = (size_t)Q2.P * Q2.R * 4, n3 = (size_t)G * Q2.P * Q2.SC * 4,
                 n4 = (size_t)Q2.Q * Q2.C * 4, n5 = (size_t)G * 8 * 2;
    const size_t words = n1 + n2 + n3 + n4 + n5;
    const unsigned int rounds = (unsigned int)std::max(max_iter, A.fixed_iters) + 8u;
    if (ws.blocks_xchg.n < words || ws.blocks_round > 0x7fff0000u - rounds || ws.blocks_round == 0) {
        // (re)start the round numbers: all words zero, first round 1
        ws.blocks_xchg.ensure(words);
        RG_CUDA(cudaMemsetAsync(ws.blocks_xchg.p, 0, sizeof(u64) * ws.blocks_xchg.n, st));
        ws.blocks_round = 1;
    }
    A.x1 = ws.blocks_xchg.p;
    A.x2 = A.x1 + n1;
    A.x3 = A.x2 + n2;
    A.x4 = A.x3 + n3;
    A.x5 = A.x4 + n4;
    A.round0 = ws.blocks_round;
    ws.blocks_round += rounds;
    ws.cg_scal.ensure(16 + (size_t)G * 8);
    if (!ws.h_cg) RG_CUDA(cudaMallocHost((void**)&ws.h_cg, sizeof(double) * 4096));
    A.out = ws.cg_scal.p;
    ws.cg_mbox.ensure();
    A.mbox = ws.cg_mbox.data;
    A.mseq = ws.cg_mbox.next();
    void* args[] = {&A};
    {
        ProfScope prof(ctx, st, 5);
        RG_CUDA(cudaLaunchCooperativeKernel((const void*)k_pcg_blocks, dim3(G), dim3(kB2Threads), args, (size_t)Q2.smem, st));
    }
    ++ctx->launches;
    ws.cg_mbox.wait(st);
    for (int k = 0; k < 4; ++k) ws.h_cg[k] = ws.cg_mbox.data[k];
#ifdef REGOT_PCG_TIMING
    {
        RG_CUDA(cudaMemcpyAsync(ws.h_cg + 8, ws.cg_scal.p + 4, sizeof(double) * (size_t)G * 8, cudaMemcpyDeviceToHost, st));
        RG_CUDA(cudaStreamSynchronize(st));
        const char* nm[8] = {"z_gather", "row", "x1_sum", "t_gather", "col", "x3_sum", "dots", "update"};
        std::fprintf(stderr, "pcg_blocks kcycles min/avg/max over CTAs:");
        for (int k = 0; k < 8; ++k) {
            double mn = 1e300, mx = 0.0, sum = 0.0;
            for (int c = 0; c < G; ++c) {
                const double v = ws.h_cg[8 + (size_t)c * 8 + k];
                mn = std::min(mn, v);
                mx = std::max(mx, v);
                sum += v;
            }
            std::fprintf(stderr, " %s %.0f/%.0f/%.0f", nm[k], mn * 1e-3, sum / G * 1e-3, mx * 1e-3);
        }
        std::fprintf(stderr, " | iters %.0f\n", ws.h_cg[0]);
    }
#endif
    static const bool show_iters = std::getenv("REGOT_B200_PCG_ITERS") != nullptr;  // experiments
    if (show_iters) std::fprintf(stderr, "pcg iters (blocks): g-system %d, u-system %d\n", (int)ws.h_cg[0], nrhs > 1 ? (int)ws.h_cg[1] : -1);
    if (ws.h_cg[3] != 0.0) return -1;
    int it = 0;
    for (int k = 0; k < nrhs; ++k) it = std::max(it, (int)ws.h_cg[k]);
    return it;
}

int pcg_schur_blocks(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, const regot_sparse& S, int nrhs, const DVec* const* rhs,
                     DVec* const* sol, double rtol, int max_iter)
{
    int it = 0;
    for (int k0 = 0; k0 < nrhs; k0 += 2) {
        const int r = pcg_blocks_launch(ctx, st, ws, S, std::min(2, nrhs - k0), rhs + k0, sol + k0, rtol, max_iter);
        if (r < 0) return -1;
        it = std::max(it, r);
    }
    return it;
}

}  // namespace rg
