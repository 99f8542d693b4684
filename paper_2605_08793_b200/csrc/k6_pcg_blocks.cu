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

#include <cooperative_groups.h>

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

// doubles of the owner's collection buffers: the Q x 2 SR row partial sums and the P x 2 SC column partial sums.  Through
// L2 they are copied there one after the other (one buffer); inside a cluster the row partials are written by the
// other CTAs at their own pace, so the two do not share
__host__ __device__ __forceinline__ long b2_xbuf_doubles(int SR, int SC, int P, int Q, int cluster)
{
    const long x1 = 2L * Q * SR, x3 = 2L * P * SC;
    return cluster ? x1 + x3 : (x1 > x3 ? x1 : x3);
}
// doubles of the staging the mat-vec phases write their sums to before they are shipped: through L2 the collection
// buffer itself serves (it is filled after the sums have left); inside a cluster other CTAs write into that buffer at
// their own pace, so the row sums (and, in a single cluster, the column sums) get their own staging, plus the t slice
// an owner sends to its block row
__host__ __device__ __forceinline__ long b2_staging_doubles(int SR, int SC, int P, int Q, int cluster)
{
    if (!cluster) return 0;
    return 2L * Q * SR + (P == 1 ? 2L * P * SC : 0L) + 2L * SR;
}

// dynamic shared memory of the solve kernel for one block (the carve-up at the top of k_pcg_blocks)
__host__ __device__ __forceinline__ long b2_smem_need(const int* h, int R, int C, int SR, int SC, int P, int Q, int cluster)
{
    const int nval = h[kH_NSL_R] + h[kH_NHE_R];
    const int segcap_r = h[kH_NHE_R] / 128 + h[kH_NHV_R], segcap_c = h[kH_NHE_C] / 128 + h[kH_NHV_C];
    const int tables = 2 * h[kH_NCH_R] + 3 * h[kH_NHV_R] + 2 * h[kH_NCH_C] + 3 * h[kH_NHV_C];
    const int derived = (h[kH_NHV_R] + h[kH_NHV_C]) + 2 + segcap_r + segcap_c + 4;
    return (long)(((nval + 1) * 8 + 15) & ~15) + 16L * C + 16L * R + 16L * (segcap_r > segcap_c ? segcap_r : segcap_c) + 2L * lay16(h).size +
           (long)(((tables + derived) * 4 + 15) & ~15) + 8L * (6 * 2 * SC + 2 * SC + SR) + 8L * (b2_xbuf_doubles(SR, SC, P, Q, cluster) + b2_staging_doubles(SR, SC, P, Q, cluster)) + 8L * (8 * P * Q) + 8L * (16 + 8 * kB2Warps) + 256 + 64 + 16 + kB2Slack;
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
__global__ void k_b2_offsets(int P, int Q, int R, int C, int SR, int SC, int cluster, int* __restrict__ hdr, int* __restrict__ summary)
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
        const long need = b2_smem_need(h, R, C, SR, SC, P, Q, cluster);
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
    const double* mB;  // Jacobi preconditioner: diag of the Schur complement (k4_sparse.cu compute_schur_diag)
    const double* rhs_a[2];
    const double* rhs_b[2];
    double* sol_a[2];
    double* sol_b[2];
    u64 *x1, *x2, *x3, *x4, *x5;  // flagged words of the five exchanges
    unsigned int round0;          // round number of this launch's first exchange
    int cluster;                  // CTAs of a block row form a thread-block cluster: their exchanges (X1, X2; with P == 1 all of them) go through distributed shared memory
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
// n flagged doubles at src -> dst (shared memory), all threads of the CTA, 4 loads in flight per thread
__device__ __noinline__ void fw_gather(const u64* src, double* dst, int n, unsigned int round)
{
#pragma unroll 1
    for (int i0 = threadIdx.x; i0 < n; i0 += kB2Threads * 4) {
        double v[4];
        unsigned pend = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (i0 + u * kB2Threads < n) pend |= 1u << u;
        const unsigned valid = pend;
        while (pend) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if ((pend >> u) & 1u)
                    if (fw_try(src + 2 * (size_t)(i0 + u * kB2Threads), round, v[u])) pend &= ~(1u << u);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if ((valid >> u) & 1u) dst[i0 + u * kB2Threads] = v[u];
    }
}

constexpr int kB2Seg = 128;  // entries of a heavy line one warp sums at a time

// shared-memory accesses of the mat-vec phase by 32-bit shared-window address: the phase is an out-of-line function,
// and through generic pointers the compiler would emit generic loads (slower than ld.shared)
__device__ __forceinline__ int lds_u16(uint32_t a)
{
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return (int)v;
}
__device__ __forceinline__ int lds_s32(uint32_t a)
{
    int v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_f64x2_b(uint32_t a, double x, double y)
{
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y) : "memory");
}

// ---- exchanges inside a thread-block cluster: remote shared-memory stores that complete on the receiver's mbarrier ----
// The receiver arms its barrier with the number of bytes a round brings (expect_tx) and waits for the phase; senders
// write plain doubles straight into the receiver's buffer (st.async ... complete_tx): no flags, no fences, no copies.
__device__ __forceinline__ uint32_t map_rank(uint32_t saddr, int rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rmbar)
{
    asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
                 "l"(__double_as_longlong(v)), "r"(rmbar)
                 : "memory");
}
__device__ __forceinline__ void st_async_f64x2(uint32_t raddr, double a, double b, uint32_t rmbar)
{
    asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
                 "l"(__double_as_longlong(a)), "l"(__double_as_longlong(b)), "r"(rmbar)
                 : "memory");
}
// all threads of the CTA: wait until the round's `bytes` have landed (thread 0 arms the barrier; data written by
// other CTAs of the cluster: acquire at cluster scope)
__device__ __forceinline__ void cluster_inbox_wait(uint32_t mbar, uint32_t bytes, uint32_t& parity)
{
    if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
    uint32_t ok;
    do {
        asm volatile(
            "{ .reg .pred p;\n"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(mbar), "r"(parity)
            : "memory");
    } while (!ok);
    parity ^= 1u;
}

struct BlockCopy {  // one copy (rows or columns) of the CTA's block in shared memory (shared-window addresses)
    uint32_t ell;     // u16 per entry: local index into the gathered slice
    uint32_t ref;     // column copy: u16 per entry, position in `val` (row copy: 0, the entry's own position)
    uint32_t lov;     // u16 per sorted position: local line
    uint32_t chunk;   // int pairs (first slot, width) per 32-line chunk
    uint32_t heavy;   // int triples (line, first entry, length) per heavy line
    uint32_t hfirst;  // int per heavy line: its first segment
    uint32_t hseg;    // int per segment: heavy line
    int nv, nch, nsl, nhv, nseg;
};

// One mat-vec phase over the CTA's block: lines are the block's rows and `vec` the z (or x) slice of the block
// column, or lines are its columns and `vec` the t slice of the block row.  Work items: segments of heavy lines
// first, then the 32-line chunks by decreasing width.  The two sums of line l land in out[l] (shared memory, 16 B per
// line, line order = owner order: the caller ships each owner's slice in one piece); with zvec != 0 (column phase)
// z . (B' t) is accumulated per system into dc[0..1] of this thread.  val, vec, zvec, out, hpart: shared-window
// addresses.  Ends with a CTA barrier: out is complete.
__device__ __noinline__ void block_phase(uint32_t Bp, uint32_t val, int zero_slot, uint32_t vec, uint32_t zvec, uint32_t out,
                                         uint32_t hpart, double* dc)
{
    BlockCopy B;
    {
        uint32_t* w = reinterpret_cast<uint32_t*>(&B);
#pragma unroll
        for (int k = 0; k < (int)(sizeof(BlockCopy) / 4); ++k) w[k] = (uint32_t)lds_s32(Bp + 4 * k);
    }
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
            const int h = lds_s32(B.hseg + 4 * item), sidx = item - lds_s32(B.hfirst + 4 * h);
            const int beg = B.nsl + lds_s32(B.heavy + 12 * h + 4) + sidx * kB2Seg;
            const int len = min(kB2Seg, lds_s32(B.heavy + 12 * h + 8) - sidx * kB2Seg);
#pragma unroll 2
            for (int t = lane; t < len; t += 32) {
                const int s = beg + t;
                const double v = lds_f64(val + 8u * (uint32_t)(B.ref ? lds_u16(B.ref + 2 * s) : s));
                const double2 g = lds_f64x2(vec + 16u * (uint32_t)lds_u16(B.ell + 2 * s));
                a0 = __fma_rn(v, g.x, a0);
                a1 = __fma_rn(v, g.y, a1);
            }
            a0 = warp_sum(a0);
            a1 = warp_sum(a1);
            if (lane == 0) sts_f64x2_b(hpart + 16u * (uint32_t)item, a0, a1);
            continue;
        }
        const int c = item - B.nseg;
        const int base = lds_s32(B.chunk + 8 * c) + lane, w = lds_s32(B.chunk + 8 * c + 4);
#pragma unroll 1
        for (int k0 = 0; k0 < w; k0 += 4) {
            int ix[4], vi[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int s = base + 32 * (k0 + u);
                const bool ok = k0 + u < w;
                const int raw = lds_u16(B.ell + 2 * s);
                ix[u] = ok ? raw : 0;
                const int rr = B.ref ? lds_u16(B.ref + 2 * s) : s;
                vi[u] = ok ? rr : zero_slot;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double v = lds_f64(val + 8u * (uint32_t)vi[u]);
                const double2 g = lds_f64x2(vec + 16u * (uint32_t)ix[u]);
                a0 = __fma_rn(v, g.x, a0);
                a1 = __fma_rn(v, g.y, a1);
            }
        }
        const int vpos = 32 * c + lane;
        if (vpos < B.nv) {
            const uint32_t line = (uint32_t)lds_u16(B.lov + 2 * vpos);
            sts_f64x2_b(out + 16u * line, a0, a1);
            if (zvec) {
                const double2 z = lds_f64x2(zvec + 16u * line);
                dc0 = __fma_rn(z.x, a0, dc0);
                dc1 = __fma_rn(z.y, a1, dc1);
            }
        }
    }
    if (B.nhv > 0) {  // uniform over the CTA
        __syncthreads();
#pragma unroll 1
        for (int h = threadIdx.x; h < B.nhv; h += kB2Threads) {
            double a0 = 0.0, a1 = 0.0;
            const int sg1 = lds_s32(B.hfirst + 4 * h + 4);
#pragma unroll 1
            for (int sg = lds_s32(B.hfirst + 4 * h); sg < sg1; ++sg) {
                const double2 hp = lds_f64x2(hpart + 16u * (uint32_t)sg);
                a0 += hp.x;
                a1 += hp.y;
            }
            const uint32_t line = (uint32_t)lds_s32(B.heavy + 12 * h);
            sts_f64x2_b(out + 16u * line, a0, a1);
            if (zvec) {
                const double2 z = lds_f64x2(zvec + 16u * line);
                dc0 = __fma_rn(z.x, a0, dc0);
                dc1 = __fma_rn(z.y, a1, dc1);
            }
        }
    }
    dc[0] = dc0;
    dc[1] = dc1;
    __syncthreads();
}

// Ship the staged sums (out of block_phase: [owner][slice][2] doubles) to their owners.  Through L2: flagged words,
// written by all threads in address order (whole lines of the owner's region instead of one 16-byte piece per
// line).  Inside a cluster: one bulk copy per owner into its collection buffer, completing on its barrier.
__device__ __forceinline__ void ship_sums(bool dsmem, const double* staged, int nowner, int slice, int me, int nsrc, u64* xbase,
                                          uint32_t xlocal, uint32_t mbar, int only_rank, unsigned int round)
{
    if (dsmem) {
        fence_proxy_async();  // the sums were written through the generic proxy, the copy engine reads them
        __syncthreads();
        if ((int)threadIdx.x < nowner) {
            const int o = threadIdx.x, dst_rank = only_rank >= 0 ? only_rank : o;
            const uint32_t bytes = 16u * (uint32_t)slice;
            asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             map_rank(xlocal + (uint32_t)me * bytes, dst_rank)),
                         "r"(smem_u32(staged) + (uint32_t)o * bytes), "r"(bytes), "r"(map_rank(mbar, dst_rank))
                         : "memory");
        }
        return;
    }
    const int per = 2 * slice, n = nowner * per;
#pragma unroll 1
    for (int i = threadIdx.x; i < n; i += kB2Threads) {
        const int o = i / per;
        fw_post(xbase + 2 * ((size_t)(o * nsrc + me) * per + (i - o * per)), staged[i], round);
    }
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
// the CTA's 8 partial dot products -> its slots of the X5 exchange; the first four (gamma, sum dB z^2) are also kept
// in bcast[8..11]: they stay valid until the owner's next update
__device__ __noinline__ void post_dots(const double* part, double* scratch, double* bcast, u64* x5_mine, int ndst, uint32_t stage_mine,
                                       uint32_t mbar, unsigned int round)
{
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = part[k];
    const double mine = block_sum8(v, scratch);
    const int tid = threadIdx.x;
    if (tid < 8 * kB2Warps && (tid & (kB2Warps - 1)) == 0) {
        const int k = tid / kB2Warps;
        if (ndst == 0) fw_post(x5_mine + k * 2, mine, round);
#pragma unroll 1
        for (int dst = 0; dst < ndst; ++dst)  // single cluster: straight into everybody's staging area
            st_async_f64(map_rank(stage_mine + 8u * (uint32_t)k, dst), mine, map_rank(mbar, dst));
        if (k < 4) bcast[8 + k] = mine;
    }
}
static_assert(2 * sizeof(BlockCopy) <= 256 && sizeof(BlockCopy) % 4 == 0, "descriptor area of the shared-memory plan");

// Owners publish their slice of a beta-space vector (z, or the solution x) and every CTA collects its block
// column's; with a single cluster (P == 1) the owner of the block column is this CTA and the slice is simply copied.
__device__ __forceinline__ void publish_slice(bool local, u64* column, int first, const double* src, int n_mine, double* dst,
                                              int n_all, unsigned int round)
{
    if (local) {
        for (int item = threadIdx.x; item < n_mine; item += kB2Threads) dst[item] = src[item];
        return;
    }
    for (int item = threadIdx.x; item < n_mine; item += kB2Threads) fw_post(column + 2 * (size_t)(first + item), src[item], round);
    fw_gather(column, dst, n_all, round);
}

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
    // What other CTAs of the cluster write into comes first: its offsets depend on the grid only, so a remote CTA
    // finds it at the same place in my shared memory as in its own.  Everything sized by this block follows.
    const bool cl = A.cluster != 0, one = cl && P == 1;
    unsigned char* sp = smem;
    // barriers of the exchanges that stay inside the cluster: row partial sums -> xbuf1, t -> vect, (single cluster:)
    // column partial sums -> xbuf3, dot products -> stage
    uint64_t* mbars = reinterpret_cast<uint64_t*>(sp);
    sp += 64;
    const uint32_t mb1 = smem_u32(mbars), mb2 = mb1 + 8, mb3 = mb1 + 16, mb5 = mb1 + 24;
    uint32_t ph1 = 0, ph2 = 0, ph3 = 0, ph5 = 0;
    double2* vect = reinterpret_cast<double2*>(sp);
    sp += 16 * (size_t)A.R;
    double* xbuf1 = reinterpret_cast<double*>(sp);  // partial sums collected by the owner: Q x 2 SR of its rows ...
    double* xbuf3 = xbuf1 + (cl ? 2 * Q * SR : 0);  // ... and P x 2 SC of its columns (one buffer when both come through L2)
    sp += 8 * (size_t)b2_xbuf_doubles(SR, SC, P, Q, A.cluster);
    // where the phases put their sums before they are shipped ([owner][slice][2]; lines beyond the last real one stay 0)
    double* stg_r = cl ? reinterpret_cast<double*>(sp) : xbuf1;
    double* stg_c = one ? stg_r + 2 * Q * SR : xbuf3;
    double* tloc = stg_r + 2 * Q * SR + (one ? 2 * P * SC : 0);  // cluster: the t slice I own, as it goes out
    sp += 8 * (size_t)b2_staging_doubles(SR, SC, P, Q, A.cluster);
    double* stage = reinterpret_cast<double*>(sp);  // 8 G: everybody's partial dot products
    sp += 8 * (size_t)(8 * G);
    double2* vecz = reinterpret_cast<double2*>(sp);
    sp += 16 * (size_t)A.C;
    double* val = reinterpret_cast<double*>(sp);
    sp += ((nval + 1) * 8 + 15) & ~15;
    double2* hpart = reinterpret_cast<double2*>(sp);
    sp += 16 * (size_t)max(segcap_r, segcap_c);
    u16* s16 = reinterpret_cast<u16*>(sp);
    sp += 2 * (size_t)L16.size;
    int* s32 = reinterpret_cast<int*>(sp);
    const int n_tables = 2 * Br.nch + 3 * Br.nhv + 2 * Bc.nch + 3 * Bc.nhv;
    const int n_derived = (Br.nhv + Bc.nhv) + 2 + segcap_r + segcap_c + 4;
    sp += ((n_tables + n_derived) * 4 + 15) & ~15;
    double* own = reinterpret_cast<double*>(sp);  // z p s x r w of the owned column slice (x2), 1/dB of it, 1/dA of the owned row slice
    sp += 8 * (size_t)(6 * 2 * SC + 2 * SC + SR);
    double* bcast = reinterpret_cast<double*>(sp);  // 8 totals, my own 4 partials, then block_sum scratch
    double* scratch = bcast + 16;
    BlockCopy* s_copy = reinterpret_cast<BlockCopy*>(scratch + 8 * kB2Warps);  // the two copies' descriptors, read by block_phase
    double *oz = own, *op = own + 2 * SC, *os = own + 4 * SC, *ox = own + 6 * SC, *orr = own + 8 * SC, *ow = own + 10 * SC,
           *oib = own + 12 * SC, *odb = own + 13 * SC, *oia = own + 14 * SC;
    int* tb = s32;
    int* const chunk_r = tb;
    tb += 2 * Br.nch;
    int* const heavy_r = tb;
    tb += 3 * Br.nhv;
    int* const chunk_c = tb;
    tb += 2 * Bc.nch;
    int* const heavy_c = tb;
    tb += 3 * Bc.nhv;
    int *hfirst_r = tb, *hfirst_c = hfirst_r + Br.nhv + 1, *hseg_r = hfirst_c + Bc.nhv + 1, *hseg_c = hseg_r + segcap_r;
    const u16 *lov_r = s16 + L16.lov_r, *lov_c = s16 + L16.lov_c;
    Br.ell = smem_u32(s16 + L16.ell_r);
    Br.ref = 0;
    Br.lov = smem_u32(lov_r);
    Br.chunk = smem_u32(chunk_r);
    Br.heavy = smem_u32(heavy_r);
    Br.hfirst = smem_u32(hfirst_r);
    Br.hseg = smem_u32(hseg_r);
    Bc.ell = smem_u32(s16 + L16.ell_c);
    Bc.ref = smem_u32(s16 + L16.ref_c);
    Bc.lov = smem_u32(lov_c);
    Bc.chunk = smem_u32(chunk_c);
    Bc.heavy = smem_u32(heavy_c);
    Bc.hfirst = smem_u32(hfirst_c);
    Bc.hseg = smem_u32(hseg_c);

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
    // staging of the sums: the padding lines of the last owner's slice are shipped as zeros (never written again)
    for (int i = tid; i < 2 * Q * SR; i += kB2Threads) stg_r[i] = 0.0;
    for (int i = tid; i < 2 * P * SC; i += kB2Threads) stg_c[i] = 0.0;
    if (tid < 2) {  // segments of the heavy lines: thread 0 the rows', thread 1 the columns'
        const int nhv = tid == 0 ? Br.nhv : Bc.nhv;
        const int* hv = tid == 0 ? heavy_r : heavy_c;
        int* hf = tid == 0 ? hfirst_r : hfirst_c;
        int* hs = tid == 0 ? hseg_r : hseg_c;
        int n = 0;
        for (int hh = 0; hh < nhv; ++hh) {
            hf[hh] = n;
            const int cnt = (hv[3 * hh + 2] + kB2Seg - 1) / kB2Seg;
            for (int k = 0; k < cnt; ++k) hs[n++] = hh;
        }
        hf[nhv] = n;
    }
    __syncthreads();
    if (tid == 0) {
        Br.nseg = hfirst_r[Br.nhv];
        Bc.nseg = hfirst_c[Bc.nhv];
        s_copy[0] = Br;
        s_copy[1] = Bc;
    }

    if (cl && tid == 0) {
        for (int k = 0; k < 4; ++k) mbar_init(mbars + k, 1);
        fence_mbar_init();
    }

    // owned slices: local rows [r_lo, r_hi) of block row p, local columns [c_lo, c_hi) of block column q
    const int r_lo = min(q * SR, Rp), r_hi = min(r_lo + SR, Rp), c_lo = min(p * SC, Cq), c_hi = min(c_lo + SC, Cq);
    const int n_own_r = r_hi - r_lo, n_own_c = c_hi - c_lo;
    // through L2: block row p of X1 is [owner][source q][SR][2] doubles, X2 [R][2]; block column q of X3 is
    // [owner][source p][SC][2], X4 [C][2]
    u64* const x1_mine = A.x1 + (size_t)(p * Q) * Q * SR * 4;
    u64* const x1_own = x1_mine + (size_t)q * Q * SR * 4;  // what I sum as owner q
    u64* const x2_row = A.x2 + (size_t)p * A.R * 4;
    u64* const x3_mine = A.x3 + (size_t)(q * P) * P * SC * 4;
    u64* const x3_own = x3_mine + (size_t)p * P * SC * 4;
    u64* const x4_col = A.x4 + (size_t)q * A.C * 4;

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
    for (int c = tid; c < n_own_c; c += kB2Threads) {
        const double d = __ldg(A.dB + q + (c_lo + c) * Q);
        odb[c] = d;
        oib[c] = 1.0 / __ldg(A.mB + q + (c_lo + c) * Q);
    }
    __syncthreads();
    if (cl) cooperative_groups::this_cluster().sync();  // every inbox of the cluster is cleared before the first post

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
    // every thread keeps the CG scalars of ONE system, k = tid & 1 (the parity of the items it owns); flags are
    // exchanged inside the lane pair, so control flow is uniform and each division is compiled once
    const int myk = tid & 1;
    double gam = 0.0, gam0 = 0.0, gam_old = 1.0, al_old = 1.0;
    bool done_mine = false, done_other = false, broke = false;
    int it_mine = 0, it = 0;
    bool init = true;
    unsigned int round = A.round0;
#pragma unroll 1
    for (;; ++round) {
        if (!init) {
            // owners publish z of their column slice; everybody collects its block column's
            publish_slice(one, x4_col, 2 * c_lo, oz, 2 * n_own_c, reinterpret_cast<double*>(vecz), 2 * Cq, round);
            __syncthreads();
            B2_TICK(0)
            block_phase(smem_u32(&s_copy[0]), smem_u32(val), nval, smem_u32(vecz), 0u, smem_u32(stg_r), smem_u32(hpart), bcast + 12);
            ship_sums(cl, stg_r, Q, SR, q, Q, x1_mine, smem_u32(xbuf1), mb1, -1, round);
            B2_TICK(1)
            // owner: the Q partials of my rows, summed in block order; t = D1^-1 sum goes to the block row
            if (cl) {
                cluster_inbox_wait(mb1, 16u * (uint32_t)(Q * SR), ph1);
            } else {
                __syncthreads();  // the staged sums (in xbuf1) have left
                fw_gather(x1_own, xbuf1, Q * 2 * SR, round);
            }
            __syncthreads();
            for (int item = tid; item < 2 * n_own_r; item += kB2Threads) {
                double s = 0.0;
#pragma unroll 1
                for (int src = 0; src < Q; ++src) s += xbuf1[src * 2 * SR + item];
                const double tv = s * oia[item >> 1];
                if (cl) tloc[item] = tv;
                else fw_post(x2_row + ((size_t)r_lo * 2 + item) * 2, tv, round);
            }
            if (cl) {  // my t slice straight into the t vector of every CTA of the block row: one bulk copy each
                fence_proxy_async();
                __syncthreads();
                if (tid < Q && n_own_r > 0)
                    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                     map_rank(smem_u32(vect) + 16u * (uint32_t)r_lo, tid)),
                                 "r"(smem_u32(tloc)), "r"(16u * (uint32_t)n_own_r), "r"(map_rank(mb2, tid))
                                 : "memory");
            }
            B2_TICK(2)
            if (cl) cluster_inbox_wait(mb2, 16u * (uint32_t)Rp, ph2);
            else fw_gather(x2_row, reinterpret_cast<double*>(vect), 2 * Rp, round);
            __syncthreads();
            B2_TICK(3)
        }
        // column phase: partial B' t of my block; z . (B' t) rides along
        block_phase(smem_u32(&s_copy[1]), smem_u32(val), nval, smem_u32(vect), smem_u32(vecz), smem_u32(stg_c), smem_u32(hpart), part + 4);
        if (init) part[4] = part[5] = 0.0;
        ship_sums(one, stg_c, P, SC, p, P, x3_mine, smem_u32(xbuf3), mb3, one ? q : -1, round);
        B2_TICK(4)
        // everybody's partial dot products are known here (except in the set-up pass): their exchange overlaps the
        // exchange of the column partial sums
        if (!init) post_dots(part, scratch, bcast, A.x5 + (size_t)b * 16, one ? Q : 0, smem_u32(stage + 8 * b), mb5, round);
        // owner: u = sum of the P partials of my columns, then the new r/z (set-up) or w = D2 z - u
        if (one) {
            cluster_inbox_wait(mb3, 16u * (uint32_t)(P * SC), ph3);
        } else {
            __syncthreads();  // the staged sums (in xbuf3) have left
            fw_gather(x3_own, xbuf3, P * 2 * SC, round);
        }
        __syncthreads();
        for (int item = tid; item < 2 * n_own_c; item += kB2Threads) {
            const int c = item >> 1, k = item & 1;
            double u = 0.0;
            #pragma unroll 1
            for (int src = 0; src < P; ++src) u += xbuf3[src * 2 * SC + item];
            const double inv = oib[c], d = odb[c];
            if (init) {
                const double rb = k < nrhs ? __ldg((k ? A.rhs_b[1] : A.rhs_b[0]) + q + (c_lo + c) * Q) : 0.0;
                const double r = rb - u, z = r * inv;  // Schur right-hand side
                orr[item] = r;
                oz[item] = z;
                ox[item] = 0.0;
                op[item] = 0.0;
                os[item] = 0.0;
                const double g0 = rb * (rb * inv);  // the stopping rule's norm: the preconditioner's
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
        if (init) post_dots(part, scratch, bcast, A.x5 + (size_t)b * 16, one ? Q : 0, smem_u32(stage + 8 * b), mb5, round);
        if (one) cluster_inbox_wait(mb5, 64u * (uint32_t)G, ph5);
        else fw_gather(A.x5, stage, 8 * G, round);
        __syncthreads();
        if (warp < 8) {
            double s = 0.0;
#pragma unroll 1
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
            gam = myk ? tot[1] : tot[0];
            gam0 = myk ? tot[7] : tot[6];
            done_mine = (myk >= nrhs) || gam0 == 0.0 || !(gam > A.tol2 * gam0);
            if (A.fixed_iters > 0 && myk < nrhs) done_mine = false;
            done_other = __shfl_xor_sync(0xffffffffu, done_mine, 1);
            if (tid == 0) {
#pragma unroll
                for (int k = 0; k < 4; ++k) part[k] = bcast[8 + k];
            }
            init = false;
        } else {
            double al = 0.0, be = 0.0;
            bool brk = false;
            if (!done_mine) {
                gam = myk ? tot[1] : tot[0];
                if (it > 0 && !(gam > A.tol2 * gam0) && A.fixed_iters == 0) {
                    done_mine = true;
                } else {
                    const double delta = (myk ? tot[3] : tot[2]) - (myk ? tot[5] : tot[4]);  // z'D2 z - z'B'D1^-1 B z
                    // beta = gamma / gamma_old; p'Sp = delta - beta gamma / alpha_old, with the two quotients independent
                    const double g_over_a = gam / al_old;
                    be = (it == 0) ? 0.0 : gam / gam_old;
                    const double denom = delta - be * g_over_a;
                    if (!(denom > 0.0) && A.fixed_iters == 0) brk = true;     // not positive definite (or NaN)
                    al = gam / denom;
                    gam_old = gam;
                    al_old = al;
                    ++it_mine;
                }
            }
            ++it;
            done_other = __shfl_xor_sync(0xffffffffu, done_mine, 1);
            const bool brk_other = __shfl_xor_sync(0xffffffffu, brk, 1);  // every lane takes part: no short-circuit around a shuffle
            broke = brk || brk_other;
            if (!broke && !done_mine) {
                // p = z + beta p, s = w + beta s, x += alpha p, r -= alpha s, z = D2^-1 r on the owned slice (a finished
                // system is frozen; its partials are not used any more)
#pragma unroll 1
                for (int item = tid; item < 2 * n_own_c; item += kB2Threads) {
                    const double inv = oib[item >> 1], d = odb[item >> 1];
                    const double pn = oz[item] + be * op[item], sn = ow[item] + be * os[item];
                    const double xn = ox[item] + al * pn, rn = orr[item] - al * sn, zn = rn * inv;
                    op[item] = pn;
                    os[item] = sn;
                    ox[item] = xn;
                    orr[item] = rn;
                    oz[item] = zn;
                    if (myk) {
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
        bool all_done = done_mine && done_other;
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
        if (k < nrhs) (k ? A.sol_b[1] : A.sol_b[0])[q + (c_lo + (item >> 1)) * Q] = ox[item];
    }
    publish_slice(one, x4_col, 2 * c_lo, ox, 2 * n_own_c, reinterpret_cast<double*>(vecz), 2 * Cq, round);
    __syncthreads();
    block_phase(smem_u32(&s_copy[0]), smem_u32(val), nval, smem_u32(vecz), 0u, smem_u32(stg_r), smem_u32(hpart), bcast + 12);
    ship_sums(cl, stg_r, Q, SR, q, Q, x1_mine, smem_u32(xbuf1), mb1, -1, round);
    if (cl) {
        cluster_inbox_wait(mb1, 16u * (uint32_t)(Q * SR), ph1);
    } else {
        __syncthreads();
        fw_gather(x1_own, xbuf1, Q * 2 * SR, round);
    }
    __syncthreads();
    for (int item = tid; item < 2 * n_own_r; item += kB2Threads) {
        const int k = item & 1, gi = p + (r_lo + (item >> 1)) * P;
        double s = 0.0;
        #pragma unroll 1
                for (int src = 0; src < Q; ++src) s += xbuf1[src * 2 * SR + item];
        if (k < nrhs) (k ? A.sol_a[1] : A.sol_a[0])[gi] = (__ldg((k ? A.rhs_a[1] : A.rhs_a[0]) + gi) - s) / __ldg(A.dA + gi);
    }
    if (cl) cooperative_groups::this_cluster().sync();  // nobody leaves while its shared memory may still be written or read
    const int it_other = __shfl_xor_sync(0xffffffffu, it_mine, 1);
    if (b == 0 && tid == 0) {
        const int iters[2] = {it_mine, it_other};
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

// How many clusters of `size` CTAs (one per SM, full shared-memory budget) the device can hold at once; 0: none
static int max_clusters_of(int size)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)size);
    cfg.blockDim = dim3(kB2Threads);
    cfg.dynamicSmemBytes = kPcgSmemBudget;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)size;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (const void*)k_pcg_blocks, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        return 0;
    }
    return n;
}

static void set_kernel_attributes()
{
    static bool attr_set = false;
    if (attr_set) return;
    RG_CUDA(cudaFuncSetAttribute(k_pcg_blocks, cudaFuncAttributeMaxDynamicSharedMemorySize, kPcgSmemBudget));
    RG_CUDA(cudaFuncSetAttribute(k_pcg_blocks, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr_set = true;
}

// host-side estimate of the shared-memory plan of one block (entries spread evenly, 8 % padding); the exact need is
// only known once the plan is built
static long estimate_smem(long nnz, long nloc, long mfree, int P, int Q, int cluster)
{
    const long G = (long)P * Q, R = (nloc + P - 1) / P, C = (mfree + Q - 1) / Q, SR = (R + Q - 1) / Q, SC = (C + P - 1) / P;
    return (long)(1.08 * 14.0 * (double)nnz / (double)G) + 18 * (R + C) +
           8 * (b2_xbuf_doubles((int)SR, (int)SC, P, Q, cluster) + b2_staging_doubles((int)SR, (int)SC, P, Q, cluster)) +
           8 * (14 * SC + SR) + 64 * G + 6144;
}

// The block grid: coprime P x Q <= sm_count.  Through L2: among the grids that use at least 93 % of the SMs the one
// with the smallest plan (a tall pattern wants more block rows: slices of n / P rows and m / Q columns sit in every
// CTA).  With clusters a block row is one cluster of Q CTAs (its exchanges stay in distributed shared memory), so P
// is bounded by the number of clusters of that size the device holds at once (GPC by GPC); small patterns take ONE
// cluster (P = 1): every exchange is then inside it.  Clusters only where the estimate says the plan fits.
static void pick_grid(regot_ctx* ctx, long nnz, long nloc, long mfree, bool allow_cluster, int& P, int& Q, int& cluster)
{
    cluster = 0;
    if (ctx->pcg_blocks_cluster != 0 && !ctx->pcg_blocks_probed) {
        set_kernel_attributes();
        for (int q = 2; q <= 16; ++q) ctx->pcg_blocks_maxcl[q] = max_clusters_of(q);
        ctx->pcg_blocks_probed = true;
        if (std::getenv("REGOT_B200_PCG_BLOCKS_INFO")) {
            std::fprintf(stderr, "pcg blocks: clusters the device holds at once, by size 2..16:");
            for (int q = 2; q <= 16; ++q) std::fprintf(stderr, " %d", ctx->pcg_blocks_maxcl[q]);
            std::fprintf(stderr, "\n");
        }
    }
    allow_cluster = allow_cluster && ctx->pcg_blocks_cluster != 0;
    if (ctx->pcg_blocks_p > 0 && ctx->pcg_blocks_q > 0) {
        P = ctx->pcg_blocks_p;
        Q = ctx->pcg_blocks_q;
        cluster = allow_cluster && Q >= 2 && Q <= 16 && ctx->pcg_blocks_maxcl[Q] >= P;
        return;
    }
    const long budget = kPcgSmemBudget - kPcgSmemBudget / 16;  // the estimate must leave some room
    int most = 0;
    for (int q = 4; q <= 32; ++q)
        for (int p = 4; p <= 32; ++p)
            if (p * q <= ctx->sm_count && gcd_int(p, q) == 1) most = std::max(most, p * q);
    P = Q = 1;
    long best = -1;
    for (int q = 4; q <= 32; ++q)
        for (int p = 4; p <= 32; ++p) {
            if (p * q > ctx->sm_count || gcd_int(p, q) != 1 || p * q * 100 < most * 93) continue;
            const long est = estimate_smem(nnz, nloc, mfree, p, q, 0);
            if (best < 0 || est < best) {
                best = est;
                P = p;
                Q = q;
            }
        }
    if (best < 0) {  // a device with very few SMs
        P = 1;
        Q = std::max(1, std::min(ctx->sm_count, 16));
        return;
    }
    if (!allow_cluster) return;
    if (nnz <= ctx->pcg_blocks_one_cluster_entries && ctx->pcg_blocks_maxcl[16] >= 1 && estimate_smem(nnz, nloc, mfree, 1, 16, 1) <= budget) {
        P = 1;
        Q = 16;
        cluster = 1;
        return;
    }
    // larger patterns are bound by their mat-vec phases, not by the exchanges: there the grid with more CTAs wins
    if (nnz > ctx->pcg_blocks_cluster_entries) return;
    int cg = 0, cp = 0, cq = 0;
    long cest = 0;
    for (int q = 4; q <= 16; ++q) {
        int p = std::min(std::min(ctx->pcg_blocks_maxcl[q], ctx->sm_count / q), 32);
        while (p > 1 && gcd_int(p, q) != 1) --p;
        if (p < 2) continue;
        const long est = estimate_smem(nnz, nloc, mfree, p, q, 1);
        if (est > budget) continue;
        if (p * q > cg || (p * q == cg && est < cest)) {
            cg = p * q;
            cp = p;
            cq = q;
            cest = est;
        }
    }
    if (cg * 10 >= P * Q * 8) {  // a cluster grid that keeps at least 80 % as many SMs busy
        P = cp;
        Q = cq;
        cluster = 1;
    }
}

// Build the block plan of the current pattern; everything is enqueued on st, the summary lands in pinned memory
// (valid after the caller's next synchronisation with st).  csc2csr[t] = CSR position of CSC entry t.
void build_pcg_blocks_plan(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, regot_sparse& S, const int* csc2csr, bool allow_cluster)
{
    PcgBlocksPlan& Q2 = S.blocks;
    Q2.fits = false;
    Q2.pending = false;
    const int nloc = (int)S.nloc, mfree = std::max((int)S.m - 1, 0), nnz = (int)S.nnz;
    if (ctx->pcg_blocks == 0 || ctx->sharded || nnz < 1 || nloc < 64 || mfree < 64) return;
    // far too large for shared memory: do not even try (12 B per entry and copy at the very least)
    if ((long)nnz * 12 > (long)ctx->sm_count * kPcgSmemBudget) return;
    int P, Q, cluster;
    pick_grid(ctx, nnz, nloc, mfree, allow_cluster, P, Q, cluster);
    if (P * Q > ctx->sm_count || gcd_int(P, Q) != 1) raise(REGOT_E_VALIDATION, "pcg blocks: grid must be coprime and fit the device");
    Q2.cluster = cluster;
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
    k_b2_offsets<<<1, 32, 0, st>>>(P, Q, R, C, Q2.SR, Q2.SC, cluster, Q2.hdr.p, summary);
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
void finish_pcg_blocks_plan(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, regot_sparse& S, const int* csc2csr)
{
    PcgBlocksPlan& Q2 = S.blocks;
    static const bool show = std::getenv("REGOT_B200_PCG_BLOCKS_INFO") != nullptr;
    for (int attempt = 0; attempt < 2 && Q2.pending; ++attempt) {
        Q2.pending = false;
        Q2.smem = ws.h_blocks[0];
        Q2.fits = ws.h_blocks[1] == 0 && Q2.smem <= kPcgSmemBudget;
        if (show)
            std::fprintf(stderr, "pcg blocks: %d x %d blocks%s, slices %d x %d, L %d/%d, smem %d B, %s\n", Q2.P, Q2.Q,
                         Q2.cluster ? " (block row = cluster)" : "", Q2.R, Q2.C, Q2.Lr, Q2.Lc, Q2.smem, Q2.fits ? "fits" : "does not fit");
        if (Q2.fits || !Q2.cluster || csc2csr == nullptr) break;
        // the cluster grid (fewer, larger blocks) was too optimistic for this pattern: once more through L2
        build_pcg_blocks_plan(ctx, st, ws, S, csc2csr, false);
        RG_CUDA(cudaStreamSynchronize(st));
    }
}

static int pcg_blocks_launch(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, const regot_sparse& S, int nrhs,
                             const DVec* const* rhs, DVec* const* sol, double rtol, int max_iter)
{
    const PcgBlocksPlan& Q2 = S.blocks;
    const int nloc = (int)S.nloc, mfree = std::max((int)S.m - 1, 0), G = Q2.P * Q2.Q;
    set_kernel_attributes();
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
    A.mB = S.dS.p;
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
    A.cluster = Q2.cluster;
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
        if (Q2.cluster) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(G);
            cfg.blockDim = dim3(kB2Threads);
            cfg.dynamicSmemBytes = (size_t)Q2.smem;
            cfg.stream = st;
            cudaLaunchAttribute attr[2];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = (unsigned)Q2.Q;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            attr[1].id = cudaLaunchAttributeCooperative;  // all clusters resident at once, or the launch fails
            attr[1].val.cooperative = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 2;
            RG_CUDA(cudaLaunchKernelExC(&cfg, (const void*)k_pcg_blocks, args));
        } else {
            RG_CUDA(cudaLaunchCooperativeKernel((const void*)k_pcg_blocks, dim3(G), dim3(kB2Threads), args, (size_t)Q2.smem, st));
        }
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
