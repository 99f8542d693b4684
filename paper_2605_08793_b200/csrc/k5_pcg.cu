// k5_pcg.cu -- K5 on one GPU: the whole direction solve in ONE persistent kernel, on the Schur
// complement of the alpha block.
//
// Replaces numeric_factorize + solve (sparse_chol.h:330-427) inside compute_direction
// (splr.h:128-167).  A = [D1 B; B' D2] (D1, D2 diagonal, B = T_Omega / eta) is SPD, so
//     S x_b = r_b - B' D1^-1 r_a,   S = D2 - B' D1^-1 B,   x_a = D1^-1 (r_a - B x_b)
// and Jacobi-preconditioned CG on S takes half the iterations of block-Jacobi CG on A (the matrix
// is 2-cyclic) on vectors of length m-1 only.  Two right-hand sides (g and u of the Woodbury
// identity, splr.h:134-140; A^-1 v needs no solve, see solver.cu) are carried through every pass,
// interleaved 2 doubles per index so one gather serves both.
//
// Single-reduction CG (Chronopoulos-Gear): z = D2^-1 r, w = S z, gamma = r'z, delta = z'w;
//   beta = gamma / gamma_old, alpha = gamma / (delta - beta gamma / alpha_old),
//   p = z + beta p, s = w + beta s, x += alpha p, r -= alpha s.
// One iteration = row phase (t = D1^-1 B z) | barrier | column phase (w = D2 z - B' t, delta
// partials) | grid reduction of (gamma, delta) | vector update (gamma partials) | barrier.
//
// What bounds a scattered gather through L2 is the number of requests an SM can issue (one per entry,
// a fraction of a request per clock measured), not bytes, and a grid-wide barrier costs ~2400 clk
// (tools/barrier_bench.cu).  So this kernel runs only when the gathered vector (16 B x length) fits
// in shared memory: every CTA copies it there with coalesced loads at the start of a phase and
// gathers from shared memory, while the matrix streams from global memory, coalesced.  Larger
// problems take the kernel-by-kernel form of the same algorithm (k4_sparse.cu), where the two half
// mat-vecs run at 32 warps / SM.
// Work schedule (built on the host per pattern, sparse.hpp PcgSchedule): rows and columns of B are
// cut into warp-sized items -- 4 short lines (8 lanes each), one medium line, or one 256-entry
// chunk of a long line -- dealt to the grid's warps longest-first; the assignment is static over the
// CG iterations and each warp caches its item descriptors in shared memory.  Every sum has a fixed
// order (lane-sequential partials, butterfly, chunk order, CTA order): results are bitwise
// reproducible.  No float atomics.
#include "common.cuh"
#include "ctx.hpp"
#include "sparse.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

namespace rg {

constexpr int kSchurThreads = 512;
constexpr int kSchurWarps = kSchurThreads / 32;
static_assert(kSchurWarps == kPcgWarpsPerCta, "schedule and kernel disagree on warps per CTA");
constexpr int kMaxGrid = 160;     // CTAs whose partials are staged in shared memory by grid_sum4
constexpr int kLongStage = 256;   // long lines whose dot contributions are staged likewise
constexpr int kSchurScratchBytes = (4 * kSchurWarps + 8 + 4 * kMaxGrid + 2 * kLongStage) * 8;

enum { kRowMain = 0, kRowFinal = 1, kColInit = 2, kColMain = 3 };

struct SchurParams {
    int nloc, mfree, nrhs, max_iter, n_long, n_long_rows, nw, fixed_iters, cluster;  // long lines: rows first; only columns carry dots
    int vec_bytes, desc_cap;  // shared-memory carve-up: vector buffer, then desc_cap descriptors per warp
    int stage_rows, stage_cols;  // whether the vector a phase gathers is staged in shared memory (else: gathered through L2)
    double tol2;
    const int* col;  // CSR of B
    const double* val;
    const int* cscrow;  // CSC of B
    const double* cscval;
    const double* dA;
    const double* dB;
    const double* mB;  // Jacobi preconditioner: diag of the Schur complement (k4_sparse.cu compute_schur_diag)
    const int* items;  // kPcgItemInts per item
    const int* wptr;   // 2 x (nw + 1)
    double* chunk_part;  // n_chunks x 2
    unsigned int* chunk_cnt;
    const double* rhs_a[2];
    const double* rhs_b[2];
    double* sol_a[2];
    double* sol_b[2];
    double *ta, *zb, *wb, *pb, *sb, *rb, *xb;  // interleaved x2
    unsigned long long* xchg;                  // flagged words of the partial-sum exchange: (gridDim.x x 4 + n_long x 2) x 2
    unsigned int* barrier;
    double* out;  // iters[2], -, breakdown flag, then timing
    double* mbox;  // host mailbox for out[0..3]
    unsigned long long seq;
};

__device__ __forceinline__ double2 ldcg_x2(const double* p) { return __ldcg(reinterpret_cast<const double2*>(p)); }

// ~2400 clk among 148 CTAs on B200 (tools/barrier_bench.cu); cooperative_groups' grid.sync costs the same
__device__ __forceinline__ void grid_barrier(unsigned int* ctr, unsigned int& target)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        target += gridDim.x;
        __threadfence();
        atomicAdd(ctr, 1u);
        unsigned int v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

// A double travels as two 64-bit words, each carrying 32 bits of the value and the 32-bit sequence number
// of the exchange it belongs to: a reader that sees both numbers has the value, with no fence, atomic or
// barrier in between (an aligned 8-byte store is single-copy atomic).
__device__ __forceinline__ void xchg_post(unsigned long long* slot, double v, unsigned int seq)
{
    const unsigned long long b = (unsigned long long)__double_as_longlong(v), f = (unsigned long long)seq << 32;
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(slot), "l"((b & 0xffffffffull) | f), "l"((b >> 32) | f) : "memory");
}
__device__ __forceinline__ double xchg_wait(const unsigned long long* slot, unsigned int seq)
{
    unsigned long long lo, hi;
    do {
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(slot) : "memory");
    } while ((unsigned int)(lo >> 32) != seq || (unsigned int)(hi >> 32) != seq);
    return __longlong_as_double((long long)((lo & 0xffffffffull) | (hi << 32)));
}

// Small systems run on ONE thread-block cluster (16 CTAs) instead of the whole GPU: the work per
// iteration is a few entries per lane either way, and the hardware cluster barrier costs a fraction of a
// barrier through L2 among 148 CTAs.
__device__ __forceinline__ void sync_all(const SchurParams& P, unsigned int& target)
{
    if (P.cluster) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
        grid_barrier(P.barrier, target);
    }
}

#ifdef REGOT_PCG_TIMING
__device__ long long g_tsub[8];
#define RG_SUB(i)                                                     \
    if (blockIdx.x == 3 && threadIdx.x == 37) {                       \
        const long long now__ = clock64();                            \
        g_tsub[i] += now__ - tsub_prev;                               \
        tsub_prev = now__;                                            \
    }
#else
#define RG_SUB(i)
#endif
// sum of 4 per-thread values over the grid, in CTA order (+ the long lines' dot contributions added
// to components [2 long_range, 2 long_range + 2)); result in every thread.  Every CTA posts its 4
// partials as flagged words and reads everybody's: one store-to-poll latency instead of a grid barrier
// followed by a round of loads.  It is also a barrier for memory: the partials are posted behind a
// fence that follows the CTA's own writes, and every reader fences after it has seen them.
// Written for instruction count: with 16 warps on 4 schedulers every instruction on this path costs
// ~4 clk per iteration of the solve (transposing warp reduction: 6 shuffles for 4 values, not 20).
__device__ __noinline__ void grid_sum4(const SchurParams& P, double (&v)[4], double* scratch, double* bcast, unsigned int seq,
                                       int long_range)
{
    double* stage = bcast + 8;
    double* stage_long = stage + 4 * kMaxGrid;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#ifdef REGOT_PCG_TIMING
    long long tsub_prev = clock64();
#endif
    {
        // lanes with (bit 4, bit 3) = (h, b) end up with the warp's sum of v[2h + b]
        const bool up = lane & 16, b3 = lane & 8;
        const double c0 = (up ? v[2] : v[0]) + shfl_xor_d(up ? v[0] : v[2], 16);
        const double c1 = (up ? v[3] : v[1]) + shfl_xor_d(up ? v[1] : v[3], 16);
        double d = (b3 ? c1 : c0) + shfl_xor_d(b3 ? c0 : c1, 8);
        d += shfl_xor_d(d, 4);
        d += shfl_xor_d(d, 2);
        d += shfl_xor_d(d, 1);
        if ((lane & 7) == 0) scratch[(lane >> 3) * kSchurWarps + warp] = d;
    }
    __syncthreads();
    RG_SUB(0)
    if (threadIdx.x < 4 * kSchurWarps) {  // 16 lanes per component
        double d = scratch[threadIdx.x];
        d += shfl_xor_d(d, 8);
        d += shfl_xor_d(d, 4);
        d += shfl_xor_d(d, 2);
        d += shfl_xor_d(d, 1);
        if ((threadIdx.x & (kSchurWarps - 1)) == 0) {
            __threadfence();
            xchg_post(P.xchg + ((size_t)blockIdx.x * 4 + (threadIdx.x / kSchurWarps)) * 2, d, seq);
        }
    }
    const int nvals = (int)gridDim.x * 4, n_dots = P.n_long - P.n_long_rows;  // the column phase's long lines
    const int nlong = long_range >= 0 ? min(n_dots, kLongStage) * 2 : 0;
#pragma unroll 1
    for (int i = threadIdx.x; i < nvals + nlong; i += kSchurThreads) {
        const double x = xchg_wait(P.xchg + (size_t)i * 2, seq);
        if (i < nvals) stage[i] = x;
        else stage_long[i - nvals] = x;
    }
    RG_SUB(1)
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    RG_SUB(2)
    __syncthreads();
    RG_SUB(3)
    if (warp < 4) {
        const int k = warp;
        double s = 0.0;
#pragma unroll 1
        for (int b = lane; b < (int)gridDim.x; b += 32) s += stage[b * 4 + k];
        if (k / 2 == long_range) {
#pragma unroll 1
            for (int q = lane; q < n_dots; q += 32)
                s += q < kLongStage ? stage_long[q * 2 + (k % 2)] : xchg_wait(P.xchg + ((size_t)nvals + (size_t)q * 2 + (k % 2)) * 2, seq);
        }
        s = warp_sum(s);
        if (lane == 0) bcast[k] = s;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = bcast[k];
    RG_SUB(4)
}

// shared-memory carve-up as 32-bit shared-window addresses
struct WarpLog {
    uint32_t vec;   // the shared copy of the gathered vector (x2)
    uint32_t desc;  // this warp's cached item descriptors (kPcgItemInts ints each)
};
__device__ __forceinline__ int lds_i32(uint32_t addr)
{
    int v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ double lds_f64v(uint32_t addr)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts_i32(uint32_t addr, int v) { asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory"); }
__device__ __forceinline__ void sts_f64(uint32_t addr, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory"); }
__device__ __forceinline__ void sts_f64x2(uint32_t addr, double2 v)
{
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(v.x), "d"(v.y) : "memory");
}

// Transposing reduction of (a0, a1) over groups of 8 lanes (full == false) or the warp: on return
// even lanes hold the group sum of a0, odd lanes that of a1.  3 / 5 shuffles; fixed order.
__device__ __forceinline__ double reduce2(double a0, double a1, int lane, bool full)
{
    const bool odd = lane & 1;
    double c = (odd ? a1 : a0) + shfl_xor_d(odd ? a0 : a1, 1);
    c += shfl_xor_d(c, 2);
    c += shfl_xor_d(c, 4);
    if (full) {
        c += shfl_xor_d(c, 8);
        c += shfl_xor_d(c, 16);
    }
    return c;
}

// gathered x2 entry at byte offset `off` of the shared copy of the vector
__device__ __forceinline__ double2 gather2(uint32_t vec, unsigned off)
{
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(vec + off));
    return v;
}

// Head of one item as every lane needs it, and the first 8 (index, value) pairs of the lane
struct ItemHead {
    int kind, nE, chunk, slot, first, cnt, line, beg, len;
    double diag;
};

// descriptor from the warp's shared-memory cache (slot >= 0) or from global memory
__device__ __forceinline__ ItemHead load_head(const SchurParams& P, const double* __restrict__ diagv, uint32_t cached,
                                              bool is_cached, int q, int lane)
{
    ItemHead h;
    if (is_cached) {
        h.kind = lds_i32(cached);
        h.nE = lds_i32(cached + 4);
        h.chunk = lds_i32(cached + 8);
        h.slot = lds_i32(cached + 12);
        h.first = lds_i32(cached + 16);
        h.cnt = lds_i32(cached + 20);
        const uint32_t sub = h.kind == 0 ? (uint32_t)(lane >> 3) : 0u;
        h.line = lds_i32(cached + 32 + 4 * sub);
        h.beg = lds_i32(cached + 48 + 4 * sub);
        h.len = lds_i32(cached + 64 + 4 * sub);
    } else {
        const int* d = P.items + (size_t)q * kPcgItemInts;
        const int4 m0 = __ldg(reinterpret_cast<const int4*>(d));
        h.kind = m0.x;
        h.nE = m0.y;
        h.chunk = m0.z;
        h.slot = m0.w;
        h.first = __ldg(d + 4);
        h.cnt = __ldg(d + 5);
        const int sub = h.kind == 0 ? lane >> 3 : 0;
        h.line = __ldg(d + 8 + sub);
        h.beg = __ldg(d + 12 + sub);
        h.len = __ldg(d + 16 + sub);
    }
    h.diag = h.line >= 0 ? __ldg(diagv + h.line) : 1.0;
    return h;
}
// One mat-vec phase over this warp's items.  kRows: lines are rows of B and the staged vector is a
// beta-space vector (x2); else lines are columns of B and it is the alpha-space vector ta (x2).  `dot`
// accumulates this lane's component (lane & 1) of gamma (kColInit) or delta (kColMain) over the lines
// this warp finished.  The matrix streams from global memory, coalesced, 8 entries per lane in
// flight; descriptors of the first n_desc items are cached in shared memory at `desc`.
template <bool kRows>
__device__ __forceinline__ void run_phase(const SchurParams& P, int mode, const WarpLog& L, int i0, int i1,
                                          uint32_t desc, int n_desc, int lane, double& dot, unsigned int seq, const double* gx,
                                          bool staged)
{
    const int* __restrict__ src_idx = kRows ? P.col : P.cscrow;
    const double* __restrict__ src_val = kRows ? P.val : P.cscval;
    const double* __restrict__ diagv = kRows ? P.dA : P.dB;
    const int kk = lane & 1;
    for (int q = i0; q < i1; ++q) {
        double a0 = 0.0, a1 = 0.0;
        const int qs = q - i0;
        const ItemHead h = load_head(P, diagv, desc + (uint32_t)qs * (kPcgItemInts * 4), qs < n_desc, q, lane);
        const int kind = h.kind, nE = h.nE, chunk = h.chunk, slot = h.slot, first = h.first, cnt = h.cnt, line = h.line;
        const double diag = h.diag;
        const int gl = kind == 0 ? lane & 7 : lane, stride = kind == 0 ? 8 : 32;
        for (int e0 = 0; e0 < nE; e0 += 8) {
            int c[8];
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int t = gl + stride * (e0 + u);
                const bool ok = (e0 + u) < nE && t < h.len;
                c[u] = ok ? __ldg(src_idx + h.beg + t) : 0;
                v[u] = ok ? __ldg(src_val + h.beg + t) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double2 g = staged ? gather2(L.vec, (unsigned)c[u] * 16u) : ldcg_x2(gx + (size_t)c[u] * 2);
                a0 += v[u] * g.x;
                a1 += v[u] * g.y;
            }
        }
        double sum = reduce2(a0, a1, lane, kind != 0);
        // lanes 0 and 1 of a group finish components 0 and 1 of the group's line
        bool finish = line >= 0 && (lane & (kind == 0 ? 6 : 30)) == 0;
        bool is_long = false;
        if (kind == 2) {
            // chunk of a long line: publish the partial; the last chunk to arrive sums them in chunk order
            if (finish) P.chunk_part[(size_t)chunk * 2 + kk] = sum;
            __syncwarp();  // lanes 0 and 1 wrote the partial: ordered before lane 0's release
            unsigned int prev = 0;
            if (lane == 0)  // one acquire-release atomic instead of two sequentially-consistent fences per warp
                asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(P.chunk_cnt + slot) : "memory");
            prev = __shfl_sync(0xffffffffu, prev, 0);
            if ((int)prev == cnt - 1) {
                double s0_ = 0.0, s1_ = 0.0;
                for (int c = lane; c < cnt; c += 32) {
                    s0_ += __ldcg(P.chunk_part + (size_t)(first + c) * 2);
                    s1_ += __ldcg(P.chunk_part + (size_t)(first + c) * 2 + 1);
                }
                s0_ = warp_sum(s0_);
                s1_ = warp_sum(s1_);
                sum = kk ? s1_ : s0_;
                if (lane == 0) P.chunk_cnt[slot] = 0u;
                is_long = true;
            } else {
                finish = false;
            }
        }
        if (finish) {
            const size_t o = (size_t)line * 2 + kk;
            if (kRows) {
                if (mode == kRowMain) {
                    P.ta[o] = sum / diag;
                } else if (kk < P.nrhs) {
                    const double* ra = kk ? P.rhs_a[1] : P.rhs_a[0];
                    double* xa = kk ? P.sol_a[1] : P.sol_a[0];
                    xa[line] = (ra[line] - sum) / diag;
                }
            } else {
                double dk;
                if (mode == kColInit) {
                    const double* rb = kk ? P.rhs_b[1] : P.rhs_b[0];
                    const double c = (kk < P.nrhs ? rb[line] : 0.0) - sum;  // Schur right-hand side
                    const double z = c / __ldg(P.mB + line);
                    P.rb[o] = c;
                    P.zb[o] = z;
                    P.xb[o] = 0.0;
                    P.pb[o] = 0.0;
                    P.sb[o] = 0.0;
                    dk = c * z;
                } else {
                    const double z = __ldcg(P.zb + o);
                    const double w = diag * z - sum;
                    P.wb[o] = w;
                    dk = z * w;
                }
                // which warp finishes a long line varies from run to run: its dot product goes to a fixed
                // slot of the ordered grid reduction (sequence number `seq`) instead of this lane's partial
                if (is_long) xchg_post(P.xchg + ((size_t)gridDim.x * 4 + (size_t)(slot - P.n_long_rows) * 2 + kk) * 2, dk, seq);
                else dot += dk;
            }
        }
    }
}

// all threads of the CTA: shared copy of an x2 vector of `count` entries (after a grid barrier)
__device__ __forceinline__ void stage_vector(uint32_t vec, const double* gx, int count)
{
    for (int i = threadIdx.x; i < count; i += kSchurThreads * 10) {
        double2 v[10];
#pragma unroll
        for (int u = 0; u < 10; ++u) {
            const int j = i + u * kSchurThreads;
            v[u] = j < count ? ldcg_x2(gx + (size_t)j * 2) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < 10; ++u) {
            const int j = i + u * kSchurThreads;
            if (j < count) sts_f64x2(vec + 16u * (uint32_t)j, v[u]);
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kSchurThreads, 1) k_pcg_schur(const __grid_constant__ SchurParams P)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    WarpLog L;
    L.vec = smem_u32(smem);
    const uint32_t desc_bytes = (uint32_t)P.desc_cap * (kPcgItemInts * 4);
    L.desc = L.vec + (uint32_t)P.vec_bytes + (uint32_t)warp * desc_bytes;
    double* scratch = reinterpret_cast<double*>(smem + P.vec_bytes + (size_t)kSchurWarps * desc_bytes);
    double* bcast = scratch + 4 * kSchurWarps;

    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nthr = gridDim.x * blockDim.x;
    // the schedule deals items CTA-first so the heaviest ones land on different SMs
    const int gw = warp * gridDim.x + blockIdx.x;
    const int nloc = P.nloc, mfree = P.mfree, nrhs = P.nrhs;
    unsigned int bar_target = 0, xchg_seq = 0;
#ifdef REGOT_PCG_TIMING  // per-section cycle counts per CTA (experiments only; costs registers)
    long long tsec[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tprev = clock64();
#define RG_TICK(i)                         \
    {                                      \
        const long long now__ = clock64(); \
        tsec[i] += now__ - tprev;          \
        tprev = now__;                     \
    }
#else
#define RG_TICK(i)
#endif

    const int r0 = P.wptr[gw], r1 = P.wptr[gw + 1];
    const int c0 = P.wptr[P.nw + 1 + gw], c1 = P.wptr[P.nw + 1 + gw + 1];
    // this warp's item descriptors, rows first
    const int nd_r = min(r1 - r0, P.desc_cap), nd_c = min(c1 - c0, P.desc_cap - nd_r);
    for (int q = 0; q < nd_r + nd_c; ++q) {
        const int item = q < nd_r ? r0 + q : c0 + (q - nd_r);
        if (lane < kPcgItemInts) sts_i32(L.desc + (uint32_t)q * (kPcgItemInts * 4) + 4u * lane, __ldg(P.items + (size_t)item * kPcgItemInts + lane));
    }
    const uint32_t desc_r = L.desc, desc_c = L.desc + (uint32_t)nd_r * (kPcgItemInts * 4);
    __syncwarp();

    // ---- t = D1^-1 r_a; gamma0 = r' D^-1 r of the FULL system (the meaning of rtol is unchanged) ----
    double red[4] = {0.0, 0.0, 0.0, 0.0};  // [0..1] gamma partials, [2..3] second quantity
    for (int i = tid; i < nloc; i += nthr) {
        const double d = P.dA[i];
        double t[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const double r = (k < nrhs) ? P.rhs_a[k][i] : 0.0;
            t[k] = r / d;
            red[2 + k] += r * t[k];
        }
        *reinterpret_cast<double2*>(P.ta + (size_t)i * 2) = make_double2(t[0], t[1]);
    }
    for (int j = tid; j < mfree; j += nthr) {
        const double d = P.mB[j];  // the stopping rule's norm: the preconditioner's
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const double r = (k < nrhs) ? P.rhs_b[k][j] : 0.0;
            red[2 + k] += r * (r / d);
        }
    }

    double gamma[2] = {0.0, 0.0}, gamma0[2] = {0.0, 0.0};
    double gamma_old[2] = {1.0, 1.0}, alpha_old[2] = {1.0, 1.0};
    bool done[2] = {false, false};
    int iters[2] = {0, 0};
    bool broke = false;
    // One loop body serves the set-up pass (no row phase, column phase forms the Schur right-hand side),
    // the CG iterations, and the final back-substitution, so each phase is instantiated once.
    int row_mode = -1, col_mode = kColInit, it = 0;
    for (;;) {
        if (row_mode >= 0) {
            // kRowMain: t = D1^-1 B z;  kRowFinal: x_a = D1^-1 (r_a - B x_b)
            double none = 0.0;
            const double* gx = row_mode == kRowMain ? P.zb : P.xb;
            if (P.stage_rows) stage_vector(L.vec, gx, mfree);
            run_phase<true>(P, row_mode, L, r0, r1, desc_r, nd_r, lane, none, 0u, gx, P.stage_rows != 0);
            if (row_mode == kRowFinal) break;
        }
        RG_TICK(1)
        sync_all(P, bar_target);
        RG_TICK(2)
        // kColInit: c = r_b - B' t, r = c, z = D2^-1 c, x = p = s = 0, gamma = r'z
        // kColMain: w = D2 z - B' t, delta = z'w
        {
            double dot = 0.0;
            if (P.stage_cols) stage_vector(L.vec, P.ta, nloc);
            ++xchg_seq;
            run_phase<false>(P, col_mode, L, c0, c1, desc_c, nd_c, lane, dot, xchg_seq, P.ta, P.stage_cols != 0);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const double dk = ((lane & 1) == k) ? dot : 0.0;
                if (col_mode == kColInit) red[k] = dk;
                else red[2 + k] = dk;  // red[k] still holds the gamma partial of the last update
            }
        }
        RG_TICK(3)
        grid_sum4(P, red, scratch, bcast, xchg_seq, col_mode == kColInit ? 0 : 1);
        RG_TICK(4)
        if (col_mode == kColInit) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                gamma[k] = red[k];
                gamma0[k] = red[2 + k];
                done[k] = (k >= nrhs) || gamma0[k] == 0.0 || !(gamma[k] > P.tol2 * gamma0[k]);
                if (P.fixed_iters > 0 && k < nrhs) done[k] = false;
                red[k] = 0.0;  // no update yet: no gamma partial for the first combined reduction
            }
            col_mode = kColMain;
        } else {
            double al[2], be[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                al[k] = be[k] = 0.0;
                if (done[k]) continue;
                if (it > 0) {  // gamma = r'z of the last update arrives with this reduction
                    gamma[k] = red[k];
                    if (!(gamma[k] > P.tol2 * gamma0[k]) && P.fixed_iters == 0) {
                        done[k] = true;
                        continue;
                    }
                }
                const double delta = red[2 + k];
                be[k] = (it == 0) ? 0.0 : gamma[k] / gamma_old[k];
                const double denom = delta - be[k] * gamma[k] / alpha_old[k];  // = p'Sp
                if (!(denom > 0.0) && P.fixed_iters == 0) broke = true;        // not positive definite (or NaN)
                al[k] = gamma[k] / denom;
                gamma_old[k] = gamma[k];
                alpha_old[k] = al[k];
                ++iters[k];
            }
            ++it;
            if (!broke && !(done[0] && done[1])) {
                // p = z + beta p, s = w + beta s, x += alpha p, r -= alpha s, z = D2^-1 r, gamma = r'z
#pragma unroll
                for (int k = 0; k < 4; ++k) red[k] = 0.0;
                // groups of 32 entries dealt CTA-first: on the critical path between two grid-wide waits it matters
                // that no SM has more than a warp or two of this to issue
                for (int j = (warp * (int)gridDim.x + (int)blockIdx.x) * 32 + lane; j < mfree; j += nthr) {
                    const size_t o = (size_t)j * 2;
                    const double2 z2 = ldcg_x2(P.zb + o), p2 = ldcg_x2(P.pb + o), w2 = ldcg_x2(P.wb + o);
                    const double2 s2 = ldcg_x2(P.sb + o), x2 = ldcg_x2(P.xb + o), r2 = ldcg_x2(P.rb + o);
                    const double dj = __ldg(P.mB + j);
                    const double zv[2] = {z2.x, z2.y}, pv[2] = {p2.x, p2.y}, wv[2] = {w2.x, w2.y};
                    const double sv[2] = {s2.x, s2.y}, xv[2] = {x2.x, x2.y}, rv[2] = {r2.x, r2.y};
                    double pn[2], sn[2], xn[2], rn[2], zn[2];
#pragma unroll
                    for (int k = 0; k < 2; ++k) {
                        pn[k] = zv[k] + be[k] * pv[k];
                        sn[k] = wv[k] + be[k] * sv[k];
                        xn[k] = xv[k] + al[k] * pn[k];
                        rn[k] = rv[k] - al[k] * sn[k];
                        zn[k] = rn[k] / dj;
                        if (done[k]) {  // a finished system is frozen
                            pn[k] = pv[k];
                            sn[k] = sv[k];
                            xn[k] = xv[k];
                            rn[k] = rv[k];
                            zn[k] = zv[k];
                        } else {
                            red[k] += rn[k] * zn[k];
                        }
                    }
                    *reinterpret_cast<double2*>(P.pb + o) = make_double2(pn[0], pn[1]);
                    *reinterpret_cast<double2*>(P.sb + o) = make_double2(sn[0], sn[1]);
                    *reinterpret_cast<double2*>(P.xb + o) = make_double2(xn[0], xn[1]);
                    *reinterpret_cast<double2*>(P.rb + o) = make_double2(rn[0], rn[1]);
                    *reinterpret_cast<double2*>(P.zb + o) = make_double2(zn[0], zn[1]);
                }
                // z is needed by the next row phase; the gamma partials ride on the next reduction
                // (one grid reduction per iteration: Chronopoulos-Gear)
                RG_TICK(5)
                sync_all(P, bar_target);
                RG_TICK(6)
            }
        }
        bool all_done = done[0] && done[1];
        if (P.fixed_iters > 0) all_done = it >= P.fixed_iters;
        row_mode = (all_done || broke || it >= P.max_iter) ? kRowFinal : kRowMain;
    }
    // planar outputs
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        if (k >= nrhs) break;
        for (int j = tid; j < mfree; j += nthr) P.sol_b[k][j] = __ldcg(P.xb + (size_t)j * 2 + k);
        if (tid == 0) P.sol_b[k][mfree] = 0.0;
    }
    RG_TICK(7)
    if (tid == 0) {
#pragma unroll
        for (int k = 0; k < 2; ++k) P.out[k] = (double)iters[k];
        P.out[3] = broke ? 1.0 : 0.0;
        // the host only needs these flags; everything it launches next is ordered behind this kernel
        if (P.mbox) {
            const double post[4] = {(double)iters[0], (double)iters[1], 0.0, broke ? 1.0 : 0.0};
            mailbox_post(P.mbox, post, 4, P.seq);
        }
    }
#ifdef REGOT_PCG_TIMING
    if (threadIdx.x == 0)
        for (int k = 0; k < 8; ++k) P.out[4 + (size_t)blockIdx.x * 8 + k] = (double)tsec[k];
#endif
#undef RG_TICK
}

// ---- host: the work schedule ------------------------------------------------------------------
// Items of one phase are produced in order of decreasing row count nE (a counting sort: nE <= 16), then
// dealt over the warps in a snake (position q of the sorted order -> round q / nw, warp q % nw, reversed
// on odd rounds) so the loads stay level; warp w's items are contiguous in `items`.  Everything is
// written straight into pinned staging and uploaded asynchronously: no allocation, no sort call.
// largest cluster (<= the requested size) of CTAs with the kernel's full shared-memory budget that this device can host
static int probe_cluster_size(int want)
{
    RG_CUDA(cudaFuncSetAttribute(k_pcg_schur, cudaFuncAttributeMaxDynamicSharedMemorySize, kPcgSmemBudget));
    RG_CUDA(cudaFuncSetAttribute(k_pcg_schur, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (int size = want; size >= 2; size /= 2) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(size);
        cfg.blockDim = dim3(kSchurThreads);
        cfg.dynamicSmemBytes = kPcgSmemBudget;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)size;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, (const void*)k_pcg_schur, &cfg) == cudaSuccess && n >= 1) return size;
        (void)cudaGetLastError();
    }
    return 0;
}

void build_pcg_schedule(regot_ctx* ctx, cudaStream_t st, regot_sparse& S, const int* rp, const int* cp, PinnedBuf<int>& staging,
                        size_t staging_used)
{
    if (ctx->pcg_cluster_size > 0 && !ctx->pcg_cluster_probed) {
        ctx->pcg_cluster_size = probe_cluster_size(std::min(ctx->pcg_cluster_size, 16));
        ctx->pcg_cluster_probed = true;
    }
    PcgSchedule& Q = S.pcg;
    const int nloc = (int)S.nloc, mm1 = std::max((int)S.m - 1, 0);
    // small systems: one cluster of CTAs (hardware barrier) instead of the whole GPU
    const long entries_per_iter = 2L * (long)rp[nloc];
    int grid = ctx->sm_count;
    if (ctx->pcg_cluster_size > 0 && entries_per_iter <= ctx->pcg_cluster_max_entries) grid = ctx->pcg_cluster_size;
    const int nw = grid * kPcgWarpsPerCta;
    Q.grid = grid;
    Q.nw = nw;
    // shared-memory plan: the larger of the two gathered vectors (16 B per entry), then the descriptor
    // cache.  fits == false: sparse_pcg takes the kernel-by-kernel path and this schedule is not used.
    const int budget = kPcgSmemBudget - kSchurScratchBytes;
    // a phase whose gathered vector does not fit gathers it through L2 instead (request-rate bound, ~14 k clk per
    // phase at 10^6 entries -- still one kernel per solve, against ~95 us per iteration kernel by kernel)
    const long need_r = 16L * std::max(mm1, 1), need_c = 16L * std::max(nloc, 1);
    Q.stage_rows = need_r <= kPcgVecSmemMax;
    Q.stage_cols = need_c <= kPcgVecSmemMax;
    Q.fits = (Q.stage_rows || Q.stage_cols) && rp[nloc] <= kPcgMaxEntriesL2Gather;
    if (Q.stage_rows && Q.stage_cols) Q.fits = true;
    const long need = std::max<long>(Q.stage_rows ? need_r : 0, Q.stage_cols ? need_c : 0);
    Q.vec_bytes = (int)((std::max<long>(need, 16) + 127) / 128 * 128);
    Q.desc_cap = std::min(40, (budget - Q.vec_bytes) / (kPcgWarpsPerCta * kPcgItemInts * 4));
    if (!Q.fits) return;

    constexpr int kMaxNE = 16;
    int* const h_items = staging.p + staging_used;  // room was reserved by the caller
    int n_items_total = 0, n_long = 0, n_chunks = 0;
    // per phase: count items by nE, then place
    int* h_wptr = nullptr;
    static thread_local std::vector<int> bucket_cnt, bucket_pos, short_sorted;
    for (int pass = 0; pass < 2; ++pass) {  // pass 0 sizes the item array (the pointer tables go behind it)
        int n_long_p = 0, n_chunks_p = 0, cursor_items = 0;
        for (int phase = 0; phase < 2; ++phase) {
            const int* ptr = phase == 0 ? rp : cp;
            const int nlines = phase == 0 ? nloc : mm1;
            // short lines sorted by decreasing length (counting sort) so a quad holds lines of similar length
            bucket_cnt.assign((size_t)kShortLine + 2, 0);
            int n_short = 0;
            for (int l = 0; l < nlines; ++l) {
                const int len = ptr[l + 1] - ptr[l];
                if (len <= kShortLine) {
                    ++bucket_cnt[(size_t)(kShortLine - len)];
                    ++n_short;
                }
            }
            bucket_pos.assign((size_t)kShortLine + 2, 0);
            for (int k = 1; k <= kShortLine + 1; ++k) bucket_pos[(size_t)k] = bucket_pos[(size_t)k - 1] + bucket_cnt[(size_t)k - 1];
            short_sorted.resize((size_t)n_short + 4);
            for (int l = 0; l < nlines; ++l) {
                const int len = ptr[l + 1] - ptr[l];
                if (len <= kShortLine) short_sorted[(size_t)bucket_pos[(size_t)(kShortLine - len)]++] = l;
            }
            // items by nE: count[nE]
            int cnt_ne[kMaxNE + 1] = {0};
            for (int l = 0; l < nlines; ++l) {
                const int len = ptr[l + 1] - ptr[l];
                if (len > kLongLine) {
                    const int full = len / kChunkLen, rest = len - full * kChunkLen;
                    cnt_ne[kChunkLen / 32] += full;
                    if (rest) ++cnt_ne[(rest + 31) / 32];
                } else if (len > kShortLine) {
                    ++cnt_ne[(len + 31) / 32];
                }
            }
            for (int q = 0; q < n_short; q += 4) {
                const int l0 = short_sorted[(size_t)q];
                ++cnt_ne[(ptr[l0 + 1] - ptr[l0] + 7) / 8];  // the quad's longest line comes first
            }
            int n_items = 0;
            for (int e = 0; e <= kMaxNE; ++e) n_items += cnt_ne[e];
            if (pass == 0) {
                cursor_items += n_items;
                continue;
            }
            // sorted position of the first item of each nE class (decreasing nE)
            int start_ne[kMaxNE + 1];
            {
                int acc = 0;
                for (int e = kMaxNE; e >= 0; --e) {
                    start_ne[e] = acc;
                    acc += cnt_ne[e];
                }
            }
            // warp w holds the items at sorted positions q with (q / nw even ? q % nw : nw - 1 - q % nw) == w,
            // in round order: its count is the number of rounds that reach it
            const int full_rounds = n_items / nw, tail = n_items % nw;
            const int base = cursor_items;
            int* wp = h_wptr + (size_t)phase * (nw + 1);
            {
                int acc = base;
                for (int w = 0; w < nw; ++w) {
                    wp[w] = acc;
                    const bool in_tail = (full_rounds & 1) ? (nw - 1 - w) < tail : w < tail;
                    acc += full_rounds + (in_tail ? 1 : 0);
                }
                wp[nw] = acc;
            }
            auto place = [&](int q) -> int* {  // slot of the item at sorted position q
                const int round = q / nw, pos = q % nw;
                const int w = (round & 1) ? nw - 1 - pos : pos;
                return h_items + (size_t)kPcgItemInts * (size_t)(wp[w] + round);
            };
            auto emit = [&](int nE, int kind, int chunk, int slot, int first, int cnt, const int (&line)[4], const int (&beg)[4],
                            const int (&len)[4]) {
                int* r = place(start_ne[nE]++);
                r[0] = kind; r[1] = nE; r[2] = chunk; r[3] = slot; r[4] = first; r[5] = cnt; r[6] = 0; r[7] = 0;
                for (int k = 0; k < 4; ++k) {
                    r[8 + k] = line[k];
                    r[12 + k] = beg[k];
                    r[16 + k] = len[k];
                    r[20 + k] = 0;
                }
            };
            for (int l = 0; l < nlines; ++l) {
                const int beg = ptr[l], len = ptr[l + 1] - beg;
                if (len > kLongLine) {
                    const int slot = n_long + n_long_p++, first = n_chunks + n_chunks_p;
                    const int cnt = (len + kChunkLen - 1) / kChunkLen;
                    for (int c = 0; c < cnt; ++c) {
                        const int clen = std::min(kChunkLen, len - c * kChunkLen);
                        const int line4[4] = {l, -1, -1, -1}, beg4[4] = {beg + c * kChunkLen, 0, 0, 0}, len4[4] = {clen, 0, 0, 0};
                        emit((clen + 31) / 32, 2, n_chunks + n_chunks_p++, slot, first, cnt, line4, beg4, len4);
                    }
                } else if (len > kShortLine) {
                    const int line4[4] = {l, -1, -1, -1}, beg4[4] = {beg, 0, 0, 0}, len4[4] = {len, 0, 0, 0};
                    emit((len + 31) / 32, 1, 0, 0, 0, 0, line4, beg4, len4);
                }
            }
            for (int q = 0; q < n_short; q += 4) {
                int line4[4] = {-1, -1, -1, -1}, beg4[4] = {0, 0, 0, 0}, len4[4] = {0, 0, 0, 0};
                for (int k = 0; k < 4 && q + k < n_short; ++k) {
                    const int l = short_sorted[(size_t)(q + k)];
                    line4[k] = l;
                    beg4[k] = ptr[l];
                    len4[k] = ptr[l + 1] - ptr[l];
                }
                emit((len4[0] + 7) / 8, 0, 0, 0, 0, 0, line4, beg4, len4);
            }
            cursor_items += n_items;
            if (pass == 1 && phase == 0) Q.n_long_rows = n_long_p;
        }
        if (pass == 0) {
            n_items_total = cursor_items;
            h_wptr = h_items + (size_t)kPcgItemInts * (size_t)n_items_total;
            if (staging_used + (size_t)kPcgItemInts * n_items_total + 2 * ((size_t)nw + 1) > staging.n)
                raise(REGOT_E_CUDA, "pcg: schedule staging too small (internal error)");
        } else {
            n_long += n_long_p;
            n_chunks += n_chunks_p;
        }
    }
    Q.n_long = n_long;
    Q.n_chunks = n_chunks;
    Q.items.ensure((size_t)kPcgItemInts * ((size_t)n_items_total + 1));
    Q.wptr.ensure(2 * ((size_t)nw + 1));
    Q.chunk_part.ensure((size_t)n_chunks * 2 + 2);
    Q.chunk_cnt.ensure((size_t)n_long + 1);
    if (n_items_total)
        RG_CUDA(cudaMemcpyAsync(Q.items.p, h_items, sizeof(int) * (size_t)kPcgItemInts * (size_t)n_items_total,
                                cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaMemcpyAsync(Q.wptr.p, h_wptr, sizeof(int) * 2 * ((size_t)nw + 1), cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaMemsetAsync(Q.chunk_cnt.p, 0, sizeof(unsigned int) * ((size_t)n_long + 1), st));
}

// ---- host: launch --------------------------------------------------------------------------------
// one launch solves up to 2 systems
static int pcg_schur_launch(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, const regot_sparse& S, int nrhs,
                            const DVec* const* rhs, DVec* const* sol, double rtol, int max_iter)
{
    const PcgSchedule& Q = S.pcg;
    const int nloc = (int)S.nloc, mfree = std::max((int)S.m - 1, 0);
    const int grid = Q.grid;
    const bool cluster = grid != ctx->sm_count;
    if (Q.nw != grid * kPcgWarpsPerCta || grid > kMaxGrid)
        raise(REGOT_E_CUDA, "pcg: schedule was built for a different grid (internal error)");
    if (!Q.fits) raise(REGOT_E_CUDA, "pcg: the persistent kernel needs the iterated vectors in shared memory (internal error)");
    const int smem = Q.vec_bytes + kPcgWarpsPerCta * Q.desc_cap * kPcgItemInts * 4 + kSchurScratchBytes;
    static bool attr_set = false;
    if (!attr_set) {
        RG_CUDA(cudaFuncSetAttribute(k_pcg_schur, cudaFuncAttributeMaxDynamicSharedMemorySize, kPcgSmemBudget));
        int per_sm = 0;
        RG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg_schur, kSchurThreads, kPcgSmemBudget));
        if (per_sm < 1) raise(REGOT_E_CUDA, "pcg: persistent kernel does not fit on an SM");
        attr_set = true;
    }
    if (smem > kPcgSmemBudget) raise(REGOT_E_CUDA, "pcg: shared-memory plan exceeds the budget (internal error)");
    const size_t va = (size_t)std::max(nloc, 1) * 2, vb = (size_t)std::max(mfree, 1) * 2;
    ws.cg.ensure(va + 6 * vb + 16);
    ws.cg_scal.ensure(16 + (size_t)grid * 8);
    if (!ws.h_cg) RG_CUDA(cudaMallocHost((void**)&ws.h_cg, sizeof(double) * 4096));

    SchurParams P;
    std::memset(&P, 0, sizeof(P));
    P.nloc = nloc;
    P.mfree = mfree;
    P.nrhs = nrhs;
    P.max_iter = max_iter;
    P.n_long = Q.n_long;
    P.n_long_rows = Q.n_long_rows;
    P.nw = Q.nw;
    P.cluster = cluster ? 1 : 0;
    P.fixed_iters = 0;
    if (const char* e = std::getenv("REGOT_B200_PCG_FIXED_ITERS")) P.fixed_iters = std::atoi(e);
    P.vec_bytes = Q.vec_bytes;
    P.stage_rows = Q.stage_rows ? 1 : 0;
    P.stage_cols = Q.stage_cols ? 1 : 0;
    P.desc_cap = Q.desc_cap;
#ifdef REGOT_PCG_TIMING
    const bool timing = true;
#else
    const bool timing = false;
#endif
    P.tol2 = rtol * rtol;
    P.col = S.col.p;
    P.val = S.val.p;
    P.cscrow = S.cscrow.p;
    P.cscval = S.cscval.p;
    P.dA = S.dA.p;
    P.dB = S.dB.p;
    P.mB = S.dS.p;
    P.items = Q.items.p;
    P.wptr = Q.wptr.p;
    P.chunk_part = Q.chunk_part.p;
    P.chunk_cnt = Q.chunk_cnt.p;
    for (int k = 0; k < 2; ++k) {
        const int kk = k < nrhs ? k : 0;
        P.rhs_a[k] = rhs[kk]->a.p;
        P.rhs_b[k] = rhs[kk]->b.p;
        sol[kk]->ensure(S.nloc, S.m);
        P.sol_a[k] = sol[kk]->a.p;
        P.sol_b[k] = sol[kk]->b.p;
    }
    double* base = ws.cg.p;
    P.ta = base;
    P.zb = base + va;
    P.wb = P.zb + vb;
    P.pb = P.wb + vb;
    P.sb = P.pb + vb;
    P.rb = P.sb + vb;
    P.xb = P.rb + vb;
    // [barrier counter | flagged words of the exchange], zeroed together: sequence numbers start at 1 in every launch
    const size_t xchg_words = ((size_t)grid * 4 + (size_t)Q.n_long * 2) * 2;
    ws.cg_xchg.ensure(2 + xchg_words);
    P.barrier = reinterpret_cast<unsigned int*>(ws.cg_xchg.p);
    P.xchg = ws.cg_xchg.p + 2;  // 16-byte aligned
    P.out = ws.cg_scal.p;
    RG_CUDA(cudaMemsetAsync(ws.cg_xchg.p, 0, sizeof(unsigned long long) * (2 + xchg_words), st));
    ws.cg_mbox.ensure();
    P.mbox = timing ? nullptr : ws.cg_mbox.data;
    P.seq = timing ? 0ULL : ws.cg_mbox.next();
    void* args[] = {&P};
    {
        ProfScope prof(ctx, st, 5);
        if (cluster) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(kSchurThreads);
            cfg.dynamicSmemBytes = (size_t)smem;
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = (unsigned)grid;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            RG_CUDA(cudaLaunchKernelExC(&cfg, (const void*)k_pcg_schur, args));
        } else {
            RG_CUDA(cudaLaunchCooperativeKernel((const void*)k_pcg_schur, dim3(grid), dim3(kSchurThreads), args, (size_t)smem, st));
        }
    }
    ++ctx->launches;
    if (timing) {
        RG_CUDA(cudaMemcpyAsync(ws.h_cg, ws.cg_scal.p, sizeof(double) * (4 + (size_t)grid * 8), cudaMemcpyDeviceToHost, st));
        RG_CUDA(cudaStreamSynchronize(st));
    } else {
        ws.cg_mbox.wait(st);
        for (int k = 0; k < 4; ++k) ws.h_cg[k] = ws.cg_mbox.data[k];
    }
    if (timing) {
        const char* nm[8] = {"init", "row", "bar1", "col", "reduce_delta", "update", "reduce_gamma", "final"};
        std::fprintf(stderr, "pcg_schur kcycles min/avg/max over CTAs:");
        for (int k = 0; k < 8; ++k) {
            double mn = 1e300, mx = 0.0, sum = 0.0;
            for (int b = 0; b < grid; ++b) {
                const double v = ws.h_cg[4 + (size_t)b * 8 + k];
                mn = std::min(mn, v);
                mx = std::max(mx, v);
                sum += v;
            }
            std::fprintf(stderr, " %s %.0f/%.0f/%.0f", nm[k], mn * 1e-3, sum / grid * 1e-3, mx * 1e-3);
        }
        std::fprintf(stderr, " | iters %.0f, %d long lines\n", ws.h_cg[0], Q.n_long);
#ifdef REGOT_PCG_TIMING
        long long tsub[8];
        RG_CUDA(cudaMemcpyFromSymbol(tsub, g_tsub, sizeof(tsub)));
        std::fprintf(stderr, "  grid_sum4 kcycles (one thread, cumulative): block_sum %lld | post+poll %lld | fence %lld | sync %lld | sum %lld\n",
                     tsub[0] / 1000, tsub[1] / 1000, tsub[2] / 1000, tsub[3] / 1000, tsub[4] / 1000);
        std::memset(tsub, 0, sizeof(tsub));
        RG_CUDA(cudaMemcpyToSymbol(g_tsub, tsub, sizeof(tsub)));
#endif
    }
    static const bool show_iters = std::getenv("REGOT_B200_PCG_ITERS") != nullptr;  // experiments
    if (show_iters) std::fprintf(stderr, "pcg iters: g-system %d, u-system %d\n", (int)ws.h_cg[0], nrhs > 1 ? (int)ws.h_cg[1] : -1);
    if (ws.h_cg[3] != 0.0) return -1;
    int it = 0;
    for (int k = 0; k < nrhs; ++k) it = std::max(it, (int)ws.h_cg[k]);
    return it;
}

int pcg_schur_persistent(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, const regot_sparse& S, int nrhs,
                         const DVec* const* rhs, DVec* const* sol, double rtol, int max_iter)
{
    int it = 0;
    for (int k0 = 0; k0 < nrhs; k0 += 2) {
        const int r = pcg_schur_launch(ctx, st, ws, S, std::min(2, nrhs - k0), rhs + k0, sol + k0, rtol, max_iter);
        if (r < 0) return -1;
        it = std::max(it, r);
    }
    return it;
}

}  // namespace rg
