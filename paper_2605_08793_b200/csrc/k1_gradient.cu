// k1_gradient.cu -- K1: the fused dual-gradient pass.
//
// Replaces regot::fused_gradient (dual.h:106-164) and, through its epilogue,
// marginal_error (dual.h:219-222), duality_gap (dual.h:225-229) and the
// phi'(gamma) = grad . d of the line search (splr.h:204-213).
//
// One coalesced pass over the row-major cost block: T_ij = exp(clamp((alpha_i +
// beta_j - M_ij) / eta)) is formed in registers from TMA-staged tiles and
// reduced to row sums, column sums and the objective.  No float atomics
// anywhere: every reduction has a fixed order, so results are bitwise
// reproducible for a fixed grid.
//
// Algorithmic bytes per launch: 8*nloc*m (M read once) + 16*(nloc+m).
#include "ctx.hpp"
#include "sweep.cuh"

#include <algorithm>
#include <cmath>
#include <cstring>

namespace rg {

struct GradParams {
    SweepGeom g;
    const double* alpha;  // nloc
    const double* beta;   // m
    ExpScale E;
    const double* exp_table;
    double* rowpart;  // n_panels x nloc
    double* colpart;  // n_segments x kTC
};

// One row of one tile for one lane: 8 plan entries from the lane's 8 staged costs.
// Returns the lane's partial row sum; column accumulators are updated in place.
template <bool kRagged>
__device__ __forceinline__ double gradient_row(const double (&mv)[kEPL], double ai, const double (&bj)[kEPL],
                                               double (&colacc)[kEPL], unsigned cmask, const ExpScale& E,
                                               uint32_t tbl_lane)
{
    double d[kEPL], T[kEPL];
#pragma unroll
    for (int k = 0; k < kEPL; ++k) d[k] = (ai + bj[k]) - mv[k];  // same association as dual.h:64
    plan_entries_dev<kEPL>(d, E, tbl_lane, T);
#pragma unroll
    for (int k = 0; k < kEPL; ++k) {
        if (kRagged) T[k] = (cmask >> k) & 1u ? T[k] : 0.0;
        colacc[k] += T[k];
    }
    return ((T[0] + T[1]) + (T[2] + T[3])) + ((T[4] + T[5]) + (T[6] + T[7]));
}

// The rows of one segment (the part of this CTA's tile range inside one column panel) for one
// consumer warp: `row` is the warp's row in the segment's first tile.  Row partials are staged per
// lane and flushed every kRowGroup tiles with one transposing sum.
template <bool kRagged, bool kCloud>
__device__ __forceinline__ void gradient_segment(const CloudRows& rows, RingCursor& ring, int lane, int row, int seg_tiles, int nloc,
                                                 const double* __restrict__ alpha, const double (&bj)[kEPL],
                                                 double (&colacc)[kEPL], unsigned cmask, const ExpScale& E,
                                                 uint32_t tbl_lane, double* stage, double* rowdst)
{
    // alpha of the next row is fetched one tile ahead so its latency hides behind the current row
    // (index clamped: the value is unused when the row does not exist)
    double ai_next = __ldg(alpha + min(row, nloc - 1));
    for (int done = 0; done < seg_tiles; done += kRowGroup) {
        const int cnt = min(kRowGroup, seg_tiles - done);
        const int row0 = row;
        for (int k = 0; k < cnt; ++k) {
            const double ai = ai_next;
            ai_next = __ldg(alpha + min(row + kTR, nloc - 1));
            double mv[kEPL];
            if (kCloud) {
                double2 m2[4];
                rows.row(m2, row, lane);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    mv[2 * q] = m2[q].x;
                    mv[2 * q + 1] = m2[q].y;
                }
            } else {
                ring.wait();
                ring.load_row(mv);
                ring.release(lane);
            }  // the costs are in registers: the slot refills while we compute
            double rs = 0.0;
            if (row < nloc) rs = gradient_row<kRagged>(mv, ai, bj, colacc, cmask, E, tbl_lane);
            stage[k * 32 + lane] = rs;
            row += kTR;
        }
        // flush: lane L sums 8 of the 32 lane-partials of staged row L/4
        __syncwarp();
        {
            const int k = lane >> 2, part = lane & 3;
            const double* src = stage + k * 32 + part * 8;
            double v = ((src[0] + src[1]) + (src[2] + src[3])) + ((src[4] + src[5]) + (src[6] + src[7]));
            v += shfl_xor_d(v, 1);
            v += shfl_xor_d(v, 2);
            const int r = row0 + k * kTR;
            if (part == 0 && k < cnt && r < nloc) rowdst[r] = v;
        }
        __syncwarp();
    }
}

template <bool kCloud>
__global__ void __launch_bounds__(sweep_threads<kCloud>(), 1)
k_gradient_sweep(const __grid_constant__ CUtensorMap tmap, const GradParams p)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const SweepSmem sm = sweep_prologue(smem, &tmap, p.exp_table, !kCloud);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    if (!kCloud && warp == kTR) {
        sweep_producer(&tmap, p.g, sm.tiles, sm.full, sm.empty);
        return;
    }
    CloudRows rows;
    if (kCloud) rows.init(p.g, sm.tiles);

    // ---- consumer warp `warp` owns row `warp` of every tile ----
    long t0, t1;
    sweep_range(p.g, t0, t1);
    if (t0 >= t1) return;
    const uint32_t tbl_lane = smem_u32(sm.table) + (uint32_t)(lane & 15) * 8u;
    double* stage = sm.scratch + warp * kTC;  // this warp's 2 KB: row staging, then column exchange
    const ExpScale E = p.E;
    const int nloc = p.g.nloc, m = p.g.m, nrt = p.g.n_row_tiles;
    int seg = p.g.cta_seg0[blockIdx.x];
    RingCursor ring;
    ring.init(sm, warp, lane);

    int left = (int)(t1 - t0);                 // tiles still to process
    int panel = (int)(t0 / nrt);
    int rt = (int)(t0 - (long)panel * nrt);    // row tile inside the panel

    while (left > 0) {
        // ---- one segment: the rest of panel `panel` (or of the range) ----
        const int seg_tiles = min(nrt - rt, left);
        const int col0 = panel * kTC;
        double bj[kEPL], colacc[kEPL];
        unsigned cmask = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int c = col0 + 64 * q + 2 * lane + e;
                const bool ok = c < m;
                bj[2 * q + e] = ok ? __ldg(p.beta + c) : 0.0;
                cmask |= (ok ? 1u : 0u) << (2 * q + e);
                colacc[2 * q + e] = 0.0;
            }
        }
        if (kCloud) rows.load_panel(col0);
        double* const rowdst = p.rowpart + (size_t)panel * nloc;
        if (col0 + kTC > m)
            gradient_segment<true, kCloud>(rows, ring, lane, rt * kTR + warp, seg_tiles, nloc, p.alpha, bj, colacc, cmask, E, tbl_lane,
                                   stage, rowdst);
        else
            gradient_segment<false, kCloud>(rows, ring, lane, rt * kTR + warp, seg_tiles, nloc, p.alpha, bj, colacc, cmask, E, tbl_lane,
                                    stage, rowdst);
        left -= seg_tiles;
        rt += seg_tiles;

        // column partials of this segment: exchange through shared memory,
        // summed over the kTR warps in warp order
#pragma unroll
        for (int q = 0; q < 4; ++q)
            reinterpret_cast<double2*>(stage)[q * 32 + lane] = make_double2(colacc[2 * q], colacc[2 * q + 1]);
        bar_sync(1, kConsumerThreads);
        if (threadIdx.x < kTC) {
            double v = 0.0;
#pragma unroll
            for (int w = 0; w < kTR; ++w) v += sm.scratch[w * kTC + threadIdx.x];
            p.colpart[(size_t)seg * kTC + threadIdx.x] = v;
        }
        bar_sync(1, kConsumerThreads);
        ++seg;
        if (rt == nrt) {
            rt = 0;
            ++panel;
        }
    }
}

// ---- epilogue 1: reduce partials, row-side scalars ---------------------------------
// pack[0..m)   = local column sums
// pack[m + k]  = row-side scalars: 0 sum(r) 1 alpha.a 2 sum|r-a| 3 alpha.(r-a) 4 |r-a|^2 5 (r-a).d_alpha
constexpr int kNScal = 8;
constexpr int kFinThreads = 256;

// double-double: an unevaluated sum hi + lo with |lo| <= ulp(hi) / 2
struct dd {
    double hi, lo;
};
__device__ __forceinline__ dd dd_add(dd a, dd b)
{
    const double s = a.hi + b.hi, bb = s - a.hi;
    const double e = ((a.hi - (s - bb)) + (b.hi - bb)) + (a.lo + b.lo);
    dd r;
    r.hi = s + e;
    r.lo = e - (r.hi - s);
    return r;
}
__device__ __forceinline__ dd dd_add_d(dd a, double b)  // b exact
{
    const double s = a.hi + b, bb = s - a.hi;
    const double e = ((a.hi - (s - bb)) + (b - bb)) + a.lo;
    dd r;
    r.hi = s + e;
    r.lo = e - (r.hi - s);
    return r;
}
__device__ __forceinline__ dd dd_add_prod(dd a, double x, double y)  // a + x y with the product's rounding error kept
{
    const double p = __dmul_rn(x, y), pe = __fma_rn(x, y, -p);  // no contraction of the product into the sums below
    dd r = dd_add_d(a, p);
    r.lo += pe;
    return r;
}
__device__ __forceinline__ dd dd_shfl_xor(dd a, int mask)
{
    dd r;
    r.hi = shfl_xor_d(a.hi, mask);
    r.lo = shfl_xor_d(a.lo, mask);
    return r;
}
// CTA-wide sum of three double-doubles in a fixed order; valid in thread 0.  scratch: 6 x (kFinThreads / 32) doubles.
__device__ __forceinline__ void dd_block_sum3(dd (&v)[3], double* scratch)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = kFinThreads / 32;
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] = dd_add(v[k], dd_shfl_xor(v[k], o));
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            scratch[(2 * k) * nwarp + warp] = v[k].hi;
            scratch[(2 * k + 1) * nwarp + warp] = v[k].lo;
        }
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            dd t;
            t.hi = lane < nwarp ? scratch[(2 * k) * nwarp + lane] : 0.0;
            t.lo = lane < nwarp ? scratch[(2 * k + 1) * nwarp + lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t = dd_add(t, dd_shfl_xor(t, o));
            v[k] = t;
        }
    }
    __syncthreads();
}
// the high part of a double-double cut into 30 + 23 significant bits (Veltkamp): sums of a few such 30-bit pieces over
// the ranks of an allreduce are exact in any order, the 23-bit remainders and the low parts sum with errors far below
// what the objective needs
__device__ __forceinline__ void split30(double hi, double& h1, double& h2)
{
    const double c = 8388609.0 * hi;  // 2^23 + 1
    h1 = c - (c - hi);
    h2 = hi - h1;
}
constexpr int kNScalPack = 13;  // row-side scalars behind the m column sums of the allreduce payload: 6 plain + 2 x 3 pieces + the
                                // rank's fast-Sinkhorn flag (summed: every rank must take the same redo decision)

struct Fin1Params {
    int nloc, m, n_panels;
    const double* rowpart;
    const double* colpart;
    const int* panel_seg0;
    const double* alpha;
    const double* a;
    const double* dir_a;  // nullable
    double* row_sums;
    double* g_alpha;
    double* pack;
    double* partials;  // gridDim.x * kNScal
    unsigned int* ticket;
    int extended;      // also sum r and alpha.a in double-double -> pack[m + 6 .. m + 12) as (30-bit, 23-bit, low) pieces
    const unsigned int* sk_flag;  // this rank's fast-Sinkhorn flag -> pack[m + 12] (the two-kernel form)
};

__device__ __forceinline__ bool last_block_done(unsigned int* ticket)
{
    __shared__ bool is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int prev = atomicAdd(ticket, 1u);
        is_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (is_last) __threadfence();
    return is_last;
}

// sum of per-block partials in block order; valid in every lane of warp 0
__device__ __forceinline__ double ordered_partial_sum(const double* partials, int k, int nblocks, int lane)
{
    double s = 0.0;
    for (int b = lane; b < nblocks; b += 32) s += partials[(size_t)b * kNScal + k];
    return warp_sum(s);
}

__global__ void __launch_bounds__(kFinThreads) k_gradient_fin1(const Fin1Params p)
{
    __shared__ double scratch[kNScal * (kFinThreads / 32)];
    double acc[6] = {0, 0, 0, 0, 0, 0};
    dd ex[3] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    const int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.nloc; i += stride) {
        // panel order (fixed), 8 loads in flight
        double r = 0.0;
        for (int P0 = 0; P0 < p.n_panels; P0 += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = (P0 + u < p.n_panels) ? p.rowpart[(size_t)(P0 + u) * p.nloc + i] : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (P0 + u < p.n_panels) r += v[u];
        }
        const double al = p.alpha[i], ai = p.a[i];
        const double ga = r - ai;
        p.row_sums[i] = r;
        p.g_alpha[i] = ga;
        acc[0] += r;
        acc[1] += al * ai;
        acc[2] += fabs(ga);
        acc[3] += al * ga;
        acc[4] += ga * ga;
        if (p.dir_a) acc[5] += ga * p.dir_a[i];
        if (p.extended) {
            ex[0] = dd_add_d(ex[0], r);
            ex[1] = dd_add_prod(ex[1], al, ai);
        }
    }
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < p.m; j += stride) {
        const int P = j / kTC, off = j - P * kTC;
        double c = 0.0;
        const int s1 = p.panel_seg0[P + 1];
        for (int sg = p.panel_seg0[P]; sg < s1; sg += 8) {  // segment order (fixed), 8 loads in flight
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = (sg + u < s1) ? p.colpart[(size_t)(sg + u) * kTC + off] : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (sg + u < s1) c += v[u];
        }
        p.pack[j] = c;
    }
    block_sum<6>(acc, scratch);
    if (threadIdx.x == 0)
        for (int k = 0; k < 6; ++k) p.partials[(size_t)blockIdx.x * kNScal + k] = acc[k];
    double* const ddpart = p.partials + (size_t)(2 * gridDim.x) * 12;  // behind the plain partials of either finalize form
    if (p.extended) {
        dd_block_sum3(ex, scratch);
        if (threadIdx.x == 0)
            for (int k = 0; k < 2; ++k) {
                ddpart[(size_t)blockIdx.x * 6 + 2 * k] = ex[k].hi;
                ddpart[(size_t)blockIdx.x * 6 + 2 * k + 1] = ex[k].lo;
            }
    }
    if (last_block_done(p.ticket)) {
        if (threadIdx.x < 32) {
            for (int k = 0; k < 6; ++k) {
                const double v = ordered_partial_sum(p.partials, k, gridDim.x, threadIdx.x);
                if (threadIdx.x == 0) p.pack[p.m + k] = v;
            }
            for (int k = 0; k < 2; ++k) {
                dd t = {0.0, 0.0};
                if (p.extended) {
                    for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) {
                        dd u = {ddpart[(size_t)b * 6 + 2 * k], ddpart[(size_t)b * 6 + 2 * k + 1]};
                        t = dd_add(t, u);
                    }
                    for (int o = 16; o > 0; o >>= 1) t = dd_add(t, dd_shfl_xor(t, o));
                }
                if (threadIdx.x == 0) {
                    double h1, h2;
                    split30(t.hi, h1, h2);
                    p.pack[p.m + 6 + 3 * k] = h1;
                    p.pack[p.m + 7 + 3 * k] = h2;
                    p.pack[p.m + 8 + 3 * k] = t.lo;
                }
            }
            if (threadIdx.x == 0) {
                p.pack[p.m + 12] = (double)*p.sk_flag;
                *p.ticket = 0u;
            }
        }
    }
}

// ---- epilogue 2 (after the allreduce of pack): column-side scalars, objective -------
struct Fin2Params {
    int m;
    double eta;
    const double* pack;  // m column sums + row-side scalars (global after allreduce)
    const double* beta;
    const double* b;
    const double* dir_b;  // nullable
    double* col_sums;
    double* g_beta;
    double* partials;
    unsigned int* ticket;
    GradScalars* out;
    double* mbox;  // host mailbox: the scalars go straight to pinned host memory
    unsigned long long seq;
    const unsigned int* sk_flag;
    int extended;  // objective in double-double from the pieces in pack[m + 6 ..) and beta.b summed here
};

__global__ void __launch_bounds__(kFinThreads) k_gradient_fin2(const Fin2Params p)
{
    __shared__ double scratch[kNScal * (kFinThreads / 32)];
    // 0 beta.b (free part) 1 sum|c-b| (all m) 2 beta.(c-b) 3 |c-b|^2 (free part) 4 (c-b).d_beta (free part)
    double acc[5] = {0, 0, 0, 0, 0};
    dd ex[3] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    const int stride = gridDim.x * blockDim.x;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < p.m; j += stride) {
        const double c = p.pack[j], bj = p.b[j], be = p.beta[j];
        const double gb = c - bj;
        if (p.extended && j < p.m - 1) ex[0] = dd_add_prod(ex[0], be, bj);
        p.col_sums[j] = c;
        p.g_beta[j] = gb;
        acc[1] += fabs(gb);
        acc[2] += be * gb;
        if (j < p.m - 1) {
            acc[0] += be * bj;
            acc[3] += gb * gb;
            if (p.dir_b) acc[4] += gb * p.dir_b[j];
        }
    }
    block_sum<5>(acc, scratch);
    if (threadIdx.x == 0)
        for (int k = 0; k < 5; ++k) p.partials[(size_t)blockIdx.x * kNScal + k] = acc[k];
    double* const ddpart = p.partials + (size_t)(2 * gridDim.x) * 12;
    if (p.extended) {
        dd_block_sum3(ex, scratch);
        if (threadIdx.x == 0) {
            ddpart[(size_t)blockIdx.x * 6] = ex[0].hi;
            ddpart[(size_t)blockIdx.x * 6 + 1] = ex[0].lo;
        }
    }
    if (last_block_done(p.ticket)) {
        if (threadIdx.x < 32) {
            double c[5];
            for (int k = 0; k < 5; ++k) c[k] = ordered_partial_sum(p.partials, k, gridDim.x, threadIdx.x);
            dd bb = {0.0, 0.0};
            if (p.extended) {
                for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) {
                    dd u = {ddpart[(size_t)b * 6], ddpart[(size_t)b * 6 + 1]};
                    bb = dd_add(bb, u);
                }
                for (int o = 16; o > 0; o >>= 1) bb = dd_add(bb, dd_shfl_xor(bb, o));
            }
            if (threadIdx.x == 0) {
                const double* S = p.pack + p.m;
                GradScalars o;
                o.total_mass = S[0];
                o.f = p.eta * S[0] - S[1] - c[0];  // dual.h:157-158
                o.row_abs = S[2];
                o.col_abs = c[1];
                o.marginal_error = S[2] + c[1];  // dual.h:219-222
                o.duality_gap = S[3] + c[2];     // dual.h:225-229
                o.grad_sqnorm = S[4] + c[3];
                o.g_dot_d = S[5] + c[4];
                o.lse_flag = p.pack[p.m + 12];  // any rank's flag (summed by the allreduce; this rank's own on one GPU)
                o.f_lo = 0.0;
                if (p.extended) {
                    // sum r and alpha.a arrive as (30-bit, 23-bit, low) pieces summed over the ranks
                    dd sr = {S[6], 0.0}, aa = {S[9], 0.0};
                    sr = dd_add_d(dd_add_d(sr, S[7]), S[8]);
                    aa = dd_add_d(dd_add_d(aa, S[10]), S[11]);
                    const double ph = __dmul_rn(p.eta, sr.hi), pe = __fma_rn(p.eta, sr.hi, -ph) + p.eta * sr.lo;
                    dd fx = {ph, pe};
                    dd neg1 = {-aa.hi, -aa.lo}, neg2 = {-bb.hi, -bb.lo};
                    fx = dd_add(fx, neg1);
                    fx = dd_add(fx, neg2);
                    o.f = fx.hi;
                    o.f_lo = fx.lo;
                }
                *p.out = o;
                *p.ticket = 0u;
                static_assert(sizeof(GradScalars) == 10 * sizeof(double), "GradScalars is 10 doubles");
                mailbox_post(p.mbox, reinterpret_cast<const double*>(&o), 10, p.seq);
            }
        }
    }
}

// ---- dense plan (tests / diagnostics; dual.h:83-94) ---------------------------------
__global__ void k_plan(int nloc, int m, const CostViewDev cost, const double* __restrict__ alpha,
                       const double* __restrict__ beta, const ExpScale E, const double* __restrict__ exp_table,
                       double* __restrict__ T)
{
    __shared__ double tbl[kExpN * kExpCopies];
    exp_table_fill(tbl, exp_table, threadIdx.x, blockDim.x);
    __syncthreads();
    const uint32_t tbl_lane = smem_u32(tbl) + (uint32_t)(threadIdx.x & 15) * 8u;
    const long total = (long)nloc * m;
    for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (long)gridDim.x * blockDim.x) {
        const int i = (int)(q / m), j = (int)(q % m);
        T[q] = plan_entry_dev((alpha[i] + beta[j]) - cost_at(cost, i, j), E, tbl_lane);
    }
}

// ---- host side ------------------------------------------------------------------------
// ---- both epilogues in one kernel (one GPU: no allreduce between them) -----------------------------------
// Same loops and the same per-thread summation order as k_gradient_fin1 followed by k_gradient_fin2 on the same
// grid (so a square problem gets bit-identical scalars); one launch and one grid-wide hand-over less per evaluation.
struct Fin12Params {
    Fin1Params r;
    Fin2Params c;
    int extended;  // the three sums of the objective in double-double
};
constexpr int kNScal12 = 12;
__global__ void __launch_bounds__(kFinThreads) k_gradient_fin12(const Fin12Params q)
{
    const Fin1Params& p = q.r;
    const Fin2Params& f = q.c;
    __shared__ double scratch[kNScal12 * (kFinThreads / 32)];
    // 0..5 as in k_gradient_fin1; 6 beta.b (free part) 7 sum|c-b| (all m) 8 beta.(c-b) 9 |c-b|^2 (free part) 10 (c-b).d_beta (free part)
    double acc[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    dd ex[3] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};  // extended: sum r, alpha.a, beta.b (free part)
    const int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.nloc; i += stride) {
        double r = 0.0;
        for (int P0 = 0; P0 < p.n_panels; P0 += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = (P0 + u < p.n_panels) ? p.rowpart[(size_t)(P0 + u) * p.nloc + i] : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (P0 + u < p.n_panels) r += v[u];
        }
        const double al = p.alpha[i], ai = p.a[i];
        const double ga = r - ai;
        p.row_sums[i] = r;
        p.g_alpha[i] = ga;
        acc[0] += r;
        acc[1] += al * ai;
        acc[2] += fabs(ga);
        acc[3] += al * ga;
        acc[4] += ga * ga;
        if (p.dir_a) acc[5] += ga * p.dir_a[i];
        if (q.extended) {
            ex[0] = dd_add_d(ex[0], r);
            ex[1] = dd_add_prod(ex[1], al, ai);
        }
    }
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < p.m; j += stride) {
        const int P = j / kTC, off = j - P * kTC;
        double c = 0.0;
        const int s1 = p.panel_seg0[P + 1];
        for (int sg = p.panel_seg0[P]; sg < s1; sg += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = (sg + u < s1) ? p.colpart[(size_t)(sg + u) * kTC + off] : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (sg + u < s1) c += v[u];
        }
        const double bj = f.b[j], be = f.beta[j];
        if (q.extended && j < p.m - 1) ex[2] = dd_add_prod(ex[2], be, bj);
        const double gb = c - bj;
        f.col_sums[j] = c;
        f.g_beta[j] = gb;
        acc[7] += fabs(gb);
        acc[8] += be * gb;
        if (j < p.m - 1) {
            acc[6] += be * bj;
            acc[9] += gb * gb;
            if (f.dir_b) acc[10] += gb * f.dir_b[j];
        }
    }
    block_sum<11>(acc, scratch);
    if (threadIdx.x == 0)
        for (int k = 0; k < 11; ++k) p.partials[(size_t)blockIdx.x * kNScal12 + k] = acc[k];
    if (q.extended) {
        dd_block_sum3(ex, scratch);
        if (threadIdx.x == 0)
            for (int k = 0; k < 3; ++k) {
                p.partials[(size_t)(2 * gridDim.x) * kNScal12 + (size_t)blockIdx.x * 6 + 2 * k] = ex[k].hi;
                p.partials[(size_t)(2 * gridDim.x) * kNScal12 + (size_t)blockIdx.x * 6 + 2 * k + 1] = ex[k].lo;
            }
    }
    if (last_block_done(p.ticket)) {
        if (threadIdx.x < 32) {
            double t[11];
            for (int k = 0; k < 11; ++k) {
                double s = 0.0;
                for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) s += p.partials[(size_t)b * kNScal12 + k];
                t[k] = warp_sum(s);
            }
            if (threadIdx.x == 0) {
                GradScalars o;
                o.total_mass = t[0];
                o.f = f.eta * t[0] - t[1] - t[6];  // dual.h:157-158
                o.row_abs = t[2];
                o.col_abs = t[7];
                o.marginal_error = t[2] + t[7];  // dual.h:219-222
                o.duality_gap = t[3] + t[8];     // dual.h:225-229
                o.grad_sqnorm = t[4] + t[9];
                o.g_dot_d = t[5] + t[10];
                o.lse_flag = (double)*f.sk_flag;
                o.f_lo = 0.0;
                *f.out = o;
            }
            if (q.extended) {
                // f = eta sum r - alpha.a - beta.b with the three sums in double-double (CTA order, then lanes)
                dd tx[3];
                for (int k = 0; k < 3; ++k) {
                    dd t = {0.0, 0.0};
                    for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) {
                        const double* src = p.partials + (size_t)(2 * gridDim.x) * kNScal12 + (size_t)b * 6 + 2 * k;
                        dd u = {src[0], src[1]};
                        t = dd_add(t, u);
                    }
                    for (int o2 = 16; o2 > 0; o2 >>= 1) t = dd_add(t, dd_shfl_xor(t, o2));
                    tx[k] = t;
                }
                if (threadIdx.x == 0) {
                    // eta * (hi + lo): product of the high parts with its error, the low part's product in plain doubles
                    const double ph = __dmul_rn(f.eta, tx[0].hi), pe = __fma_rn(f.eta, tx[0].hi, -ph) + f.eta * tx[0].lo;
                    dd fx = {ph, pe};
                    dd neg1 = {-tx[1].hi, -tx[1].lo}, neg2 = {-tx[2].hi, -tx[2].lo};
                    fx = dd_add(fx, neg1);
                    fx = dd_add(fx, neg2);
                    f.out->f = fx.hi;
                    f.out->f_lo = fx.lo;
                }
            }
            if (threadIdx.x == 0) {
                GradScalars o = *f.out;
                *p.ticket = 0u;
                mailbox_post(f.mbox, reinterpret_cast<const double*>(&o), 10, f.seq);
            }
        }
    }
}

static int fin_grid(const regot_ctx* ctx, long work)
{
    long g = (work + kFinThreads - 1) / kFinThreads;
    return (int)std::max<long>(1, std::min<long>(g, 2L * ctx->sm_count));
}

static GradParams make_params(regot_ctx* ctx, SweepWS& ws, const double* alpha, const double* beta)
{
    GradParams p;
    p.g.nloc = (int)ctx->prob.nloc;
    p.g.m = (int)ctx->prob.m;
    p.g.n_row_tiles = ctx->plan.n_row_tiles;
    p.g.n_panels = ctx->plan.n_panels;
    p.g.total_tiles = ctx->plan.total_tiles;
    p.g.cta_seg0 = ctx->plan.d_cta_seg0.p;
    // M larger than ~half of L2 streams through with evict-first; small problems stay L2 resident
    p.g.evict_first = ((double)ctx->prob.nloc * (double)ctx->prob.ld * 8.0 > 48e6) ? 1 : 0;
    p.g.cloud = cloud_geom(ctx);
    p.alpha = alpha;
    p.beta = beta;
    p.E = make_exp_scale(ctx->prob.eta);
    p.exp_table = ctx->exp_table.p;
    p.rowpart = ws.rowpart.p;
    p.colpart = ws.colpart.p;
    return p;
}

void launch_gradient_sweep_only(regot_ctx* ctx, cudaStream_t st, SweepWS& ws, const double* alpha, const double* beta)
{
    static bool attr_set = false;
    if (!attr_set) {
        RG_CUDA(cudaFuncSetAttribute(k_gradient_sweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSweepSmem));
        RG_CUDA(cudaFuncSetAttribute(k_gradient_sweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSweepSmem));
        attr_set = true;
    }
    const GradParams p = make_params(ctx, ws, alpha, beta);
    ProfScope prof(ctx, st, 0);
    if (ctx->prob.on_the_fly)
        k_gradient_sweep<true><<<ctx->plan.grid, kCloudSweepThreads, kSweepSmem, st>>>(ctx->prob.tmap, p);
    else
        k_gradient_sweep<false><<<ctx->plan.grid, kSweepThreads, kSweepSmem, st>>>(ctx->prob.tmap, p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
}

void launch_gradient(regot_ctx* ctx, cudaStream_t st, SweepWS& ws, ncclComm* comm, const double* alpha,
                     const double* beta, const double* dir_a, const double* dir_b, GradOut& out)
{
    const DeviceProblem& pr = ctx->prob;
    out.ensure(pr.nloc, pr.m);
    ProfScope prof_op(ctx, st, 7);  // the whole fused_gradient: sweep + both finalize kernels (+ the allreduce)
    launch_gradient_sweep_only(ctx, st, ws, alpha, beta);

    const int g1 = fin_grid(ctx, std::max<long>(pr.nloc, pr.m));
    Fin1Params f1;
    f1.nloc = (int)pr.nloc;
    f1.m = (int)pr.m;
    f1.n_panels = ctx->plan.n_panels;
    f1.rowpart = ws.rowpart.p;
    f1.colpart = ws.colpart.p;
    f1.panel_seg0 = ctx->plan.d_panel_seg0.p;
    f1.alpha = alpha;
    f1.a = pr.a;
    f1.dir_a = dir_a;
    f1.row_sums = out.sums.a.p;
    f1.g_alpha = out.g.a.p;
    f1.pack = ws.pack.p;
    f1.partials = ws.partials.p;
    f1.ticket = ws.ticket.p;
    f1.extended = ctx->extended_f ? 1 : 0;
    f1.sk_flag = ws.sk_flag.p;
    const bool fused = !ctx->sharded && ctx->fused_finalize;
    if (!fused) {
        k_gradient_fin1<<<g1, kFinThreads, 0, st>>>(f1);
        RG_CUDA(cudaGetLastError());
        ++ctx->launches;
    }

    if (ctx->sharded) allreduce_sum(ctx, comm, ws.pack.p, (size_t)pr.m + kNScalPack, st);

    const int g2 = fin_grid(ctx, pr.m);
    Fin2Params f2;
    f2.m = (int)pr.m;
    f2.eta = pr.eta;
    f2.pack = ws.pack.p;
    f2.beta = beta;
    f2.b = pr.b;
    f2.dir_b = dir_b;
    f2.col_sums = out.sums.b.p;
    f2.g_beta = out.g.b.p;
    f2.partials = ws.partials.p;
    f2.ticket = ws.ticket.p + 1;
    f2.out = ws.d_scal.p;
    f2.mbox = ws.mbox.data;
    f2.seq = ws.mbox.next();
    f2.sk_flag = ws.sk_flag.p;
    f2.extended = ctx->extended_f ? 1 : 0;
    if (fused) {
        Fin12Params f12;
        f12.r = f1;
        f12.c = f2;
        f12.extended = ctx->extended_f ? 1 : 0;
        k_gradient_fin12<<<g1, kFinThreads, 0, st>>>(f12);
    } else {
        k_gradient_fin2<<<g2, kFinThreads, 0, st>>>(f2);
    }
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
}

void sync_scalars(regot_ctx* ctx, cudaStream_t st, SweepWS& ws, GradOut& out)
{
    (void)ctx;
    ws.mbox.wait(st);
    std::memcpy(&out.sc, ws.mbox.data, sizeof(GradScalars));
}

void launch_plan(regot_ctx* ctx, cudaStream_t st, const double* alpha, const double* beta, double* T_rowmajor)
{
    const DeviceProblem& pr = ctx->prob;
    const long total = (long)pr.nloc * pr.m;
    const int grid = (int)std::max<long>(1, std::min<long>((total + 255) / 256, 8L * ctx->sm_count));
    k_plan<<<grid, 256, 0, st>>>((int)pr.nloc, (int)pr.m, cost_view_dev(ctx), alpha, beta,
                                 make_exp_scale(pr.eta), ctx->exp_table.p, T_rowmajor);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
}

}  // namespace rg
