// sweep.cuh -- the TMA-fed panel sweep skeleton shared by the fused-gradient
// (K1) and log-sum-exp (K7/K8) kernels.
//
// Layout: M is row-major (nloc x ld) in HBM.  It is cut into tiles of
// kTR rows x kTC columns; tiles are ordered column-panel-major and every CTA
// of a persistent grid owns one contiguous range of tile ids (SweepPlan in
// ctx.hpp), so the load is balanced to within one tile without atomics.
//
// CTA = kTR consumer warps + 1 producer warp.  The producer's elected lane
// streams tiles with cp.async.bulk.tensor.2d (TMA) into a kStages-deep ring of
// shared-memory buffers, signalling `full` mbarriers; consumer warp w owns row
// w of every tile (lane l owns columns 2l+64q+{0,1}, q=0..3, read with
// conflict-free 128-bit shared loads) and releases the slot through the
// `empty` mbarrier.  Out-of-range rows/columns of edge tiles are zero-filled by
// TMA and masked in the consumers.
#pragma once

#include "common.cuh"
#include "ctx.hpp"

namespace rg {

constexpr int kTR = 16;               // tile rows == consumer warps
constexpr int kTC = 256;              // tile columns (8 per lane)
constexpr int kStages = 4;            // TMA ring depth
constexpr int kEPL = kTC / kWarp;     // elements per lane per row = 8
constexpr int kTileElems = kTR * kTC;
constexpr int kTileBytes = kTileElems * 8;
constexpr int kConsumerThreads = kTR * kWarp;
constexpr int kSweepThreads = kConsumerThreads + kWarp;
constexpr int kRowGroup = 8;          // row partials staged per warp before a flush
// point-cloud problems whose cost is formed on the fly have no producer warp and no tile ring: every
// consumer warp computes its own row from the row's point and a shared-memory copy of the panel's
// 256 target points (CloudRows below), which takes the ring's place in shared memory
constexpr int kCloudSweepThreads = kConsumerThreads;
constexpr int kCloudMaxD = (kStages * kTileBytes) / (kTC * 8);  // coordinates that fit: 64

// dynamic shared memory carve-up (bytes)
constexpr int kSmemTiles = 0;
constexpr int kSmemTable = kSmemTiles + kStages * kTileBytes;
constexpr int kSmemScratch = kSmemTable + kExpTableBytes;        // kTR x kTC doubles
constexpr int kSmemBars = kSmemScratch + kTR * kTC * 8;
constexpr int kSweepSmem = kSmemBars + 2 * kStages * 8 + 64;

// Squared-Euclidean cost of point clouds, normalised by its maximum (problem.h:53-61, 124-132):
// the ONE definition used by the materialising kernel, the on-the-fly tile producers and the
// entry-wise readers, so a cost entry has the same bits wherever it is formed.  Coordinates are
// accumulated in order with separately rounded multiply and add (what the reference's and the host
// generators' loops do), then divided by the maximum.
struct CloudGeom {
    const double* X;  // nloc x d, this rank's rows
    const double* Y;  // m x d
    int d;
    double cmax;      // maximum of the un-normalised cost over the GLOBAL matrix
    double inv_cmax;  // RN(1 / cmax)
    int fast_div;     // set_pointcloud verified cloud_div_fast == true division on every entry of this block
};
// s / cmax, correctly rounded, from the reciprocal and two residual corrections (Markstein): 5 fused
// multiply-adds that interleave across entries, where the generic division is a ~20-instruction
// dependent sequence with a slow-path call.  The identity with true division is not assumed: it is
// CHECKED on every entry of the block when the problem is set (k_cloud_verify_div) and the exact
// division is used if a single entry differs.
__device__ __forceinline__ double cloud_div_fast(double s, double cmax, double inv_cmax)
{
    const double q0 = s * inv_cmax;
    const double q1 = __fma_rn(__fma_rn(-q0, cmax, s), inv_cmax, q0);
    return __fma_rn(__fma_rn(-q1, cmax, s), inv_cmax, q1);
}
__device__ __forceinline__ double cloud_div(double s, const CloudGeom& c)
{
    return c.fast_div ? cloud_div_fast(s, c.cmax, c.inv_cmax) : __ddiv_rn(s, c.cmax);
}
__device__ __forceinline__ double cloud_sqdist(const double* __restrict__ xi, const double* __restrict__ yj, int d)
{
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
        const double df = __dsub_rn(__ldg(xi + k), __ldg(yj + k));
        s = __dadd_rn(s, __dmul_rn(df, df));
    }
    return s;
}
__device__ __forceinline__ double cloud_cost(const CloudGeom& c, int i, int j)
{
    return cloud_div(cloud_sqdist(c.X + (size_t)i * c.d, c.Y + (size_t)j * c.d, c.d), c);
}

struct SweepGeom {
    int nloc, m;
    int n_row_tiles, n_panels;
    long total_tiles;
    const int* cta_seg0;  // grid + 1
    int evict_first;      // stream M through L2 with an evict-first policy
    CloudGeom cloud;      // on-the-fly cost (kCloud kernels only)
};

__device__ __forceinline__ void sweep_range(const SweepGeom& g, long& t0, long& t1)
{
    t0 = (g.total_tiles * (long)blockIdx.x) / (long)gridDim.x;
    t1 = (g.total_tiles * (long)(blockIdx.x + 1)) / (long)gridDim.x;
}

// Producer warp body: stream this CTA's tile range through the ring.
__device__ __forceinline__ void sweep_producer(const CUtensorMap* tmap, const SweepGeom& g, double* tiles,
                                               uint64_t* full, uint64_t* empty)
{
    if ((threadIdx.x & 31) != 0) return;
    long t0, t1;
    sweep_range(g, t0, t1);
    const uint64_t pol = l2_policy_evict_first();
    int s = 0;
    uint32_t ph = 0;
    for (long t = t0; t < t1; ++t) {
        mbar_wait(&empty[s], ph ^ 1u);
        const int panel = (int)(t / g.n_row_tiles), rt = (int)(t % g.n_row_tiles);
        mbar_arrive_expect_tx(&full[s], kTileBytes);
        if (g.evict_first) tma_load_2d(tiles + (size_t)s * kTileElems, tmap, &full[s], panel * kTC, rt * kTR, pol);
        else tma_load_2d(tiles + (size_t)s * kTileElems, tmap, &full[s], panel * kTC, rt * kTR);
        if (++s == kStages) {
            s = 0;
            ph ^= 1u;
        }
    }
}

// Common prologue: barriers + exp table.  Returns pointers into dynamic smem.
struct SweepSmem {
    double* tiles;
    double* table;
    double* scratch;
    uint64_t* full;
    uint64_t* empty;
};
// use_tma == false (on-the-fly cost): the ring and its barriers stay unused
__device__ __forceinline__ SweepSmem sweep_prologue(unsigned char* smem, const CUtensorMap* tmap,
                                                    const double* __restrict__ exp_table, bool use_tma = true)
{
    SweepSmem s;
    s.tiles = reinterpret_cast<double*>(smem + kSmemTiles);
    s.table = reinterpret_cast<double*>(smem + kSmemTable);
    s.scratch = reinterpret_cast<double*>(smem + kSmemScratch);
    s.full = reinterpret_cast<uint64_t*>(smem + kSmemBars);
    s.empty = s.full + kStages;
    if (threadIdx.x == 0) {
        if (use_tma) tma_prefetch_desc(tmap);
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&s.full[i], 1);
            mbar_init(&s.empty[i], kTR);
        }
        fence_mbar_init();
    }
    exp_table_fill(s.table, exp_table, threadIdx.x, blockDim.x);
    __syncthreads();
    return s;
}

template <bool kCloud>
constexpr int sweep_threads() { return kCloud ? kCloudSweepThreads : kSweepThreads; }

// Consumer side of the on-the-fly kernels.  load_panel(): the consumer warps copy the panel's 256
// target points into shared memory, coordinate-major ([k][256], so a lane's 8 columns of one
// coordinate are four conflict-free 16-byte loads).  row(): the lane's 8 cost entries of one row, in
// the column order of the resident-matrix tiles (columns 2 lane + 64 q + {0, 1}), with the arithmetic
// of cloud_sqdist / cloud_div -- the same bits as the materialised matrix.
struct CloudRows {
    uint32_t ysm;
    CloudGeom c;
    int nloc, m;
    __device__ __forceinline__ void init(const SweepGeom& g, const double* tiles)
    {
        ysm = smem_u32(tiles);
        c = g.cloud;
        nloc = g.nloc;
        m = g.m;
    }
    // all kConsumerThreads threads; named barrier 2 fences the previous panel's readers and this copy
    __device__ __forceinline__ void load_panel(int col0) const
    {
        bar_sync(2, kConsumerThreads);
        for (int q = threadIdx.x; q < kTC * c.d; q += kConsumerThreads) {
            const int col = q / c.d, k = q - col * c.d;  // consecutive threads read consecutive doubles of Y
            const int j = min(col0 + col, m - 1);        // columns past the block: finite dummies, masked by the caller
            const double y = __ldg(c.Y + (size_t)j * c.d + k);
            asm volatile("st.shared.f64 [%0], %1;" ::"r"(ysm + (uint32_t)(k * kTC + col) * 8u), "d"(y) : "memory");
        }
        bar_sync(2, kConsumerThreads);
    }
    __device__ __forceinline__ void row(double2 (&mv)[4], int row, int lane) const
    {
        const double* xr = c.X + (size_t)min(row, nloc - 1) * c.d;
        double acc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.0;
        uint32_t yk = ysm + (uint32_t)lane * 16u;
        for (int k = 0; k < c.d; ++k) {
            const double x = __ldg(xr + k);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double2 y = lds_f64x2(yk + (uint32_t)q * 512u);
                const double da = __dsub_rn(x, y.x), db = __dsub_rn(x, y.y);
                acc[2 * q] = __dadd_rn(acc[2 * q], __dmul_rn(da, da));
                acc[2 * q + 1] = __dadd_rn(acc[2 * q + 1], __dmul_rn(db, db));
            }
            yk += kTC * 8u;
        }
        if (c.fast_div) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                mv[q] = make_double2(cloud_div_fast(acc[2 * q], c.cmax, c.inv_cmax), cloud_div_fast(acc[2 * q + 1], c.cmax, c.inv_cmax));
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) mv[q] = make_double2(__ddiv_rn(acc[2 * q], c.cmax), __ddiv_rn(acc[2 * q + 1], c.cmax));
        }
    }
};

// single cost entry for the low-volume kernels (dense plan, pattern gathers)
struct CostViewDev {
    const double* M;
    long ld;
    CloudGeom cloud;
};
__device__ __forceinline__ double cost_at(const CostViewDev& c, int i, int j)
{
    return c.M ? c.M[(size_t)i * c.ld + j] : cloud_cost(c.cloud, i, j);
}

// Consumer-side view of the ring, all in 32-bit shared-window addresses so the per-tile
// bookkeeping is a handful of integer instructions (no generic->shared conversions in the loop).
struct RingCursor {
    uint32_t full0, empty0;  // &full[0], &empty[0]
    uint32_t row0;           // this warp's row of stage 0, this lane's first double2
    uint32_t full, empty, row;  // the same for the current stage
    int s;
    uint32_t ph;
    __device__ __forceinline__ void init(const SweepSmem& sm, int warp, int lane)
    {
        full0 = smem_u32(sm.full);
        empty0 = smem_u32(sm.empty);
        row0 = smem_u32(sm.tiles) + (uint32_t)warp * (kTC * 8) + (uint32_t)lane * 16u;
        full = full0;
        empty = empty0;
        row = row0;
        s = 0;
        ph = 0;
    }
    // block until the current stage has landed
    __device__ __forceinline__ void wait() const { mbar_wait_s(full, ph); }
    // this lane's 8 entries of its warp's row: columns 2 lane + 64 q + {0, 1}
    __device__ __forceinline__ void load_row(double (&mv)[kEPL]) const
    {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double2 v = lds_f64x2(row + (uint32_t)q * 512u);
            mv[2 * q] = v.x;
            mv[2 * q + 1] = v.y;
        }
    }
    // hand the stage back to the producer and step to the next one
    __device__ __forceinline__ void release(int lane)
    {
        __syncwarp();
        if (lane == 0) mbar_arrive_s(empty);
        if (++s == kStages) {
            s = 0;
            ph ^= 1u;
            full = full0;
            empty = empty0;
            row = row0;
        } else {
            full += 8u;
            empty += 8u;
            row += (uint32_t)kTileBytes;
        }
    }
};

// host: views of the resident problem for the kernels
inline CloudGeom cloud_geom(const regot_ctx* ctx)
{
    CloudGeom c;
    c.X = ctx->prob.X_own.p;
    c.Y = ctx->prob.Y_own.p;
    c.d = ctx->prob.cloud_d;
    c.cmax = ctx->prob.cloud_max;
    c.inv_cmax = 1.0 / ctx->prob.cloud_max;
    c.fast_div = ctx->prob.cloud_fast_div ? 1 : 0;
    return c;
}
inline CostViewDev cost_view_dev(const regot_ctx* ctx)
{
    CostViewDev v;
    v.M = ctx->prob.on_the_fly ? nullptr : ctx->prob.M;
    v.ld = (long)ctx->prob.ld;
    v.cloud = cloud_geom(ctx);
    return v;
}

}  // namespace rg
