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
// point-cloud problems whose cost is formed on the fly: the TMA producer warp is replaced by
// kCloudWarps warps that compute the tiles into the same ring
constexpr int kCloudWarps = 4;
constexpr int kCloudSweepThreads = kConsumerThreads + kCloudWarps * kWarp;

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
    double cmax;  // maximum of the un-normalised cost over the GLOBAL matrix
};
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
    return __ddiv_rn(cloud_sqdist(c.X + (size_t)i * c.d, c.Y + (size_t)j * c.d, c.d), c.cmax);
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

// Body of the warps above the consumers: stream (kCloud == false, one TMA warp) or compute
// (kCloud == true, kCloudWarps warps) this CTA's tiles into the ring.
template <bool kCloud>
__device__ __forceinline__ void sweep_feed(const CUtensorMap* tmap, const SweepGeom& g, double* tiles, uint64_t* full,
                                           uint64_t* empty, int warp, int lane);

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

// Producer warps of the on-the-fly kernels: thread p of the kCloudWarps * 32 producers owns columns
// 2p, 2p + 1 of every 256-wide tile and computes them for the tile's 16 rows (32 running sums, the
// coordinate loop outermost so any d works), then stores them with one conflict-free 16-byte store
// per row.  Rows / columns outside the block get finite dummies; consumers mask them like TMA's
// zero fill.
__device__ __forceinline__ void cloud_producer(const SweepGeom& g, double* tiles, uint64_t* full, uint64_t* empty, int pw,
                                               int lane)
{
    long t0, t1;
    sweep_range(g, t0, t1);
    const int p = pw * kWarp + lane;
    const CloudGeom& c = g.cloud;
    int s = 0;
    uint32_t ph = 0;
    for (long t = t0; t < t1; ++t) {
        const int panel = (int)(t / g.n_row_tiles), rt = (int)(t % g.n_row_tiles);
        const int j0 = min(panel * kTC + 2 * p, g.m - 1), j1 = min(panel * kTC + 2 * p + 1, g.m - 1);
        const double* y0 = c.Y + (size_t)j0 * c.d;
        const double* y1 = c.Y + (size_t)j1 * c.d;
        const int row0 = rt * kTR;
        double acc0[kTR], acc1[kTR];
#pragma unroll
        for (int r = 0; r < kTR; ++r) acc0[r] = acc1[r] = 0.0;
        for (int k = 0; k < c.d; ++k) {
            const double ya = __ldg(y0 + k), yb = __ldg(y1 + k);
#pragma unroll
            for (int r = 0; r < kTR; ++r) {
                const double x = __ldg(c.X + (size_t)min(row0 + r, g.nloc - 1) * c.d + k);
                const double da = __dsub_rn(x, ya), db = __dsub_rn(x, yb);
                acc0[r] = __dadd_rn(acc0[r], __dmul_rn(da, da));
                acc1[r] = __dadd_rn(acc1[r], __dmul_rn(db, db));
            }
        }
        mbar_wait(&empty[s], ph ^ 1u);
        double* dst = tiles + (size_t)s * kTileElems + 2 * p;
#pragma unroll
        for (int r = 0; r < kTR; ++r)
            *reinterpret_cast<double2*>(dst + r * kTC) = make_double2(__ddiv_rn(acc0[r], c.cmax), __ddiv_rn(acc1[r], c.cmax));
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
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
// full_count: arrivals that complete a stage (1 for the TMA producer, kCloudWarps for on-the-fly tiles)
__device__ __forceinline__ SweepSmem sweep_prologue(unsigned char* smem, const CUtensorMap* tmap,
                                                    const double* __restrict__ exp_table, int full_count = 1)
{
    SweepSmem s;
    s.tiles = reinterpret_cast<double*>(smem + kSmemTiles);
    s.table = reinterpret_cast<double*>(smem + kSmemTable);
    s.scratch = reinterpret_cast<double*>(smem + kSmemScratch);
    s.full = reinterpret_cast<uint64_t*>(smem + kSmemBars);
    s.empty = s.full + kStages;
    if (threadIdx.x == 0) {
        if (full_count == 1) tma_prefetch_desc(tmap);
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&s.full[i], full_count);
            mbar_init(&s.empty[i], kTR);
        }
        fence_mbar_init();
    }
    exp_table_fill(s.table, exp_table, threadIdx.x, blockDim.x);
    __syncthreads();
    return s;
}

template <bool kCloud>
__device__ __forceinline__ void sweep_feed(const CUtensorMap* tmap, const SweepGeom& g, double* tiles, uint64_t* full,
                                           uint64_t* empty, int warp, int lane)
{
    if (kCloud) cloud_producer(g, tiles, full, empty, warp - kTR, lane);
    else sweep_producer(tmap, g, tiles, full, empty);
}
template <bool kCloud>
constexpr int sweep_threads() { return kCloud ? kCloudSweepThreads : kSweepThreads; }

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
