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

// dynamic shared memory carve-up (bytes)
constexpr int kSmemTiles = 0;
constexpr int kSmemTable = kSmemTiles + kStages * kTileBytes;
constexpr int kSmemScratch = kSmemTable + kExpTableBytes;        // kTR x kTC doubles
constexpr int kSmemBars = kSmemScratch + kTR * kTC * 8;
constexpr int kSweepSmem = kSmemBars + 2 * kStages * 8 + 64;

struct SweepGeom {
    int nloc, m;
    int n_row_tiles, n_panels;
    long total_tiles;
    const int* cta_seg0;  // grid + 1
    int evict_first;      // stream M through L2 with an evict-first policy
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
__device__ __forceinline__ SweepSmem sweep_prologue(unsigned char* smem, const CUtensorMap* tmap,
                                                    const double* __restrict__ exp_table)
{
    SweepSmem s;
    s.tiles = reinterpret_cast<double*>(smem + kSmemTiles);
    s.table = reinterpret_cast<double*>(smem + kSmemTable);
    s.scratch = reinterpret_cast<double*>(smem + kSmemScratch);
    s.full = reinterpret_cast<uint64_t*>(smem + kSmemBars);
    s.empty = s.full + kStages;
    if (threadIdx.x == 0) {
        tma_prefetch_desc(tmap);
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

}  // namespace rg
