// k2_topk.cu -- K2: device sparsification.
//
// Replaces regot::plan + select_topk (dual.h:83-94, sparsity.h:44-91) and the
// structural half of assemble (sparsity.h:226-289).  The dense plan is never
// materialised: three TMA sweeps over the cost block recompute T on the fly
//   1. HIST   4096-bin histogram of the top 12 bits of an order-preserving key (skipped when the previous refresh's
//             threshold bin, tried first by the COUNT sweep with its own histogram of the candidates, still holds)
//   2. COUNT  per (row, panel) count of candidates (coarse bin >= b* or Omega*)
//   3. WRITE  warp-ballot compaction of the candidates in row-major order
// then the exact k-th largest key K* inside bin b* is found by a 4 x 13-bit
// radix refinement on the (small) candidate list, ties at K* are taken in
// row-major order (the reference's comparator: value desc, index asc,
// sparsity.h:69-71), and the survivors united with Omega* (first row / first
// column) are compacted into CSR.  Every step is order-deterministic, so the
// pattern is bit-exact given identical T.
#include "ctx.hpp"
#include "sparse.hpp"
#include "sweep.cuh"

#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstring>

namespace rg {

constexpr int kCoarseBins = 4096;
constexpr int kFineBits = 13;
constexpr int kFineBins = 1 << kFineBits;

// order-preserving map double -> uint64 (-0 canonicalised to +0 so that equal
// values get equal keys, like the reference's `a.value == b.value`)
__device__ __forceinline__ unsigned long long order_key(double v)
{
    v = v + 0.0;
    const long long b = __double_as_longlong(v);
    return b < 0 ? ~(unsigned long long)b : ((unsigned long long)b | 0x8000000000000000ULL);
}

enum { kPassHist = 0, kPassCount = 1, kPassWrite = 2 };

struct TopkParams {
    SweepGeom g;
    const double* alpha;
    const double* beta;
    ExpScale E;
    const double* exp_table;
    int row_begin;  // global index of local row 0 (Omega* first row lives on rank 0)
    int mm1;        // m - 1: the last column is never a candidate
    unsigned bstar; // coarse threshold bin
    int count_hist; // COUNT pass: also histogram the entries whose bin is >= bstar (bstar is a guess)
    unsigned long long* hist;  // kCoarseBins
    const int* candptr;        // nloc + 1
    const int* pre;            // n_panels x nloc
    int* cnt;                  // n_panels x nloc
    unsigned long long* cand_key;
    int* cand_col;
    int* cand_row;
    double* cand_m;
};

template <int kPass, int kSrc, bool kCloud>
__global__ void __launch_bounds__(sweep_threads<kCloud>(), 1)
k_topk_sweep(const __grid_constant__ CUtensorMap tmap, const TopkParams p)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const SweepSmem sm = sweep_prologue(smem, &tmap, p.exp_table, !kCloud);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned int* shist = reinterpret_cast<unsigned int*>(sm.scratch);
    const bool hist_here = kPass == kPassHist || (kPass == kPassCount && p.count_hist);
    if (hist_here) {
        for (int q = threadIdx.x; q < kCoarseBins; q += blockDim.x) shist[q] = 0u;
        __syncthreads();
    }
    if (!kCloud && warp == kTR) {
        sweep_producer(&tmap, p.g, sm.tiles, sm.full, sm.empty);
        return;
    }
    CloudRows rows;
    if (kCloud) rows.init(p.g, sm.tiles);
    long t0, t1;
    sweep_range(p.g, t0, t1);
    const uint32_t tbl_lane = smem_u32(sm.table) + (uint32_t)(lane & 15) * 8u;
    const double2* tile_row = reinterpret_cast<const double2*>(sm.tiles + warp * kTC);
    const ExpScale E = p.E;
    const int nloc = p.g.nloc, nrt = p.g.n_row_tiles, mm1 = p.mm1;
    int s = 0;
    uint32_t ph = 0;
    long left = t1 - t0;
    int panel = left > 0 ? (int)(t0 / nrt) : 0;
    int rt = left > 0 ? (int)(t0 - (long)panel * nrt) : 0;
    const unsigned lt_mask = (1u << lane) - 1u;

    while (left > 0) {
        const int seg_tiles = (int)min((long)(nrt - rt), left);
        const int col0 = panel * kTC;
        double bj[kEPL];
        unsigned cmask = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int c = col0 + 64 * q + 2 * lane + e;
                const bool ok = c < mm1;
                bj[2 * q + e] = (kSrc == kFromDual && ok) ? __ldg(p.beta + c) : 0.0;
                cmask |= (ok ? 1u : 0u) << (2 * q + e);
            }
        }
        if (kCloud) rows.load_panel(col0);
        for (int it = 0; it < seg_tiles; ++it) {
            const int row = rt * kTR + warp;
            if (!kCloud) mbar_wait(&sm.full[s], ph);
            if (row < nloc) {
                double2 mv[4];
                if (kCloud) {
                    rows.row(mv, row, lane);
                } else {
                    const double2* trow = tile_row + (size_t)s * (kTileElems / 2);
#pragma unroll
                    for (int q = 0; q < 4; ++q) mv[q] = trow[q * 32 + lane];
                }
                double T[kEPL], cost[kEPL];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    cost[2 * q] = mv[q].x;
                    cost[2 * q + 1] = mv[q].y;
                }
                if (kSrc == kFromDual) {
                    const double ai = __ldg(p.alpha + row);
                    double d[kEPL];
#pragma unroll
                    for (int k = 0; k < kEPL; ++k) d[k] = (ai + bj[k]) - cost[k];
                    plan_entries_dev<kEPL>(d, E, tbl_lane, T);  // identical arithmetic to K1 / k_plan
                } else {
#pragma unroll
                    for (int k = 0; k < kEPL; ++k) T[k] = cost[k];
                }
                unsigned long long key[kEPL];
#pragma unroll
                for (int k = 0; k < kEPL; ++k) key[k] = order_key(T[k]);

                if (kPass == kPassHist) {
#pragma unroll
                    for (int k = 0; k < kEPL; ++k) {
                        const bool ok = (cmask >> k) & 1u;
                        const unsigned bin = (unsigned)(key[k] >> 52);
                        // warp-uniform bins (flat regions, clamped entries) cost one atomic, not 32
                        const unsigned b0 = __shfl_sync(0xffffffffu, bin, 0);
                        const unsigned okm = __ballot_sync(0xffffffffu, ok);
                        if (__all_sync(0xffffffffu, bin == b0 || !ok)) {
                            if (lane == 0 && okm) atomicAdd(&shist[b0], (unsigned)__popc(okm));
                        } else if (ok) {
                            atomicAdd(&shist[bin], 1u);
                        }
                    }
                } else {
                    const bool first_row = (p.row_begin + row) == 0;
                    bool sel[kEPL];
#pragma unroll
                    for (int k = 0; k < kEPL; ++k) {
                        const int c = col0 + 64 * (k >> 1) + 2 * lane + (k & 1);
                        sel[k] = ((cmask >> k) & 1u) && ((unsigned)(key[k] >> 52) >= p.bstar || first_row || c == 0);
                    }
                    if (kPass == kPassCount) {
                        if (p.count_hist) {  // by value only (Omega* is no part of the ranking): a few percent of the entries
#pragma unroll
                            for (int k = 0; k < kEPL; ++k) {
                                const unsigned bin = (unsigned)(key[k] >> 52);
                                if (((cmask >> k) & 1u) && bin >= p.bstar) atomicAdd(&shist[bin], 1u);
                            }
                        }
                        int tot = 0;
#pragma unroll
                        for (int k = 0; k < kEPL; ++k) tot += __popc(__ballot_sync(0xffffffffu, sel[k]));
                        if (lane == 0) p.cnt[(size_t)panel * nloc + row] = tot;
                    } else {
                        int base = p.candptr[row] + p.pre[(size_t)panel * nloc + row];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const unsigned e0 = __ballot_sync(0xffffffffu, sel[2 * q]);
                            const unsigned e1 = __ballot_sync(0xffffffffu, sel[2 * q + 1]);
                            int pos = base + __popc(e0 & lt_mask) + __popc(e1 & lt_mask);
                            const int c = col0 + 64 * q + 2 * lane;
                            if (sel[2 * q]) {
                                p.cand_key[pos] = key[2 * q];
                                p.cand_col[pos] = c;
                                p.cand_row[pos] = row;
                                p.cand_m[pos] = cost[2 * q];
                                ++pos;
                            }
                            if (sel[2 * q + 1]) {
                                p.cand_key[pos] = key[2 * q + 1];
                                p.cand_col[pos] = c + 1;
                                p.cand_row[pos] = row;
                                p.cand_m[pos] = cost[2 * q + 1];
                            }
                            base += __popc(e0) + __popc(e1);
                        }
                    }
                }
            }
            if (!kCloud) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.empty[s]);
                if (++s == kStages) {
                    s = 0;
                    ph ^= 1u;
                }
            }
            ++rt;
            --left;
        }
        if (rt == nrt) {
            rt = 0;
            ++panel;
        }
    }
    if (hist_here) {
        bar_sync(1, kConsumerThreads);
        for (int q = threadIdx.x; q < kCoarseBins; q += kConsumerThreads)
            if (shist[q]) atomicAdd(&p.hist[q], (unsigned long long)shist[q]);
    }
}

// per row: exclusive prefix of the per-panel counts, and the row total
__global__ void k_row_prefix(int nloc, int n_panels, const int* __restrict__ cnt, int* __restrict__ pre,
                             int* __restrict__ rowtot)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += gridDim.x * blockDim.x) {
        int run = 0;
        for (int P = 0; P < n_panels; ++P) {
            pre[(size_t)P * nloc + i] = run;
            run += cnt[(size_t)P * nloc + i];
        }
        rowtot[i] = run;
    }
}

// radix refinement inside coarse bin b*: histogram of one 13-bit digit over the
// candidates whose already-fixed high bits match
__global__ void k_refine_hist(int nc, const unsigned long long* __restrict__ key, unsigned long long fixed_mask,
                              unsigned long long fixed_val, int shift, unsigned long long* __restrict__ hist)
{
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nc; t += gridDim.x * blockDim.x) {
        const unsigned long long k = key[t];
        if ((k & fixed_mask) == fixed_val) atomicAdd(&hist[(k >> shift) & (kFineBins - 1)], 1ULL);
    }
}

// keep = Omega* or key > K*; tie = key == K* (ties are ranked afterwards)
__global__ void k_flag(int nc, const unsigned long long* __restrict__ key, const int* __restrict__ col,
                       const int* __restrict__ row, int row_begin, unsigned long long kstar, int any_topk,
                       int* __restrict__ keep, int* __restrict__ tie)
{
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nc; t += gridDim.x * blockDim.x) {
        const unsigned long long k = key[t];
        const bool star = (row[t] + row_begin == 0) || col[t] == 0;
        keep[t] = (star || (any_topk && k > kstar)) ? 1 : 0;
        tie[t] = (any_topk && k == kstar) ? 1 : 0;
    }
}

__global__ void k_apply_ties(int nc, const int* __restrict__ tie, const int* __restrict__ tie_rank, long tie_offset,
                             long need_eq, int* __restrict__ keep)
{
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nc; t += gridDim.x * blockDim.x)
        if (tie[t] && tie_offset + tie_rank[t] < need_eq) keep[t] = 1;
}

__global__ void k_compact(int nc, const int* __restrict__ keep, const int* __restrict__ pos, const int* __restrict__ col,
                          const int* __restrict__ row, const double* __restrict__ cm, int* __restrict__ ocol,
                          int* __restrict__ orow, double* __restrict__ om, int* __restrict__ rowcnt)
{
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nc; t += gridDim.x * blockDim.x) {
        if (!keep[t]) continue;
        const int q = pos[t];
        ocol[q] = col[t];
        orow[q] = row[t];
        om[q] = cm[t];
        atomicAdd(&rowcnt[row[t]], 1);
    }
}

__global__ void k_count_cols(int nnz, const int* __restrict__ col, int* __restrict__ colcnt)
{
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nnz; t += gridDim.x * blockDim.x) atomicAdd(&colcnt[col[t]], 1);
}
__global__ void k_iota(int n, int* __restrict__ v)
{
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) v[t] = t;
}
// after the stable sort by column: sorted position q holds CSR entry src[q]
// (colsorted[q] = column of sorted position q; the gathered cost travels along so that the CSC copy of the values can be
// computed in place instead of scattered from the CSR copy)
__global__ void k_build_csc(int nnz, const int* __restrict__ src, const int* __restrict__ row, const int* __restrict__ colsorted,
                            const double* __restrict__ mval, int* __restrict__ cscrow, int* __restrict__ csccol,
                            double* __restrict__ cscmval)
{
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nnz; q += gridDim.x * blockDim.x) {
        const int t = src[q];
        cscrow[q] = row[t];
        csccol[q] = colsorted[q];
        cscmval[q] = mval[t];
    }
}
__global__ void k_gather_cost(int nnz, const int* __restrict__ row, const int* __restrict__ col, const CostViewDev cost,
                              double* __restrict__ mval)
{
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nnz; t += gridDim.x * blockDim.x)
        mval[t] = cost_at(cost, row[t], col[t]);
}

// ---- host side ----------------------------------------------------------------------------------
namespace {
struct RefreshTimer {  // experiments: REGOT_B200_REFRESH_TIMING=1 prints the host wall time of each section
    bool on;
    cudaStream_t st;
    std::chrono::steady_clock::time_point t0;
    std::string line;
    RefreshTimer(cudaStream_t s) : on(std::getenv("REGOT_B200_REFRESH_TIMING") != nullptr), st(s), t0(std::chrono::steady_clock::now()) {}
    void tick(const char* name)
    {
        if (!on) return;
        cudaStreamSynchronize(st);
        const auto t1 = std::chrono::steady_clock::now();
        line += std::string(name) + " " + std::to_string((int)std::chrono::duration<double, std::micro>(t1 - t0).count()) + " us | ";
        t0 = t1;
    }
    ~RefreshTimer()
    {
        if (on) std::fprintf(stderr, "refresh: %s\n", line.c_str());
    }
};
}  // namespace

static int lin_grid(const regot_ctx* ctx, long work)
{
    return (int)std::max<long>(1, std::min<long>((work + 255) / 256, 8L * ctx->sm_count));
}

// out[0..n] = exclusive prefix sums of in[0..n) (out has n + 1 entries; in[n] is ignored/zeroed)
static void exclusive_scan(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, int* in_np1, int* out_np1, long n)
{
    RG_CUDA(cudaMemsetAsync(in_np1 + n, 0, sizeof(int), st));
    size_t bytes = 0;
    RG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in_np1, out_np1, (int)(n + 1), st));
    ws.cub_tmp.ensure(bytes);
    RG_CUDA(cub::DeviceScan::ExclusiveSum(ws.cub_tmp.p, bytes, in_np1, out_np1, (int)(n + 1), st));
    ctx->launches += 2;
}

static int read_int(cudaStream_t st, SparseWS& ws, const int* dev)
{
    if (!ws.h_small) RG_CUDA(cudaMallocHost((void**)&ws.h_small, 64 * sizeof(int)));
    RG_CUDA(cudaMemcpyAsync(ws.h_small, dev, sizeof(int), cudaMemcpyDeviceToHost, st));
    RG_CUDA(cudaStreamSynchronize(st));
    return ws.h_small[0];
}

void allreduce_sum_u64(regot_ctx* ctx, ncclComm* comm, unsigned long long* buf, size_t count, cudaStream_t st);

static void fetch_hist(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, size_t bins)
{
    if (!ws.h_hist) RG_CUDA(cudaMallocHost((void**)&ws.h_hist, sizeof(unsigned long long) * kFineBins));
    if (ctx->sharded) allreduce_sum_u64(ctx, ctx->comm, ws.hist.p, bins, st);
    RG_CUDA(cudaMemcpyAsync(ws.h_hist, ws.hist.p, sizeof(unsigned long long) * bins, cudaMemcpyDeviceToHost, st));
    RG_CUDA(cudaStreamSynchronize(st));
}

template <int kPass, int kSrc>
static void launch_sweep(regot_ctx* ctx, cudaStream_t st, const TopkParams& p)
{
    ProfScope prof(ctx, st, 3);
    if (kSrc == kFromDual && ctx->prob.on_the_fly) {
        RG_CUDA(cudaFuncSetAttribute(k_topk_sweep<kPass, kFromDual, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSweepSmem));
        k_topk_sweep<kPass, kFromDual, true><<<ctx->plan.grid, kCloudSweepThreads, kSweepSmem, st>>>(ctx->prob.tmap, p);
    } else {
        RG_CUDA(cudaFuncSetAttribute(k_topk_sweep<kPass, kSrc, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSweepSmem));
        k_topk_sweep<kPass, kSrc, false><<<ctx->plan.grid, kSweepThreads, kSweepSmem, st>>>(ctx->prob.tmap, p);
    }
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
}
template <int kPass>
static void launch_sweep_src(regot_ctx* ctx, cudaStream_t st, TopkSource src, const TopkParams& p)
{
    if (src == kFromDual) launch_sweep<kPass, kFromDual>(ctx, st, p);
    else launch_sweep<kPass, kFromDenseT>(ctx, st, p);
}

void topk_build_pattern(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, TopkSource src, const double* alpha,
                        const double* beta, int64_t k, regot_sparse& S)
{
    const DeviceProblem& pr = ctx->prob;
    if (k < 0) raise(REGOT_E_VALIDATION, "select_topk: k must be >= 0");
    const int nloc = (int)pr.nloc, m = (int)pr.m, mm1 = m - 1;
    S.ctx = ctx;
    S.device = ctx->device;
    S.n = pr.n;
    S.m = pr.m;
    S.nloc = pr.nloc;
    S.row_begin = pr.row_begin;
    S.nnz = 0;
    S.rowptr.ensure((size_t)nloc + 1);
    if (mm1 <= 0) {  // sparsity.h:55-56: empty block
        RG_CUDA(cudaMemsetAsync(S.rowptr.p, 0, sizeof(int) * ((size_t)nloc + 1), st));
        finish_structure(ctx, st, ws, S);
        return;
    }
    const long long total = (long long)pr.n * (long long)mm1;
    const long long take = std::min<long long>(k, total);

    RefreshTimer rt(st);
    TopkParams p;
    std::memset(&p, 0, sizeof(p));
    p.g.nloc = nloc;
    p.g.m = m;
    p.g.n_row_tiles = ctx->plan.n_row_tiles;
    p.g.n_panels = ctx->plan.n_panels;
    p.g.total_tiles = ctx->plan.total_tiles;
    p.g.cta_seg0 = ctx->plan.d_cta_seg0.p;
    p.g.evict_first = ((double)pr.nloc * (double)pr.ld * 8.0 > 48e6) ? 1 : 0;
    p.g.cloud = cloud_geom(ctx);
    p.alpha = alpha;
    p.beta = beta;
    p.E = make_exp_scale(pr.eta);
    p.exp_table = ctx->exp_table.p;
    p.row_begin = (int)pr.row_begin;
    p.mm1 = mm1;

    const size_t np = (size_t)ctx->plan.n_panels * (size_t)nloc;
    ws.hist.ensure(kFineBins);
    ws.cnt.ensure(np);
    ws.pre.ensure(np);
    ws.rowtot.ensure((size_t)nloc + 1);
    ws.candptr.ensure((size_t)nloc + 1);
    p.cnt = ws.cnt.p;
    p.hist = ws.hist.p;
    unsigned bstar = kCoarseBins;  // take == 0: nothing qualifies by value
    long long need = 0;            // how many keys of bin b* belong to the top-k
    unsigned count_bin = kCoarseBins;  // the bin the COUNT and WRITE sweeps select from (<= b*)
    bool counted = false;

    // ---- the previous refresh's threshold bin as a guess: COUNT from it, histogramming the candidates on the way.  A bin is
    // a binade of T; from one refresh to the next the threshold stays in it most of the time (config D: 3041 five times in
    // a row, config C: 3049 for the last 25 refreshes).  The guess is good when the candidates are at least `take`: b* is
    // then read off their histogram (b* > guess just means a few candidates too many); a guess that is too high costs the
    // count sweep it took. ----
    if (take > 0 && src == kFromDual && ctx->topk_guess && ctx->topk_prev_bin >= 0 && ctx->topk_prev_take == take) {
        RG_CUDA(cudaMemsetAsync(ws.hist.p, 0, sizeof(unsigned long long) * kCoarseBins, st));
        p.bstar = (unsigned)ctx->topk_prev_bin;
        p.count_hist = 1;
        launch_sweep_src<kPassCount>(ctx, st, src, p);
        fetch_hist(ctx, st, ws, kCoarseBins);
        int b = -1;
        int64_t above = 0;
        regot_b200_host_pick_bucket((const uint64_t*)ws.h_hist, kCoarseBins, take, &b, &above);
        // a guess far below the threshold is as useless as one above it: the candidates would be a large part of the block
        // (second refresh of config D: the threshold moves up by 111 binades, 1.1e9 candidates for 2.5e7 places)
        long long total = 0;
        for (int q = ctx->topk_prev_bin; q < kCoarseBins; ++q) total += (long long)ws.h_hist[q];
        if (b >= ctx->topk_prev_bin && total <= 2 * take + 1024) {
            bstar = (unsigned)b;
            need = take - above;
            count_bin = (unsigned)ctx->topk_prev_bin;
            counted = true;
        }
        rt.tick(counted ? "count sweep from the previous bin (hit)" : "count sweep from the previous bin (miss)");
    }
    p.count_hist = 0;

    // ---- pass 1: coarse histogram, pick the bin b* that holds the take-th largest key ----
    if (take > 0 && !counted) {
        RG_CUDA(cudaMemsetAsync(ws.hist.p, 0, sizeof(unsigned long long) * kCoarseBins, st));
        launch_sweep_src<kPassHist>(ctx, st, src, p);
        fetch_hist(ctx, st, ws, kCoarseBins);
        int b = -1;
        int64_t above = 0;
        regot_b200_host_pick_bucket((const uint64_t*)ws.h_hist, kCoarseBins, take, &b, &above);
        if (b < 0) raise(REGOT_E_CUDA, "select_topk: histogram does not cover the block (internal error)");
        bstar = (unsigned)b;
        need = take - above;
    }
    if (src == kFromDual) {
        ctx->topk_prev_bin = take > 0 ? (int)bstar : -1;
        ctx->topk_prev_take = take;
    }

    rt.tick("hist sweep + pick");
    // ---- pass 2 + 3: count and write the candidates in row-major order ----
    if (!counted) {
        count_bin = bstar;
        p.bstar = count_bin;
        launch_sweep_src<kPassCount>(ctx, st, src, p);
    }
    p.bstar = count_bin;
    k_row_prefix<<<lin_grid(ctx, nloc), 256, 0, st>>>(nloc, ctx->plan.n_panels, ws.cnt.p, ws.pre.p, ws.rowtot.p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
    exclusive_scan(ctx, st, ws, ws.rowtot.p, ws.candptr.p, nloc);
    const int nc = read_int(st, ws, ws.candptr.p + nloc);
    ws.cand_key.ensure((size_t)nc + 1);
    ws.cand_col.ensure((size_t)nc + 1);
    ws.cand_row.ensure((size_t)nc + 1);
    ws.cand_m.ensure((size_t)nc + 1);
    ws.keep.ensure((size_t)nc + 1);
    ws.tie.ensure((size_t)nc + 1);
    ws.scan_a.ensure((size_t)nc + 1);
    ws.scan_b.ensure((size_t)nc + 1);
    p.candptr = ws.candptr.p;
    p.pre = ws.pre.p;
    p.cand_key = ws.cand_key.p;
    p.cand_col = ws.cand_col.p;
    p.cand_row = ws.cand_row.p;
    p.cand_m = ws.cand_m.p;
    rt.tick("count sweep + scan");
    if (rt.on) rt.line += "bin " + std::to_string(bstar) + " candidates " + std::to_string(nc) + " take " + std::to_string((long long)take) + " | ";
    launch_sweep_src<kPassWrite>(ctx, st, src, p);
    rt.tick("write sweep");

    // ---- exact threshold K* inside bin b*: 4 x 13-bit radix refinement ----
    unsigned long long kstar = 0;
    long long need_eq = 0;
    if (take > 0) {
        unsigned long long fixed_mask = 0xFFFULL << 52, fixed_val = (unsigned long long)bstar << 52;
        long long rem = need;
        for (int shift = 39; shift >= 0; shift -= kFineBits) {
            RG_CUDA(cudaMemsetAsync(ws.hist.p, 0, sizeof(unsigned long long) * kFineBins, st));
            k_refine_hist<<<lin_grid(ctx, nc), 256, 0, st>>>(nc, ws.cand_key.p, fixed_mask, fixed_val, shift, ws.hist.p);
            RG_CUDA(cudaGetLastError());
            ++ctx->launches;
            fetch_hist(ctx, st, ws, kFineBins);
            int d = -1;
            int64_t above = 0;
            regot_b200_host_pick_bucket((const uint64_t*)ws.h_hist, kFineBins, rem, &d, &above);
            if (d < 0) raise(REGOT_E_CUDA, "select_topk: radix refinement lost the threshold (internal error)");
            rem -= above;
            fixed_mask |= (unsigned long long)(kFineBins - 1) << shift;
            fixed_val |= (unsigned long long)d << shift;
        }
        kstar = fixed_val;
        need_eq = rem;  // ties at K* taken in row-major order
    }

    rt.tick("radix refinement");
    // ---- flags, tie ranking, compaction into CSR ----
    k_flag<<<lin_grid(ctx, nc), 256, 0, st>>>(nc, ws.cand_key.p, ws.cand_col.p, ws.cand_row.p, (int)pr.row_begin, kstar,
                                              take > 0 ? 1 : 0, ws.keep.p, ws.tie.p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
    if (take > 0) {
        exclusive_scan(ctx, st, ws, ws.tie.p, ws.scan_a.p, nc);
        long tie_offset = 0;
        if (ctx->sharded) {
            // ties are taken in global row-major order: ranks before this one go first
            ws.hist.ensure(kFineBins);
            RG_CUDA(cudaMemsetAsync(ws.hist.p, 0, sizeof(unsigned long long) * (size_t)ctx->world, st));
            const int mine = read_int(st, ws, ws.scan_a.p + nc);
            const unsigned long long v = (unsigned long long)mine;
            RG_CUDA(cudaMemcpyAsync(ws.hist.p + ctx->rank, &v, sizeof(v), cudaMemcpyHostToDevice, st));
            fetch_hist(ctx, st, ws, (size_t)ctx->world);
            for (int r = 0; r < ctx->rank; ++r) tie_offset += (long)ws.h_hist[r];
        }
        k_apply_ties<<<lin_grid(ctx, nc), 256, 0, st>>>(nc, ws.tie.p, ws.scan_a.p, tie_offset, (long)need_eq, ws.keep.p);
        RG_CUDA(cudaGetLastError());
        ++ctx->launches;
    }
    exclusive_scan(ctx, st, ws, ws.keep.p, ws.scan_b.p, nc);
    const int nnz = read_int(st, ws, ws.scan_b.p + nc);
    S.nnz = nnz;
    S.col.ensure((size_t)nnz + 1);
    S.row.ensure((size_t)nnz + 1);
    S.mval.ensure((size_t)nnz + 1);
    RG_CUDA(cudaMemsetAsync(ws.rowtot.p, 0, sizeof(int) * ((size_t)nloc + 1), st));
    k_compact<<<lin_grid(ctx, nc), 256, 0, st>>>(nc, ws.keep.p, ws.scan_b.p, ws.cand_col.p, ws.cand_row.p, ws.cand_m.p,
                                                 S.col.p, S.row.p, S.mval.p, ws.rowtot.p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
    exclusive_scan(ctx, st, ws, ws.rowtot.p, S.rowptr.p, nloc);
    rt.tick("flags + compaction");
    finish_structure(ctx, st, ws, S);
    rt.tick("finish_structure (CSC, line lists, PCG schedule)");
}

void pattern_from_coords(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, const int32_t* coords, int64_t ncoords,
                         regot_sparse& S)
{
    const DeviceProblem& pr = ctx->prob;
    const int nloc = (int)pr.nloc, mm1 = (int)pr.m - 1;
    S.ctx = ctx;
    S.device = ctx->device;
    S.n = pr.n;
    S.m = pr.m;
    S.nloc = pr.nloc;
    S.row_begin = pr.row_begin;
    // keep this rank's rows; validate order, range and Omega* (sparsity.h:19-40, 226-243)
    std::vector<int> rows, cols, rowptr((size_t)nloc + 1, 0);
    long prev_i = -1, prev_j = -1;
    std::vector<char> row0((size_t)std::max(mm1, 0), 0), col0((size_t)pr.n, 0);
    for (int64_t t = 0; t < ncoords; ++t) {
        const long i = coords[2 * t], j = coords[2 * t + 1];
        if (i < 0 || i >= pr.n || j < 0 || j >= mm1) raise(REGOT_E_VALIDATION, "assemble: pattern/problem shape mismatch");
        if (i < prev_i || (i == prev_i && j <= prev_j))
            raise(REGOT_E_VALIDATION, "assemble: pattern coordinates must be sorted and unique");
        prev_i = i;
        prev_j = j;
        if (i == 0) row0[(size_t)j] = 1;
        if (j == 0) col0[(size_t)i] = 1;
        if (i >= pr.row_begin && i < pr.row_begin + nloc) {
            rows.push_back((int)(i - pr.row_begin));
            cols.push_back((int)j);
            ++rowptr[(size_t)(i - pr.row_begin) + 1];
        }
    }
    for (char c : row0)
        if (!c) raise(REGOT_E_VALIDATION, "assemble: pattern must contain the first row of the block");
    for (char c : col0)
        if (!c) raise(REGOT_E_VALIDATION, "assemble: pattern must contain the first column of the block");
    for (int i = 0; i < nloc; ++i) rowptr[(size_t)i + 1] += rowptr[(size_t)i];
    const int nnz = (int)rows.size();
    S.nnz = nnz;
    S.rowptr.ensure((size_t)nloc + 1);
    S.col.ensure((size_t)nnz + 1);
    S.row.ensure((size_t)nnz + 1);
    S.mval.ensure((size_t)nnz + 1);
    RG_CUDA(cudaMemcpyAsync(S.rowptr.p, rowptr.data(), sizeof(int) * rowptr.size(), cudaMemcpyHostToDevice, st));
    if (nnz) {
        RG_CUDA(cudaMemcpyAsync(S.row.p, rows.data(), sizeof(int) * (size_t)nnz, cudaMemcpyHostToDevice, st));
        RG_CUDA(cudaMemcpyAsync(S.col.p, cols.data(), sizeof(int) * (size_t)nnz, cudaMemcpyHostToDevice, st));
        k_gather_cost<<<lin_grid(ctx, nnz), 256, 0, st>>>(nnz, S.row.p, S.col.p, cost_view_dev(ctx), S.mval.p);
        RG_CUDA(cudaGetLastError());
        ++ctx->launches;
    }
    RG_CUDA(cudaStreamSynchronize(st));  // host vectors go out of scope
    finish_structure(ctx, st, ws, S);
}

void finish_structure(regot_ctx* ctx, cudaStream_t st, SparseWS& ws, regot_sparse& S)
{
    const int nloc = (int)S.nloc, mm1 = (int)S.m - 1, nnz = (int)S.nnz;
    ++S.structure_stamp;
    S.val.ensure((size_t)nnz + 1);
    S.cscval.ensure((size_t)nnz + 1);
    S.cscrow.ensure((size_t)nnz + 1);
    S.cscptr.ensure((size_t)std::max(mm1, 0) + 2);
    S.dA.ensure((size_t)nloc);
    S.dB.ensure((size_t)std::max(mm1, 1));
    RG_CUDA(cudaMemsetAsync(S.cscptr.p, 0, sizeof(int) * ((size_t)std::max(mm1, 0) + 2), st));
    if (nnz > 0) {
        // column counts -> cscptr; stable radix sort of (col, csr index) gives rows ascending per column
        ws.scan_a.ensure((size_t)std::max(mm1, 0) + 2);
        RG_CUDA(cudaMemsetAsync(ws.scan_a.p, 0, sizeof(int) * ((size_t)mm1 + 2), st));
        k_count_cols<<<lin_grid(ctx, nnz), 256, 0, st>>>(nnz, S.col.p, ws.scan_a.p);
        RG_CUDA(cudaGetLastError());
        ++ctx->launches;
        exclusive_scan(ctx, st, ws, ws.scan_a.p, S.cscptr.p, mm1);
        ws.sort_k1.ensure((size_t)nnz);
        ws.sort_v0.ensure((size_t)nnz);
        ws.sort_v1.ensure((size_t)nnz);
        k_iota<<<lin_grid(ctx, nnz), 256, 0, st>>>(nnz, ws.sort_v0.p);
        RG_CUDA(cudaGetLastError());
        int bits = 1;
        while ((1L << bits) < mm1) ++bits;
        size_t bytes = 0;
        RG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, S.col.p, ws.sort_k1.p, ws.sort_v0.p, ws.sort_v1.p, nnz, 0,
                                                bits, st));
        ws.cub_tmp.ensure(bytes);
        RG_CUDA(cub::DeviceRadixSort::SortPairs(ws.cub_tmp.p, bytes, S.col.p, ws.sort_k1.p, ws.sort_v0.p, ws.sort_v1.p, nnz,
                                                0, bits, st));
        S.csccol.ensure((size_t)nnz + 1);
        S.cscmval.ensure((size_t)nnz + 1);
        k_build_csc<<<lin_grid(ctx, nnz), 256, 0, st>>>(nnz, ws.sort_v1.p, S.row.p, ws.sort_k1.p, S.mval.p, S.cscrow.p, S.csccol.p, S.cscmval.p);
        RG_CUDA(cudaGetLastError());
        ctx->launches += 4;
        // the block plan of the resident PCG kernel is built on the device behind the CSC (sort_v1[t] = CSR position of
        // CSC entry t); its 4-int summary travels with the pointer arrays below
        build_pcg_blocks_plan(ctx, st, ws, S, ws.sort_v1.p);
    } else {
        S.blocks.fits = S.blocks.pending = false;
    }
    // Lines (rows of B, columns of B) longer than a threshold -- always row 0 and column 0 of Omega*
    // at scale -- are cut into chunks of kChunkLen entries that different warps process; the last warp
    // to finish a line sums its chunk partials in chunk order (deterministic).  The others are binned
    // by length.  All of this is host work on the two pointer arrays: pinned staging both ways, no
    // allocation, one synchronisation.
    const size_t np = (size_t)nloc + 1 + (size_t)std::max(mm1, 0) + 1;
    ws.h_ptrs.ensure(np);
    int* rp = ws.h_ptrs.p;
    int* cp = rp + nloc + 1;
    RG_CUDA(cudaMemcpyAsync(rp, S.rowptr.p, sizeof(int) * ((size_t)nloc + 1), cudaMemcpyDeviceToHost, st));
    RG_CUDA(cudaMemcpyAsync(cp, S.cscptr.p, sizeof(int) * ((size_t)std::max(mm1, 0) + 1), cudaMemcpyDeviceToHost, st));
    if (ws.after_pointer_download) {
        // wait for the pointers only; what the hook enqueues behind them keeps the GPU busy during the host work below
        if (!ws.ev_ptrs) RG_CUDA(cudaEventCreateWithFlags(&ws.ev_ptrs, cudaEventDisableTiming));
        RG_CUDA(cudaEventRecord(ws.ev_ptrs, st));
        auto hook = std::move(ws.after_pointer_download);
        ws.after_pointer_download = nullptr;
        hook();
        RG_CUDA(cudaEventSynchronize(ws.ev_ptrs));
    } else {
        RG_CUDA(cudaStreamSynchronize(st));
    }
    finish_pcg_blocks_plan(ctx, st, ws, S, nnz > 0 ? ws.sort_v1.p : nullptr);
    // The threshold grows with the problem: once a warp of the mat-vec grid has thousands of entries to
    // process anyway, a line of that length is balanced work for ONE warp, and chunking it would only
    // add the cross-warp combine (a fence and an atomic per chunk).  At config B it stays kLongLine.
    const long spmv_warps = 8L * ctx->sm_count * 8;
    const int long_thr = (int)std::max<long>(kLongLine, std::min<long>(4096, (long)nnz / (2 * spmv_warps)));
    // pass 1: sizes (rows first in every list)
    int n_s[2] = {0, 0}, n_m[2] = {0, 0}, n_c[2] = {0, 0}, n_l[2] = {0, 0};
    for (int side = 0; side < 2; ++side) {
        const int* ptr = side == 0 ? rp : cp;
        const int nl = side == 0 ? nloc : mm1;
        for (int l = 0; l < nl; ++l) {
            const int len = ptr[l + 1] - ptr[l];
            if (len <= kShortLine) ++n_s[side];
            else if (len <= long_thr) ++n_m[side];
            else {
                ++n_l[side];
                n_c[side] += (len + kChunkLen - 1) / kChunkLen;
            }
        }
    }
    S.n_lines_s_rows = n_s[0];
    S.n_lines_m_rows = n_m[0];
    S.n_chunks_rows = n_c[0];
    S.n_lines_s = n_s[0] + n_s[1];
    S.n_lines_m = n_m[0] + n_m[1];
    S.n_chunks = n_c[0] + n_c[1];
    S.n_long = n_l[0] + n_l[1];
    // pass 2: fill the staging  [lines_s | lines_m | chunks (4 ints) | longlines (2 ints)]
    const size_t o_s = 0, o_m = o_s + (size_t)S.n_lines_s, o_c = o_m + (size_t)S.n_lines_m, o_l = o_c + 4 * (size_t)S.n_chunks;
    const size_t used = o_l + 2 * (size_t)S.n_long;
    // room for the PCG schedule behind the lists: one item per 1..4 lines / chunk, 2 pointer tables
    const size_t sched_max = (size_t)kPcgItemInts * ((size_t)S.n_lines_s + S.n_lines_m + S.n_chunks + 16) +
                             2 * ((size_t)ctx->sm_count * kPcgWarpsPerCta + 1);
    ws.h_lines.ensure(used + sched_max + 64);
    int* hs = ws.h_lines.p;
    {
        size_t is = o_s, im = o_m, ic = 0, il = 0;  // ic / il count chunks / long lines
        for (int side = 0; side < 2; ++side) {
            const int* ptr = side == 0 ? rp : cp;
            const int nl = side == 0 ? nloc : mm1, base = side == 0 ? 0 : nloc;
            for (int l = 0; l < nl; ++l) {
                const int beg = ptr[l], end = ptr[l + 1], len = end - beg;
                if (len <= kShortLine) hs[is++] = base + l;
                else if (len <= long_thr) hs[im++] = base + l;
                else {
                    hs[o_l + 2 * il] = (int)ic;
                    int cnt = 0;
                    for (int b0 = beg; b0 < end; b0 += kChunkLen, ++cnt, ++ic) {
                        int* c4 = hs + o_c + 4 * ic;
                        c4[0] = base + l;
                        c4[1] = b0;
                        c4[2] = std::min(end, b0 + kChunkLen);
                        c4[3] = (int)il;
                    }
                    hs[o_l + 2 * il + 1] = cnt;
                    ++il;
                }
            }
        }
    }
    S.lines_s.ensure((size_t)S.n_lines_s + 1);
    S.lines_m.ensure((size_t)S.n_lines_m + 1);
    S.chunks.ensure(4 * (size_t)S.n_chunks + 4);
    S.longlines.ensure(2 * (size_t)S.n_long + 2);
    S.chunk_part.ensure((size_t)S.n_chunks * 3 + 3);
    S.chunk_cnt.ensure((size_t)S.n_long + 1);
    RG_CUDA(cudaMemsetAsync(S.chunk_cnt.p, 0, sizeof(unsigned int) * ((size_t)S.n_long + 1), st));
    if (S.n_lines_s) RG_CUDA(cudaMemcpyAsync(S.lines_s.p, hs + o_s, sizeof(int) * (size_t)S.n_lines_s, cudaMemcpyHostToDevice, st));
    if (S.n_lines_m) RG_CUDA(cudaMemcpyAsync(S.lines_m.p, hs + o_m, sizeof(int) * (size_t)S.n_lines_m, cudaMemcpyHostToDevice, st));
    if (S.n_chunks) RG_CUDA(cudaMemcpyAsync(S.chunks.p, hs + o_c, sizeof(int) * 4 * (size_t)S.n_chunks, cudaMemcpyHostToDevice, st));
    if (S.n_long) RG_CUDA(cudaMemcpyAsync(S.longlines.p, hs + o_l, sizeof(int) * 2 * (size_t)S.n_long, cudaMemcpyHostToDevice, st));
    // the older persistent kernel (k5_pcg.cu) only where the block-resident one does not take the pattern
    S.pcg.fits = false;
    if (!ctx->sharded && !S.blocks.fits) build_pcg_schedule(ctx, st, S, rp, cp, ws.h_lines, used);
    RG_CUDA(cudaStreamSynchronize(st));  // the staging is free again
}

}  // namespace rg
