// k7_lse.cu -- K7/K8/K9: log-domain Sinkhorn updates.
//
// Replaces regot::optimal_alpha (sinkhorn.h:44-74), optimal_beta
// (sinkhorn.h:77-101) and the gauge shift of sinkhorn_step (sinkhorn.h:105-115).
// The reference makes two sweeps of M per update (max, then exp-sum); here each
// update is ONE pass: per (row, panel) / (column, segment) a max-shifted
// exp-sum pair (max, sum) is produced and pairs are merged exactly,
//   (M1, s1) + (M2, s2) = (M, s1 e^{M1-M} + s2 e^{M2-M}),  M = max(M1, M2),
// which equals the reference's sum up to rounding.  Like the reference the LSE
// does not clamp its exponents; shifted exponents below -700 contribute less
// than 1e-304 to a sum that is at least 1 and are evaluated at -700.
//
// Algorithmic bytes per Sinkhorn step: 2 * 8 * nloc * m.
#include "ctx.hpp"
#include "sweep.cuh"

#include <algorithm>
#include <cmath>

namespace rg {

struct LseParams {
    SweepGeom g;
    const double* vec;  // row LSE: beta (m); column LSE: alpha (nloc)
    double inv_eta;
    const double* exp_table;
    double* part_sum;  // row: n_panels x nloc ; column: n_segments x kTC
    double* part_max;
    int fast_shift;  // row LSE: shift by the warp's approximate maximum (warp_shift) instead of the exact one
};

__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }

// (default; REGOT_B200_LSE_FAST_SHIFT=0 subtracts the exact maximum like sinkhorn.h:57-68)
// The shift of a log-sum-exp need not be the exact maximum: any value within a few hundred of it keeps every
// exponential in range, and lse = shift + log(sum exp(v - shift)) holds for all of them.  The warp's shift is the
// maximum of the HIGH WORDS of the lanes' maxima (one redux.sync on an order-preserving integer key instead of five
// 64-bit shuffle + compare rounds), i.e. the true maximum with its low 32 bits cleared: within 2^-20 relative of it.
__device__ __forceinline__ double warp_shift(double lane_max)
{
    const int hi = __double2hiint(lane_max);
    int key = hi >= 0 ? hi : (hi ^ 0x7fffffff);  // sign-magnitude -> two's complement order
    key = __reduce_max_sync(0xffffffffu, key);
    return __hiloint2double(key >= 0 ? key : (key ^ 0x7fffffff), 0);
}

// ---- K7: row LSE sweep ---------------------------------------------------------------
// v_ij = (beta_j - M_ij) / eta.  Warp w owns row w of each tile: lane max ->
// warp max (shuffles) -> sum of exp(v - max) -> staged transposing flush.
template <bool kRagged>
__device__ __forceinline__ void row_lse_row(const double2 (&mv)[4], const double (&bj)[kEPL], unsigned cmask,
                                            double inv_eta, uint32_t tbl_lane, bool fast_shift, double& wmax, double& lsum)
{
    double v[kEPL];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        v[2 * q] = (bj[2 * q] - mv[q].x) * inv_eta;
        v[2 * q + 1] = (bj[2 * q + 1] - mv[q].y) * inv_eta;
    }
    if (kRagged) {
#pragma unroll
        for (int k = 0; k < kEPL; ++k) v[k] = (cmask >> k) & 1u ? v[k] : -INFINITY;
    }
    double mx = dmax(dmax(dmax(v[0], v[1]), dmax(v[2], v[3])), dmax(dmax(v[4], v[5]), dmax(v[6], v[7])));
    mx = fast_shift ? warp_shift(mx) : warp_max(mx);
    double sacc[kEPL];
    unsigned amax = 0;
#pragma unroll
    for (int k = 0; k < kEPL; ++k) {
        sacc[k] = v[k] - mx;  // <= |mx| 2^-20, -inf for masked columns
        amax = max(amax, abs_hi(sacc[k]));
    }
    if (amax >= kHi700) {
#pragma unroll
        for (int k = 0; k < kEPL; ++k) sacc[k] = clamp700(sacc[k]);
    }
#pragma unroll
    for (int k = 0; k < kEPL; ++k) {
        sacc[k] = exp_tbl(sacc[k], tbl_lane);
        if (kRagged) sacc[k] = (cmask >> k) & 1u ? sacc[k] : 0.0;
    }
    wmax = mx;
    lsum = ((sacc[0] + sacc[1]) + (sacc[2] + sacc[3])) + ((sacc[4] + sacc[5]) + (sacc[6] + sacc[7]));
}

template <bool kCloud>
__global__ void __launch_bounds__(sweep_threads<kCloud>(), 1)
k_row_lse_sweep(const __grid_constant__ CUtensorMap tmap, const LseParams p)
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
    long t0, t1;
    sweep_range(p.g, t0, t1);
    if (t0 >= t1) return;
    const uint32_t tbl_lane = smem_u32(sm.table) + (uint32_t)(lane & 15) * 8u;
    double* stage = sm.scratch + warp * kTC;
    const double2* tile_row = reinterpret_cast<const double2*>(sm.tiles + warp * kTC);
    const double inv_eta = p.inv_eta;
    const int nloc = p.g.nloc, m = p.g.m, nrt = p.g.n_row_tiles;
    int s = 0;
    uint32_t ph = 0;
    long left = t1 - t0;
    int panel = (int)(t0 / nrt);
    int rt = (int)(t0 - (long)panel * nrt);

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
                const bool ok = c < m;
                bj[2 * q + e] = ok ? __ldg(p.vec + c) : 0.0;
                cmask |= (ok ? 1u : 0u) << (2 * q + e);
            }
        }
        const bool ragged = (col0 + kTC > m);
        if (kCloud) rows.load_panel(col0);
        int done = 0;
        while (done < seg_tiles) {
            const int cnt = min(kRowGroup, seg_tiles - done);
            const int rt0 = rt;
            double my_max = 0.0;  // lane k of the group keeps the warp max of staged row k
            for (int k = 0; k < cnt; ++k) {
                const int row = rt * kTR + warp;
                if (!kCloud) mbar_wait(&sm.full[s], ph);
                double wmax = -INFINITY, lsum = 0.0;
                if (row < nloc) {
                    double2 mv[4];
                    if (kCloud) {
                        rows.row(mv, row, lane);
                    } else {
                        const double2* trow = tile_row + (size_t)s * (kTileElems / 2);
#pragma unroll
                        for (int q = 0; q < 4; ++q) mv[q] = trow[q * 32 + lane];
                    }
                    if (ragged) row_lse_row<true>(mv, bj, cmask, inv_eta, tbl_lane, p.fast_shift != 0, wmax, lsum);
                    else row_lse_row<false>(mv, bj, cmask, inv_eta, tbl_lane, p.fast_shift != 0, wmax, lsum);
                }
                if (!kCloud) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sm.empty[s]);
                    if (++s == kStages) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                stage[k * 32 + lane] = lsum;
                if (lane == 4 * k) my_max = wmax;
                ++rt;
                --left;
            }
            done += cnt;
            __syncwarp();
            {
                const int k = lane >> 2, part = lane & 3;
                const double* src = stage + k * 32 + part * 8;
                double v = ((src[0] + src[1]) + (src[2] + src[3])) + ((src[4] + src[5]) + (src[6] + src[7]));
                v += shfl_xor_d(v, 1);
                v += shfl_xor_d(v, 2);
                const int row = (rt0 + k) * kTR + warp;
                if (part == 0 && k < cnt && row < nloc) {
                    p.part_sum[(size_t)panel * nloc + row] = v;
                    p.part_max[(size_t)panel * nloc + row] = my_max;
                }
            }
            __syncwarp();
        }
        if (rt == nrt) {
            rt = 0;
            ++panel;
        }
    }
}

// alpha_i = eta (log a_i - (M + log S)) with (M, S) merged over panels (sinkhorn.h:70-72)
__global__ void k_row_lse_fin(int nloc, int n_panels, double eta, const double* __restrict__ part_sum,
                              const double* __restrict__ part_max, const double* __restrict__ a,
                              double* __restrict__ alpha_out)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += gridDim.x * blockDim.x) {
        double M = -INFINITY;
        for (int P0 = 0; P0 < n_panels; P0 += 8) {  // 8 loads in flight
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = (P0 + u < n_panels) ? part_max[(size_t)(P0 + u) * nloc + i] : -INFINITY;
#pragma unroll
            for (int u = 0; u < 8; ++u) M = dmax(M, v[u]);
        }
        double S = 0.0;
        for (int P0 = 0; P0 < n_panels; P0 += 8) {  // panel order (fixed)
            double ps[8], pm[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const bool ok = P0 + u < n_panels;
                ps[u] = ok ? part_sum[(size_t)(P0 + u) * nloc + i] : 0.0;
                pm[u] = ok ? part_max[(size_t)(P0 + u) * nloc + i] : M;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (P0 + u < n_panels) S += ps[u] * exp(pm[u] - M);
        }
        alpha_out[i] = eta * (log(a[i]) - (M + log(S)));
    }
}

// ---- K8: column LSE sweep --------------------------------------------------------------
// v_ij = (alpha_i - M_ij) / eta.  Each lane keeps an online (max, sum) pair for
// its 8 columns across the rows of a segment: one exp per element,
//   d = v - max;  d > 0: sum = sum e^{-d} + 1, max = v;  else: sum += e^{d}.
template <bool kCloud>
__global__ void __launch_bounds__(sweep_threads<kCloud>(), 1)
k_col_lse_sweep(const __grid_constant__ CUtensorMap tmap, const LseParams p)
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
    long t0, t1;
    sweep_range(p.g, t0, t1);
    if (t0 >= t1) return;
    const uint32_t tbl_lane = smem_u32(sm.table) + (uint32_t)(lane & 15) * 8u;
    double* stage = sm.scratch + warp * kTC;
    const double2* tile_row = reinterpret_cast<const double2*>(sm.tiles + warp * kTC);
    const double inv_eta = p.inv_eta;
    const int nloc = p.g.nloc, nrt = p.g.n_row_tiles;
    int seg = p.g.cta_seg0[blockIdx.x];
    int s = 0;
    uint32_t ph = 0;
    long left = t1 - t0;
    int panel = (int)(t0 / nrt);
    int rt = (int)(t0 - (long)panel * nrt);
    double ai_next = (rt * kTR + warp < nloc) ? __ldg(p.vec + rt * kTR + warp) : 0.0;

    while (left > 0) {
        const int seg_tiles = (int)min((long)(nrt - rt), left);
        if (kCloud) rows.load_panel(panel * kTC);
        double cmax[kEPL], csum[kEPL];
#pragma unroll
        for (int k = 0; k < kEPL; ++k) {
            cmax[k] = -INFINITY;
            csum[k] = 0.0;
        }
        for (int it = 0; it < seg_tiles; ++it) {
            const int row = rt * kTR + warp;
            const double ai = ai_next;
            {
                int nrow = row + kTR;
                if (rt + 1 == nrt) nrow = warp;
                ai_next = (nrow < nloc && left > 1) ? __ldg(p.vec + nrow) : 0.0;
            }
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
                double v[kEPL], e[kEPL];
                unsigned amax = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    v[2 * q] = (ai - mv[q].x) * inv_eta;
                    v[2 * q + 1] = (ai - mv[q].y) * inv_eta;
                }
#pragma unroll
                for (int k = 0; k < kEPL; ++k) {
                    const double d = v[k] - cmax[k];
                    // -|d|: set the sign bit
                    e[k] = __hiloint2double(__double2hiint(d) | (int)0x80000000, __double2loint(d));
                    amax = max(amax, abs_hi(d));
                }
                if (amax >= kHi700) {
#pragma unroll
                    for (int k = 0; k < kEPL; ++k) e[k] = clamp700(e[k]);
                }
#pragma unroll
                for (int k = 0; k < kEPL; ++k) {
                    const double ex = exp_tbl(e[k], tbl_lane);
                    const bool up = v[k] > cmax[k];
                    csum[k] = __fma_rn(csum[k], up ? ex : 1.0, up ? 1.0 : ex);
                    cmax[k] = up ? v[k] : cmax[k];
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
        // ---- merge the kTR warps' pairs for this segment through shared memory ----
#pragma unroll
        for (int q = 0; q < 4; ++q)
            reinterpret_cast<double2*>(stage)[q * 32 + lane] = make_double2(cmax[2 * q], cmax[2 * q + 1]);
        bar_sync(1, kConsumerThreads);
        double gmax = -INFINITY;
        if (threadIdx.x < kTC) {
#pragma unroll
            for (int w = 0; w < kTR; ++w) gmax = dmax(gmax, sm.scratch[w * kTC + threadIdx.x]);
        }
        bar_sync(1, kConsumerThreads);
        if (threadIdx.x < kTC) sm.scratch[threadIdx.x] = gmax;  // row 0 now holds the column maxima
        bar_sync(1, kConsumerThreads);
        double scale[kEPL];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double2 g2 = reinterpret_cast<const double2*>(sm.scratch)[q * 32 + lane];
            // a warp that saw no row keeps (-inf, 0): contributes 0
            scale[2 * q] = (cmax[2 * q] == -INFINITY) ? 0.0 : exp(cmax[2 * q] - g2.x);
            scale[2 * q + 1] = (cmax[2 * q + 1] == -INFINITY) ? 0.0 : exp(cmax[2 * q + 1] - g2.y);
        }
        bar_sync(1, kConsumerThreads);
#pragma unroll
        for (int q = 0; q < 4; ++q)
            reinterpret_cast<double2*>(stage)[q * 32 + lane] =
                make_double2(csum[2 * q] * scale[2 * q], csum[2 * q + 1] * scale[2 * q + 1]);
        bar_sync(1, kConsumerThreads);
        if (threadIdx.x < kTC) {
            double v = 0.0;
#pragma unroll
            for (int w = 0; w < kTR; ++w) v += sm.scratch[w * kTC + threadIdx.x];
            p.part_sum[(size_t)seg * kTC + threadIdx.x] = v;
            p.part_max[(size_t)seg * kTC + threadIdx.x] = gmax;
        }
        bar_sync(1, kConsumerThreads);
        ++seg;
        if (rt == nrt) {
            rt = 0;
            ++panel;
        }
    }
}

// merge the segments of each panel: local (max, sum) per column
__global__ void k_col_lse_merge(int m, const int* __restrict__ panel_seg0, const double* __restrict__ part_sum,
                                const double* __restrict__ part_max, double* __restrict__ loc_max,
                                double* __restrict__ loc_sum)
{
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
        const int P = j / kTC, off = j - P * kTC;
        const int s0 = panel_seg0[P], s1 = panel_seg0[P + 1];
        double M = -INFINITY;
        for (int sg = s0; sg < s1; ++sg) M = dmax(M, part_max[(size_t)sg * kTC + off]);
        double S = 0.0;
        for (int sg = s0; sg < s1; ++sg) {
            const double pm = part_max[(size_t)sg * kTC + off];
            if (pm != -INFINITY) S += part_sum[(size_t)sg * kTC + off] * exp(pm - M);
        }
        loc_max[j] = M;
        loc_sum[j] = S;
    }
}

// multi-GPU: after allreduce(MAX) of the maxima, rescale the local sums
__global__ void k_col_lse_rescale(int m, const double* __restrict__ loc_max, const double* __restrict__ glob_max,
                                  double* __restrict__ sum_io)
{
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x)
        sum_io[j] = (loc_max[j] == -INFINITY) ? 0.0 : sum_io[j] * exp(loc_max[j] - glob_max[j]);
}

// beta_j = eta (log b_j - (M + log S)) (sinkhorn.h:98), then the gauge shift of
// sinkhorn_step (sinkhorn.h:110-113): c = beta[m-1]; alpha += c; beta -= c; beta[m-1] = 0.
__global__ void k_col_lse_fin(int nloc, int m, double eta, const double* __restrict__ gmax,
                              const double* __restrict__ gsum, const double* __restrict__ b,
                              double* __restrict__ beta_out, double* __restrict__ alpha_io, int gauge)
{
    const double c = gauge ? eta * (log(b[m - 1]) - (gmax[m - 1] + log(gsum[m - 1]))) : 0.0;
    const int stride = gridDim.x * blockDim.x;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += stride) {
        const double bj = eta * (log(b[j]) - (gmax[j] + log(gsum[j])));
        beta_out[j] = (gauge && j == m - 1) ? 0.0 : bj - c;
    }
    if (gauge)
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += stride) alpha_io[i] += c;
}

// ---- host side ----------------------------------------------------------------------------
static LseParams make_lse_params(regot_ctx* ctx, const double* vec, double* psum, double* pmax)
{
    LseParams p;
    p.g.nloc = (int)ctx->prob.nloc;
    p.g.m = (int)ctx->prob.m;
    p.g.n_row_tiles = ctx->plan.n_row_tiles;
    p.g.n_panels = ctx->plan.n_panels;
    p.g.total_tiles = ctx->plan.total_tiles;
    p.g.cta_seg0 = ctx->plan.d_cta_seg0.p;
    p.g.evict_first = ((double)ctx->prob.nloc * (double)ctx->prob.ld * 8.0 > 48e6) ? 1 : 0;
    p.g.cloud = cloud_geom(ctx);
    p.vec = vec;
    p.inv_eta = 1.0 / ctx->prob.eta;
    p.exp_table = ctx->exp_table.p;
    p.part_sum = psum;
    p.fast_shift = ctx->lse_fast_shift ? 1 : 0;
    p.part_max = pmax;
    return p;
}

static int vec_grid(const regot_ctx* ctx, long work)
{
    return (int)std::max<long>(1, std::min<long>((work + 255) / 256, 4L * ctx->sm_count));
}

void launch_row_lse_sweep_only(regot_ctx* ctx, cudaStream_t st, SweepWS& ws, const double* beta)
{
    static bool attr_set = false;
    if (!attr_set) {
        RG_CUDA(cudaFuncSetAttribute(k_row_lse_sweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSweepSmem));
        RG_CUDA(cudaFuncSetAttribute(k_row_lse_sweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSweepSmem));
        attr_set = true;
    }
    const LseParams p = make_lse_params(ctx, beta, ws.rowpart.p, ws.rowpart2.p);
    ProfScope prof(ctx, st, 1);
    if (ctx->prob.on_the_fly) k_row_lse_sweep<true><<<ctx->plan.grid, kCloudSweepThreads, kSweepSmem, st>>>(ctx->prob.tmap, p);
    else k_row_lse_sweep<false><<<ctx->plan.grid, kSweepThreads, kSweepSmem, st>>>(ctx->prob.tmap, p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
}

void launch_col_lse_sweep_only(regot_ctx* ctx, cudaStream_t st, SweepWS& ws, const double* alpha)
{
    static bool attr_set = false;
    if (!attr_set) {
        RG_CUDA(cudaFuncSetAttribute(k_col_lse_sweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSweepSmem));
        RG_CUDA(cudaFuncSetAttribute(k_col_lse_sweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSweepSmem));
        attr_set = true;
    }
    const LseParams p = make_lse_params(ctx, alpha, ws.colpart.p, ws.colpart2.p);
    ProfScope prof(ctx, st, 2);
    if (ctx->prob.on_the_fly) k_col_lse_sweep<true><<<ctx->plan.grid, kCloudSweepThreads, kSweepSmem, st>>>(ctx->prob.tmap, p);
    else k_col_lse_sweep<false><<<ctx->plan.grid, kSweepThreads, kSweepSmem, st>>>(ctx->prob.tmap, p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
}

// optimal_alpha: alpha_out (nloc) from beta (m).  Rows are local: no collective.
void launch_optimal_alpha(regot_ctx* ctx, cudaStream_t st, SweepWS& ws, const double* beta, double* alpha_out)
{
    const DeviceProblem& pr = ctx->prob;
    launch_row_lse_sweep_only(ctx, st, ws, beta);
    k_row_lse_fin<<<vec_grid(ctx, pr.nloc), 256, 0, st>>>((int)pr.nloc, ctx->plan.n_panels, pr.eta, ws.rowpart.p,
                                                          ws.rowpart2.p, pr.a, alpha_out);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
}

// optimal_beta: beta_out (m) from alpha (nloc); with gauge != 0 also applies the
// gauge shift of sinkhorn_step to (alpha, beta_out).
void launch_optimal_beta(regot_ctx* ctx, cudaStream_t st, SweepWS& ws, ncclComm* comm, double* alpha_io,
                         double* beta_out, int gauge)
{
    const DeviceProblem& pr = ctx->prob;
    const int m = (int)pr.m;
    launch_col_lse_sweep_only(ctx, st, ws, alpha_io);
    // pack2 = [local max (m) | global max (m)], pack = sums
    double* loc_max = ws.pack2.p;
    double* glob_max = ws.pack2.p;
    k_col_lse_merge<<<vec_grid(ctx, m), 256, 0, st>>>(m, ctx->plan.d_panel_seg0.p, ws.colpart.p, ws.colpart2.p, loc_max,
                                                      ws.pack.p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
    if (ctx->sharded) {
        glob_max = ws.pack2.p + (size_t)m + 16;
        RG_CUDA(cudaMemcpyAsync(glob_max, loc_max, sizeof(double) * (size_t)m, cudaMemcpyDeviceToDevice, st));
        allreduce_max(ctx, comm, glob_max, (size_t)m, st);
        k_col_lse_rescale<<<vec_grid(ctx, m), 256, 0, st>>>(m, loc_max, glob_max, ws.pack.p);
        RG_CUDA(cudaGetLastError());
        ++ctx->launches;
        allreduce_sum(ctx, comm, ws.pack.p, (size_t)m, st);
    }
    k_col_lse_fin<<<vec_grid(ctx, std::max<long>(pr.nloc, m)), 256, 0, st>>>((int)pr.nloc, m, pr.eta, glob_max, ws.pack.p,
                                                                            pr.b, beta_out, alpha_io, gauge);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
}

// ---- the Sinkhorn update from fused-gradient sweeps ---------------------------------------------------
// T(alpha, beta) row sums r give LSE_j((beta_j - M_ij) / eta) = log r_i - alpha_i / eta, so
// optimal_alpha (sinkhorn.h:44-74) is alpha_i + eta (log a_i - log r_i); likewise for beta.  One exp per
// entry and no row maxima: the pass runs at K1's speed.  K1 clamps its exponents to +-700 (dual.h:65-69)
// where the LSE does not, so the identity is exact only while no clamped entry matters: a sum inside
// [e^-600, e^600] has its largest exponent above -600 - log(m), every clamped entry is below e^-700, and
// nothing was clamped from above.  Sums outside that range (or non-finite) raise the flag instead.
constexpr double kSafeLo = 0x1.4dd4d0d12c071p-866;  // e^-600
constexpr double kSafeHi = 0x1.88a122d234b39p+865;  // e^600

__global__ void k_sk_alpha_fin(int nloc, int n_panels, double eta, const double* __restrict__ rowpart,
                               const double* __restrict__ a, double* __restrict__ alpha_io, unsigned int* flag)
{
    bool bad = false;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += gridDim.x * blockDim.x) {
        double r = 0.0;
        for (int P = 0; P < n_panels; ++P) r += rowpart[(size_t)P * nloc + i];  // panel order, as k_gradient_fin1
        if (r >= kSafeLo && r <= kSafeHi) alpha_io[i] += eta * (log(a[i]) - log(r));
        else bad = true;
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

// the same from row sums already on the device (the gradient pass at this very point)
__global__ void k_sk_alpha_from_sums(int nloc, double eta, const double* __restrict__ row_sums, const double* __restrict__ a,
                                     double* __restrict__ alpha_io, unsigned int* flag)
{
    bool bad = false;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += gridDim.x * blockDim.x) {
        const double r = row_sums[i];
        if (r >= kSafeLo && r <= kSafeHi) alpha_io[i] += eta * (log(a[i]) - log(r));
        else bad = true;
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

__global__ void k_sk_cols(int m, const int* __restrict__ panel_seg0, const double* __restrict__ colpart,
                          double* __restrict__ pack)
{
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
        const int P = j / kTC, off = j - P * kTC;
        double c = 0.0;
        for (int sg = panel_seg0[P]; sg < panel_seg0[P + 1]; ++sg) c += colpart[(size_t)sg * kTC + off];
        pack[j] = c;
    }
}

// beta_j += eta (log b_j - log c_j), then the gauge shift of sinkhorn_step (sinkhorn.h:110-113)
__global__ void k_sk_beta_fin(int nloc, int m, double eta, const double* __restrict__ colsum,
                              const double* __restrict__ b, double* __restrict__ beta_io, double* __restrict__ alpha_io,
                              unsigned int* flag)
{
    const double cl = colsum[m - 1];
    const bool last_ok = cl >= kSafeLo && cl <= kSafeHi;
    const double c = last_ok ? beta_io[m - 1] + eta * (log(b[m - 1]) - log(cl)) : 0.0;  // the new beta[m-1]
    bool bad = !last_ok;
    const int stride = gridDim.x * blockDim.x;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m - 1; j += stride) {
        const double cj = colsum[j];
        if (cj >= kSafeLo && cj <= kSafeHi) beta_io[j] = (beta_io[j] + eta * (log(b[j]) - log(cj))) - c;
        else bad = true;
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += stride) alpha_io[i] += c;
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}
// beta[m-1] is read by every block above, so it is zeroed by a separate launch
__global__ void k_sk_gauge_zero(double* beta_io, int m)
{
    if (threadIdx.x == 0 && blockIdx.x == 0) beta_io[m - 1] = 0.0;
}

void launch_sinkhorn_step_fast(regot_ctx* ctx, cudaStream_t st, SweepWS& ws, ncclComm* comm, double* alpha_io,
                               double* beta_io, const double* row_sums_here)
{
    const DeviceProblem& pr = ctx->prob;
    const int nloc = (int)pr.nloc, m = (int)pr.m;
    // alpha from the row sums at (alpha, beta): rows are local, no collective.  When a gradient pass was
    // just made at this point its row sums are those very numbers and the sweep is skipped.
    if (row_sums_here) {
        k_sk_alpha_from_sums<<<vec_grid(ctx, nloc), 256, 0, st>>>(nloc, pr.eta, row_sums_here, pr.a, alpha_io, ws.sk_flag.p);
    } else {
        launch_gradient_sweep_only(ctx, st, ws, alpha_io, beta_io);
        k_sk_alpha_fin<<<vec_grid(ctx, nloc), 256, 0, st>>>(nloc, ctx->plan.n_panels, pr.eta, ws.rowpart.p, pr.a, alpha_io,
                                                            ws.sk_flag.p);
    }
    // beta from the column sums at (alpha', beta), summed over the row blocks
    launch_gradient_sweep_only(ctx, st, ws, alpha_io, beta_io);
    k_sk_cols<<<vec_grid(ctx, m), 256, 0, st>>>(m, ctx->plan.d_panel_seg0.p, ws.colpart.p, ws.pack.p);
    RG_CUDA(cudaGetLastError());
    if (ctx->sharded) allreduce_sum(ctx, comm, ws.pack.p, (size_t)m, st);
    k_sk_beta_fin<<<vec_grid(ctx, std::max(nloc, m)), 256, 0, st>>>(nloc, m, pr.eta, ws.pack.p, pr.b, beta_io, alpha_io,
                                                                    ws.sk_flag.p);
    k_sk_gauge_zero<<<1, 32, 0, st>>>(beta_io, m);
    RG_CUDA(cudaGetLastError());
    ctx->launches += 4;
}

// would the first fast update from these row sums stay in its safe range?  (out[0] = rows outside it)
__global__ void k_rows_outside_safe_range(int nloc, const double* __restrict__ row_sums, double* __restrict__ out)
{
    __shared__ int any;
    if (threadIdx.x == 0) any = 0;
    __syncthreads();
    bool bad = false;
    for (int i = threadIdx.x; i < nloc; i += blockDim.x) {
        const double r = row_sums[i];
        bad |= !(r >= kSafeLo && r <= kSafeHi);
    }
    if (bad) any = 1;
    __syncthreads();
    if (threadIdx.x == 0) out[0] = any ? 1.0 : 0.0;
}

bool fast_sinkhorn_update_is_safe(regot_ctx* ctx, cudaStream_t st, ncclComm* comm, const double* row_sums, DevBuf<double>& scratch)
{
    scratch.ensure(1);
    k_rows_outside_safe_range<<<1, 1024, 0, st>>>((int)ctx->prob.nloc, row_sums, scratch.p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
    allreduce_sum(ctx, comm, scratch.p, 1, st);  // sharded runs: every rank takes the same form of the chain
    double h = 0.0;
    RG_CUDA(cudaMemcpyAsync(&h, scratch.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    RG_CUDA(cudaStreamSynchronize(st));
    return h == 0.0;
}

void reset_sinkhorn_flag(regot_ctx* ctx, cudaStream_t st, SweepWS& ws)
{
    (void)ctx;
    RG_CUDA(cudaMemsetAsync(ws.sk_flag.p, 0, sizeof(unsigned int), st));
}

// sinkhorn_step (sinkhorn.h:105-115) in place on (alpha, beta)
void launch_sinkhorn_step(regot_ctx* ctx, cudaStream_t st, SweepWS& ws, ncclComm* comm, double* alpha_io,
                          double* beta_io)
{
    launch_optimal_alpha(ctx, st, ws, beta_io, alpha_io);
    launch_optimal_beta(ctx, st, ws, comm, alpha_io, beta_io, 1);
}

}  // namespace rg
