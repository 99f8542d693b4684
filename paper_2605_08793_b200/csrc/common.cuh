// common.cuh -- device helpers shared by the sm_100a kernels: mbarrier / TMA
// PTX wrappers, the table-driven fp64 exponential, warp reductions.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rg {

constexpr int kWarp = 32;

// ---- shared-memory address + mbarrier --------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// make mbarrier.init visible to the async (TMA) proxy
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    while (!mbar_try_wait(bar, parity)) {
    }
}

// ---- TMA: 2-D tiled bulk tensor load, completion on an mbarrier -------------
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map)
{
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_first()
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// c0 = innermost (column) coordinate, c1 = row coordinate, in elements
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;"
        ::"r"(smem_u32(smem_dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];"
        ::"r"(smem_u32(smem_dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// named barrier among a subset of the CTA's warps (id 1..15; 0 is __syncthreads)
__device__ __forceinline__ void bar_sync(int id, int nthreads)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---- fp64 exponential --------------------------------------------------------
// exp(t) = 2^(k/N) * exp(r), N = 256, k = rint(t N / ln2), r = t - k ln2/N,
// |r| <= ln2/512.  2^(j/N) (j = k mod N) comes from a 256-entry table, the
// integer part of k/N goes straight into the exponent field, exp(r)-1 is a
// degree-4 Taylor polynomial (truncation r^5/120 < 4e-17 relative).  Valid for
// |t| <= 700 where every intermediate and the result are normal numbers, which
// the reference's clamp (dual.h:65-69) guarantees.  Error < 1 ulp.
//
// The table stores the high word of 2^(j/N) pre-biased by -(j << 12), so the
// exponent insertion is one integer multiply-add: hi + (k << 12) ==
// hi(2^(j/N)) + ((k >> 8) << 20).
constexpr int kExpN = 256;
constexpr int kExpShift = 8;    // log2(kExpN)
constexpr int kExpCopies = 16;  // table replicated so each lane of a half-warp owns a bank pair
constexpr int kExpTableBytes = kExpN * kExpCopies * 8;

struct ExpConst {
    static constexpr double inv_ln2_n = 0x1.71547652b82fep+8;  // N / ln2
    static constexpr double shift = 0x1.8p52;
    static constexpr double ln2_n_hi = 0x1.62e42fef00000p-9;  // ln2 / N, 33 significant bits
    static constexpr double ln2_n_lo = 0x1.473de6af278edp-42;
    static constexpr double c2 = 0.5, c3 = 1.0 / 6.0, c4 = 1.0 / 24.0;
};

// Fill the replicated shared-memory table from the 256-entry (biased) global
// table.  Entry j of copy c lives at double index j * kExpCopies + c.
__device__ __forceinline__ void exp_table_fill(double* tbl_smem, const double* __restrict__ tbl_gmem, int tid,
                                               int nthreads)
{
    for (int q = tid; q < kExpN * kExpCopies; q += nthreads) tbl_smem[q] = tbl_gmem[q / kExpCopies];
}

// tbl_lane = shared address (u32) of this lane's copy: base + (lane & 15) * 8
__device__ __forceinline__ double exp_tbl(double t, uint32_t tbl_lane)
{
    const double kd = __fma_rn(t, ExpConst::inv_ln2_n, ExpConst::shift);
    const int ki = __double2loint(kd);
    const double kf = kd - ExpConst::shift;
    double r = __fma_rn(kf, -ExpConst::ln2_n_hi, t);
    r = __fma_rn(kf, -ExpConst::ln2_n_lo, r);
    double s;
    asm("ld.shared.f64 %0, [%1];" : "=d"(s) : "r"(tbl_lane + (((uint32_t)ki & (kExpN - 1)) << 7)));
    s = __hiloint2double(__double2hiint(s) + (int)((unsigned)ki << (20 - kExpShift)), __double2loint(s));
    const double r2 = r * r;
    double p = __fma_rn(r, ExpConst::c3, ExpConst::c2);
    p = __fma_rn(r2, ExpConst::c4, p);
    const double q = __fma_rn(r2, p, r);
    return __fma_rn(s, q, s);
}

// same function with the (non-replicated) table read through the read-only
// global path; for low-volume kernels that do not stage the table in smem
__device__ __forceinline__ double exp_tbl_g(double t, const double* __restrict__ tbl)
{
    const double kd = __fma_rn(t, ExpConst::inv_ln2_n, ExpConst::shift);
    const int ki = __double2loint(kd);
    const double kf = kd - ExpConst::shift;
    double r = __fma_rn(kf, -ExpConst::ln2_n_hi, t);
    r = __fma_rn(kf, -ExpConst::ln2_n_lo, r);
    double s = __ldg(tbl + ((unsigned)ki & (kExpN - 1)));
    s = __hiloint2double(__double2hiint(s) + (int)((unsigned)ki << (20 - kExpShift)), __double2loint(s));
    const double r2 = r * r;
    double p = __fma_rn(r, ExpConst::c3, ExpConst::c2);
    p = __fma_rn(r2, ExpConst::c4, p);
    const double q = __fma_rn(r2, p, r);
    return __fma_rn(s, q, s);
}

// |t| >= 700 (or NaN) test on the high word; amax accumulates max |hi|
__device__ __forceinline__ unsigned abs_hi(double t) { return (unsigned)__double2hiint(t) & 0x7fffffffu; }
constexpr unsigned kHi700 = 0x4085E000u;

// reference clamp (dual.h:65-69): |t| > 700 -> +-700, decided on the high word
__device__ __forceinline__ double clamp700(double t)
{
    const int hi = __double2hiint(t);
    if (((unsigned)hi & 0x7fffffffu) >= kHi700) {
        // |t| >= 700 (or NaN): replace by +-700 keeping the sign
        t = __hiloint2double((hi & 0x80000000) | (int)kHi700, 0);
    }
    return t;
}

// ---- warp reductions ---------------------------------------------------------
__device__ __forceinline__ double shfl_xor_d(double v, int mask) { return __shfl_xor_sync(0xffffffffu, v, mask); }
__device__ __forceinline__ double shfl_idx_d(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += shfl_xor_d(v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, shfl_xor_d(v, o));
    return v;
}

// Transposing reduction of 8 per-lane values across the warp: after the call
// lane L with (L & 3) == 0 holds in the return value the warp-wide sum of
// v[(L >> 2) & 7].  9 adds + 9 64-bit shuffles instead of 40 + 40.  The
// summation order is fixed (a butterfly), so results are run-to-run identical.
__device__ __forceinline__ double warp_sum8_transpose(const double (&v)[8], int lane)
{
    double a[4], b[2], c;
    const bool h16 = (lane & 16) != 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double send = h16 ? v[k] : v[k + 4];
        const double keep = h16 ? v[k + 4] : v[k];
        a[k] = keep + shfl_xor_d(send, 16);
    }
    const bool h8 = (lane & 8) != 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const double send = h8 ? a[k] : a[k + 2];
        const double keep = h8 ? a[k + 2] : a[k];
        b[k] = keep + shfl_xor_d(send, 8);
    }
    const bool h4 = (lane & 4) != 0;
    {
        const double send = h4 ? b[0] : b[1];
        const double keep = h4 ? b[1] : b[0];
        c = keep + shfl_xor_d(send, 4);
    }
    c += shfl_xor_d(c, 2);
    c += shfl_xor_d(c, 1);
    // lane bits (4,3,2) = (h16,h8,h4) select index 4*h16 + 2*h8 + h4
    return c;
}
// index held by lane L after warp_sum8_transpose
__device__ __forceinline__ int warp_sum8_index(int lane) { return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1); }

// Deterministic block reduction of `NV` doubles per thread (sum); result valid
// in thread 0.  scratch must hold NV * (blockDim.x / 32) doubles.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* scratch)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) scratch[k * nwarp + warp] = v[k];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double s = 0.0;
            for (int w = lane; w < nwarp; w += 32) s += scratch[k * nwarp + w];
            v[k] = warp_sum(s);
        }
    }
    __syncthreads();
}

}  // namespace rg
