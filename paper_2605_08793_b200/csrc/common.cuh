// common.cuh -- device helpers shared by the sm_100a kernels: mbarrier / TMA
// PTX wrappers, the table-driven fp64 exponential, warp reductions.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

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
// the same on a precomputed shared-window address (keeps generic->shared conversions out of hot loops)
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t parity)
{
    uint32_t ok;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void mbar_arrive_s(uint32_t bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ double2 lds_f64x2(uint32_t addr)
{
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
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

// ---- the same exponential in the scaled domain (the sweep kernels' fast path) ---------
// T = exp(d / eta) straight from d = (alpha_i + beta_j) - M_ij:  with cN = N / (eta ln2),
// k = rint(d cN) comes out of one fused multiply-add against the shift constant and the
// reduced argument rw = d cN - k (|rw| <= 1/2, in units of ln2/N) out of a second one with a
// single rounding, so no Cody-Waite split is needed; exp(rw ln2/N) - 1 is the same degree-4
// Taylor polynomial with the powers of ln2/N folded into its coefficients.  9 fp64
// instructions from d to T (the t-domain form above needs 10 from t, 11 from d).  Valid for
// |d / eta| < 700; callers test that on the high word of d (ExpScale::dl_hi) and fall back to
// the clamped t-domain form, so every plan entry has ONE definition (plan_entry_dev) no
// matter which kernel evaluates it.
struct ExpScale {
    double cN;       // N / (eta ln2)
    double inv_eta;  // 1 / eta (slow path, same as the t-domain form)
    unsigned dl_hi;  // high word of a double slightly below 700 eta: abs_hi(d) < dl_hi  =>  |d / eta| < 700
};
inline ExpScale make_exp_scale(double eta)
{
    ExpScale E;
    E.cN = (double)((long double)kExpN / ((long double)eta * 0.693147180559945309417232121458176568L));
    E.inv_eta = 1.0 / eta;
    const double lim = 700.0 * eta * (1.0 - 1e-9);
    unsigned long long bits;
    memcpy(&bits, &lim, sizeof(bits));
    E.dl_hi = (unsigned)(bits >> 32);  // truncation of the low word only lowers the bound
    return E;
}
struct ExpPoly {
    static constexpr double a1 = 0x1.62e42fefa39efp-9;   // (ln2/N)
    static constexpr double a2 = 0x1.ebfbdff82c58fp-19;  // (ln2/N)^2 / 2
    static constexpr double a3 = 0x1.c6b08d704a0c0p-29;  // (ln2/N)^3 / 6
    static constexpr double a4 = 0x1.3b2ab6fba4e77p-39;  // (ln2/N)^4 / 24
};

// shared address of table entry (ki mod N) of this lane's copy: LOP3 + LEA
__device__ __forceinline__ uint32_t exp_tbl_addr(int ki, uint32_t tbl_lane)
{
    uint32_t a;
    asm("{\n\t.reg .u32 j;\n\tand.b32 j, %1, 255;\n\tmad.lo.u32 %0, j, 128, %2;\n\t}" : "=r"(a) : "r"(ki), "r"(tbl_lane));
    return a;
}
__device__ __forceinline__ double lds_f64(uint32_t addr)
{
    double s;
    asm("ld.shared.f64 %0, [%1];" : "=d"(s) : "r"(addr));
    return s;
}
// 2^(k/N) from the table word and k: exponent inserted with one integer multiply-add
__device__ __forceinline__ double exp_scale_pow2(double s, int ki)
{
    return __hiloint2double(__double2hiint(s) + (int)((unsigned)ki << (20 - kExpShift)), __double2loint(s));
}

__device__ __forceinline__ double exp_scaled(double d, double cN, uint32_t tbl_lane)
{
    const double kd = __fma_rn(d, cN, ExpConst::shift);
    const int ki = __double2loint(kd);
    const double rw = __fma_rn(d, cN, ExpConst::shift - kd);  // shift - kd == -k exactly
    const double s = exp_scale_pow2(lds_f64(exp_tbl_addr(ki, tbl_lane)), ki);
    double p = __fma_rn(rw, ExpPoly::a4, ExpPoly::a3);
    p = __fma_rn(rw, p, ExpPoly::a2);
    p = __fma_rn(rw, p, ExpPoly::a1);
    return __fma_rn(s, rw * p, s);
}

// NE independent entries, written stage by stage so the NE dependency chains interleave
template <int NE>
__device__ __forceinline__ void exp_scaled_vec(const double (&d)[NE], double cN, uint32_t tbl_lane, double (&T)[NE])
{
    double kd[NE], rw[NE], s[NE], p[NE];
#pragma unroll
    for (int k = 0; k < NE; ++k) kd[k] = __fma_rn(d[k], cN, ExpConst::shift);
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        s[k] = lds_f64(exp_tbl_addr(__double2loint(kd[k]), tbl_lane));
        rw[k] = __fma_rn(d[k], cN, ExpConst::shift - kd[k]);
    }
#pragma unroll
    for (int k = 0; k < NE; ++k) p[k] = __fma_rn(rw[k], ExpPoly::a4, ExpPoly::a3);
#pragma unroll
    for (int k = 0; k < NE; ++k) p[k] = __fma_rn(rw[k], p[k], ExpPoly::a2);
#pragma unroll
    for (int k = 0; k < NE; ++k) p[k] = __fma_rn(rw[k], p[k], ExpPoly::a1);
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        s[k] = exp_scale_pow2(s[k], __double2loint(kd[k]));
        T[k] = __fma_rn(s[k], rw[k] * p[k], s[k]);
    }
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

// plan_entry (dual.h:62-70) on the device, from d = (alpha_i + beta_j) - M_ij: the ONE definition
// every kernel uses (gradient sweep, top-k sweeps, value refresh, dense plan), so a plan entry has
// the same bits wherever it is evaluated:
//     |d / eta| >= 700  ->  exp(+-700) exactly (the reference's clamp, as correctly rounded constants)
//     otherwise         ->  exp_scaled(d)
// The cheap filter abs_hi(d) < dl_hi proves |d / eta| < 700; only entries (or 8-entry groups) that
// fail it pay for t = d / eta and the saturation selects.
constexpr double kExp700 = 0x1.d945df4f8ec8ep+1009;    // exp(700)
constexpr double kExpM700 = 0x1.14f2b0fb9307fp-1010;   // exp(-700)

__device__ __forceinline__ bool saturates(double d, double inv_eta, double& sat_value)
{
    const double t = d * inv_eta;
    const int hi = __double2hiint(t);
    sat_value = hi < 0 ? kExpM700 : kExp700;
    return ((unsigned)hi & 0x7fffffffu) >= kHi700;  // |t| >= 700 (low word of 700.0 is zero), inf or NaN
}
__device__ __forceinline__ double plan_entry_dev(double d, const ExpScale& E, uint32_t tbl_lane)
{
    double c;
    if (abs_hi(d) >= E.dl_hi && saturates(d, E.inv_eta, c)) return c;
    return exp_scaled(d, E.cN, tbl_lane);
}
// NE entries of one lane: the whole group skips the saturation test when the filter clears it
template <int NE>
__device__ __forceinline__ void plan_entries_dev(const double (&d)[NE], const ExpScale& E, uint32_t tbl_lane,
                                                 double (&T)[NE])
{
    unsigned amax = 0;
#pragma unroll
    for (int k = 0; k < NE; ++k) amax = max(amax, abs_hi(d[k]));
    // warp-uniform choice (all 32 lanes call this together): one lane with a saturating entry sends
    // the whole warp down the second branch instead of serialising both; per-entry results do not
    // depend on the branch taken
    if (!__any_sync(0xffffffffu, amax >= E.dl_hi)) {
        exp_scaled_vec<NE>(d, E.cN, tbl_lane, T);
    } else {
        double dc[NE], c[NE];
        bool sat[NE];
#pragma unroll
        for (int k = 0; k < NE; ++k) {
            sat[k] = saturates(d[k], E.inv_eta, c[k]);
            dc[k] = sat[k] ? 0.0 : d[k];
        }
        exp_scaled_vec<NE>(dc, E.cN, tbl_lane, T);
#pragma unroll
        for (int k = 0; k < NE; ++k) T[k] = sat[k] ? c[k] : T[k];
    }
}
// the same with the (non-replicated) table read through the read-only global path
__device__ __forceinline__ double plan_entry_dev_g(double d, const ExpScale& E, const double* __restrict__ tbl)
{
    double c;
    if (abs_hi(d) >= E.dl_hi && saturates(d, E.inv_eta, c)) return c;
    const double kd = __fma_rn(d, E.cN, ExpConst::shift);
    const int ki = __double2loint(kd);
    const double rw = __fma_rn(d, E.cN, ExpConst::shift - kd);
    const double s = exp_scale_pow2(__ldg(tbl + ((unsigned)ki & (kExpN - 1))), ki);
    double p = __fma_rn(rw, ExpPoly::a4, ExpPoly::a3);
    p = __fma_rn(rw, p, ExpPoly::a2);
    p = __fma_rn(rw, p, ExpPoly::a1);
    return __fma_rn(s, rw * p, s);
}

// ---- host mailbox (ctx.hpp HostMailbox): one thread posts n doubles, then the sequence number ----
__device__ __forceinline__ void mailbox_post(double* mbox, const double* vals, int n, unsigned long long seq)
{
    volatile double* d = mbox;
    for (int k = 0; k < n; ++k) d[k] = vals[k];
    __threadfence_system();
    reinterpret_cast<volatile unsigned long long*>(mbox)[31] = seq;
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
