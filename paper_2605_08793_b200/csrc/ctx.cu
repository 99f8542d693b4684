// ctx.cu -- context lifetime, problem upload (with on-device transposition of
// column-major input), TMA tensor map, sweep plan, NCCL plumbing.
#include "ctx.hpp"
#include "sweep.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>

namespace rg {

// ---- NCCL, resolved lazily so single-GPU use has no libnccl dependency ---------------
namespace {
struct NcclApi {
    void* lib = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string why;
};
NcclApi& nccl()
{
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // REGOT_B200_NCCL_LIB names another library with the same five entry points: the tests point it at a
        // loopback communicator (tests/fake_nccl) that runs R ranks as R contexts of one process on one GPU
        if (const char* path = std::getenv("REGOT_B200_NCCL_LIB")) {
            api.lib = dlopen(path, RTLD_NOW | RTLD_LOCAL);
            if (!api.lib) {
                api.why = std::string("REGOT_B200_NCCL_LIB: ") + (dlerror() ? dlerror() : "dlopen failed");
                return;
            }
        }
        // RTLD_NOLOAD first: reuse the copy torch already mapped (same SONAME)
        if (!api.lib) api.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!api.lib) api.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!api.lib) {
            const char* why = dlerror();
            api.why = why ? why : "dlopen(libnccl.so.2) failed";
            return;
        }
        api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(api.lib, "ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))dlsym(api.lib, "ncclCommInitRank");
        api.AllReduce = (decltype(api.AllReduce))dlsym(api.lib, "ncclAllReduce");
        api.CommDestroy = (decltype(api.CommDestroy))dlsym(api.lib, "ncclCommDestroy");
        api.GetErrorString = (decltype(api.GetErrorString))dlsym(api.lib, "ncclGetErrorString");
        if (!api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.CommDestroy) {
            api.why = "libnccl.so.2 lacks a required symbol";
            api.lib = nullptr;
        }
    });
    return api;
}
void nccl_check(ncclResult_t r, const char* what)
{
    if (r != ncclSuccess)
        raise(REGOT_E_NCCL, std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error"));
}
}  // namespace

void nccl_unique_id(void* out128)
{
    if (!nccl().lib) raise(REGOT_E_NCCL, "NCCL unavailable: " + nccl().why);
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, 128);
}

void comm_init(regot_ctx* ctx, int rank, int world, const void* id128)
{
    if (world < 1 || rank < 0 || rank >= world) raise(REGOT_E_VALIDATION, "comm_init: bad rank/world");
    ctx->rank = rank;
    ctx->world = world;
    // REGOT_B200_SHARDED_SINGLE: a one-rank communicator takes the sharded path (row-block upload, every collective
    // issued) -- how the tests run the real libnccl on one GPU
    const char* single = std::getenv("REGOT_B200_SHARDED_SINGLE");
    ctx->sharded = world > 1 || (id128 != nullptr && single && single[0] == '1');
    if (world == 1 && id128 == nullptr) return;
    if (!nccl().lib) raise(REGOT_E_NCCL, "NCCL unavailable: " + nccl().why);
    // two communicators from two ids packed back to back (2 x 128 bytes): the
    // side stream's collectives must not interleave with the main stream's
    ncclUniqueId id[2];
    std::memcpy(id, id128, sizeof(id));
    RG_CUDA(cudaSetDevice(ctx->device));
    nccl_check(nccl().CommInitRank(&ctx->comm, world, id[0], rank), "ncclCommInitRank(main)");
    nccl_check(nccl().CommInitRank(&ctx->comm_side, world, id[1], rank), "ncclCommInitRank(side)");
}

void comm_destroy(regot_ctx* ctx)
{
    if (ctx->comm) nccl().CommDestroy(ctx->comm);
    if (ctx->comm_side) nccl().CommDestroy(ctx->comm_side);
    ctx->comm = ctx->comm_side = nullptr;
}

void allreduce_sum(regot_ctx* ctx, ncclComm* comm, double* buf, size_t count, cudaStream_t st)
{
    if (!ctx->sharded) return;
    if (!comm) raise(REGOT_E_NCCL, "allreduce: communicator not initialised (regot_b200_comm_init)");
    nccl_check(nccl().AllReduce(buf, buf, count, ncclDouble, ncclSum, comm, st), "ncclAllReduce(sum)");
}
void allreduce_max(regot_ctx* ctx, ncclComm* comm, double* buf, size_t count, cudaStream_t st)
{
    if (!ctx->sharded) return;
    if (!comm) raise(REGOT_E_NCCL, "allreduce: communicator not initialised (regot_b200_comm_init)");
    nccl_check(nccl().AllReduce(buf, buf, count, ncclDouble, ncclMax, comm, st), "ncclAllReduce(max)");
}

void allreduce_sum_u64(regot_ctx* ctx, ncclComm* comm, unsigned long long* buf, size_t count, cudaStream_t st)
{
    if (!ctx->sharded) return;
    if (!comm) raise(REGOT_E_NCCL, "allreduce: communicator not initialised (regot_b200_comm_init)");
    nccl_check(nccl().AllReduce(buf, buf, count, ncclUint64, ncclSum, comm, st), "ncclAllReduce(u64)");
}

// ---- context ---------------------------------------------------------------------------
void ctx_require_problem(const regot_ctx* ctx)
{
    if (!ctx->prob.loaded) raise(REGOT_E_VALIDATION, "no problem uploaded (regot_b200_set_problem)");
}

regot_ctx* ctx_create(int device)
{
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        raise(REGOT_E_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e) +
                                " -- this library has no CPU fallback");
    if (device < 0 || device >= count) raise(REGOT_E_VALIDATION, "create: device index out of range");
    RG_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    RG_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        raise(REGOT_E_UNSUPPORTED, std::string("device '") + prop.name + "' is sm_" + std::to_string(prop.major) +
                                       std::to_string(prop.minor) + "; this build contains sm_100a code only");
    auto* ctx = new regot_ctx();
    try {
        ctx->device = device;
        ctx->sm_count = prop.multiProcessorCount;
        if (const char* e = std::getenv("REGOT_B200_MULTIKERNEL_PCG")) ctx->force_multikernel_pcg = e[0] == '1';
        if (const char* e = std::getenv("REGOT_B200_PANEL_SPMV")) ctx->panel_spmv = std::atoi(e);
        if (const char* e = std::getenv("REGOT_B200_PANEL_WIDTH")) ctx->panel_width = std::atoi(e);
        if (const char* e = std::getenv("REGOT_B200_PANEL_ELL")) ctx->panel_ell = std::atoi(e);
        if (const char* e = std::getenv("REGOT_B200_PANEL_AHEAD")) ctx->panel_ahead = std::max(0, std::atoi(e));
        // off by default: measured 11 % (config A) / 1 % (1600 x 1200) of the direction solve, slower above ~50k entries
        ctx->pcg_cluster_size = 0;
        ctx->pcg_cluster_max_entries = 50000;
        if (const char* e = std::getenv("REGOT_B200_FUSED_FINALIZE")) ctx->fused_finalize = e[0] != '0';
        if (const char* e = std::getenv("REGOT_B200_EXTENDED_F")) ctx->extended_f = e[0] != '0';
        if (const char* e = std::getenv("REGOT_B200_SCHUR_DIAG")) ctx->schur_diag = std::atoi(e);
        if (const char* e = std::getenv("REGOT_B200_TOPK_GUESS")) ctx->topk_guess = std::atoi(e);
        if (const char* e = std::getenv("REGOT_B200_PATTERN_DRIFT")) ctx->pattern_drift = std::max(0.0, std::atof(e));
        if (const char* e = std::getenv("REGOT_B200_PATTERN_MAX_SKIPS")) ctx->pattern_max_skips = std::max(0, std::atoi(e));
        if (const char* e = std::getenv("REGOT_B200_PCG_BLOCKS")) ctx->pcg_blocks = std::atoi(e);
        if (const char* e = std::getenv("REGOT_B200_PCG_BLOCKS_CLUSTER")) ctx->pcg_blocks_cluster = std::atoi(e);
        if (const char* e = std::getenv("REGOT_B200_PCG_BLOCKS_ONE_CLUSTER_ENTRIES")) ctx->pcg_blocks_one_cluster_entries = std::atol(e);
        if (const char* e = std::getenv("REGOT_B200_PCG_BLOCKS_CLUSTER_ENTRIES")) ctx->pcg_blocks_cluster_entries = std::atol(e);
        if (const char* e = std::getenv("REGOT_B200_PCG_BLOCKS_GRID")) {
            int bp = 0, bq = 0;
            if (std::sscanf(e, "%dx%d", &bp, &bq) == 2 && bp >= 1 && bq >= 1 && bp <= 32 && bq <= 32) {
                ctx->pcg_blocks_p = bp;
                ctx->pcg_blocks_q = bq;
            }
        }
        if (const char* e = std::getenv("REGOT_B200_PCG_CLUSTER")) ctx->pcg_cluster_size = std::atoi(e);
        if (const char* e = std::getenv("REGOT_B200_PCG_CLUSTER_ENTRIES")) ctx->pcg_cluster_max_entries = std::atol(e);
        if (const char* e = std::getenv("REGOT_B200_EXACT_LSE")) ctx->fast_sinkhorn = e[0] != '1';
        if (const char* e = std::getenv("REGOT_B200_LSE_FAST_SHIFT")) ctx->lse_fast_shift = e[0] != '0';
        if (const char* e = std::getenv("REGOT_B200_FAST_CHAIN")) ctx->fast_sinkhorn_chain = e[0] != '0';
        RG_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        RG_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
        RG_CUDA(cudaEventCreate(&ctx->ev_a));
        RG_CUDA(cudaEventCreate(&ctx->ev_b));
        RG_CUDA(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
        RG_CUDA(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
        // 2^(j/N) correctly rounded from long double, high word biased by -(j << 12)
        // (see exp_tbl in common.cuh)
        double tbl[kExpN];
        for (int j = 0; j < kExpN; ++j) {
            const double v = (double)exp2l((long double)j / (long double)kExpN);
            std::uint64_t bits;
            std::memcpy(&bits, &v, 8);
            bits -= (std::uint64_t)j << (32 + 20 - kExpShift);
            std::memcpy(&tbl[j], &bits, 8);
        }
        ctx->exp_table.ensure(kExpN);
        RG_CUDA(cudaMemcpy(ctx->exp_table.p, tbl, sizeof(tbl), cudaMemcpyHostToDevice));
    } catch (...) {
        delete ctx;
        throw;
    }
    return ctx;
}

void ctx_destroy(regot_ctx* ctx)
{
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    comm_destroy(ctx);
    extern void solver_ws_free(regot_ctx*);
    solver_ws_free(ctx);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    for (cudaEvent_t ev : {ctx->ev_a, ctx->ev_b, ctx->ev_fork, ctx->ev_join})
        if (ev) cudaEventDestroy(ev);
    delete ctx;
}

// ---- tensor map ----------------------------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled()
{
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        RG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) raise(REGOT_E_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = (EncodeTiledFn)p;
    }
    return fn;
}

static void build_tensor_map(regot_ctx* ctx)
{
    DeviceProblem& pr = ctx->prob;
    if ((reinterpret_cast<uintptr_t>(pr.M) & 15u) != 0 || (pr.ld % 2) != 0)
        raise(REGOT_E_VALIDATION, "set_problem: device cost matrix must be 16-byte aligned with an even pitch");
    const cuuint64_t dims[2] = {(cuuint64_t)pr.m, (cuuint64_t)pr.nloc};
    const cuuint64_t strides[1] = {(cuuint64_t)pr.ld * 8u};
    const cuuint32_t box[2] = {(cuuint32_t)kTC, (cuuint32_t)kTR};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_tiled()(&pr.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(pr.M), dims,
                                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) raise(REGOT_E_CUDA, "cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r));
}

// ---- sweep plan -----------------------------------------------------------------------------
void make_sweep_plan(regot_ctx* ctx)
{
    const DeviceProblem& pr = ctx->prob;
    SweepPlan& pl = ctx->plan;
    pl.tile_rows = kTR;
    pl.tile_cols = kTC;
    pl.n_row_tiles = (int)((pr.nloc + kTR - 1) / kTR);
    pl.n_panels = (int)((pr.m + kTC - 1) / kTC);
    pl.total_tiles = (long)pl.n_row_tiles * pl.n_panels;
    pl.grid = (int)std::max<long>(1, std::min<long>(ctx->sm_count, pl.total_tiles));
    std::vector<int> cta_seg0((size_t)pl.grid + 1, 0), panel_seg0((size_t)pl.n_panels + 1, 0);
    std::vector<int> panel_cnt((size_t)pl.n_panels, 0);
    int seg = 0;
    for (int b = 0; b < pl.grid; ++b) {
        cta_seg0[(size_t)b] = seg;
        const long t0 = pl.total_tiles * b / pl.grid, t1 = pl.total_tiles * (b + 1) / pl.grid;
        if (t1 > t0) {
            const int p0 = (int)(t0 / pl.n_row_tiles), p1 = (int)((t1 - 1) / pl.n_row_tiles);
            for (int P = p0; P <= p1; ++P) ++panel_cnt[(size_t)P];
            seg += p1 - p0 + 1;
        }
    }
    cta_seg0[(size_t)pl.grid] = seg;
    pl.n_segments = seg;
    // segments are numbered in tile order, so each panel's segments are contiguous
    for (int P = 0; P < pl.n_panels; ++P) panel_seg0[(size_t)P + 1] = panel_seg0[(size_t)P] + panel_cnt[(size_t)P];
    pl.d_cta_seg0.ensure(cta_seg0.size());
    pl.d_panel_seg0.ensure(panel_seg0.size());
    RG_CUDA(cudaMemcpy(pl.d_cta_seg0.p, cta_seg0.data(), sizeof(int) * cta_seg0.size(), cudaMemcpyHostToDevice));
    RG_CUDA(cudaMemcpy(pl.d_panel_seg0.p, panel_seg0.data(), sizeof(int) * panel_seg0.size(), cudaMemcpyHostToDevice));
}

void ensure_sweep_ws(regot_ctx* ctx, SweepWS& ws)
{
    const DeviceProblem& pr = ctx->prob;
    const SweepPlan& pl = ctx->plan;
    ws.rowpart.ensure((size_t)pl.n_panels * (size_t)pr.nloc);
    ws.rowpart2.ensure((size_t)pl.n_panels * (size_t)pr.nloc);
    ws.colpart.ensure((size_t)pl.n_segments * kTC);
    ws.colpart2.ensure((size_t)pl.n_segments * kTC);
    ws.pack.ensure((size_t)pr.m + 16);
    ws.pack2.ensure(2 * (size_t)pr.m + 32);
    ws.partials.ensure((size_t)(2 * ctx->sm_count + 8) * (12 * 2 + 6));  // per CTA: 8 (two-kernel finalize) or 12 (fused) scalars, + 3 double-doubles behind 2 x grid of them
    if (!ws.ticket.p) {
        ws.ticket.ensure(8);
        RG_CUDA(cudaMemset(ws.ticket.p, 0, 8 * sizeof(unsigned int)));
    }
    ws.d_scal.ensure(1);
    if (!ws.sk_flag.p) {
        ws.sk_flag.ensure(1);
        RG_CUDA(cudaMemset(ws.sk_flag.p, 0, sizeof(unsigned int)));
    }
    ws.mbox.ensure();
}

// ---- problem upload ---------------------------------------------------------------------------
// out[i * ldo + j] = in[j * ldi + i] for i < rows, j < cols (in: column-major block)
__global__ void k_transpose(int rows, int cols, const double* __restrict__ in, long ldi, double* __restrict__ out,
                            long ldo)
{
    __shared__ double tile[32][33];
    const int bi = blockIdx.x * 32, bj = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int i = bi + threadIdx.x, j = bj + r;
        if (i < rows && j < cols) tile[r][threadIdx.x] = in[(size_t)j * ldi + i];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int i = bi + r, j = bj + threadIdx.x;
        if (i < rows && j < cols) out[(size_t)i * ldo + j] = tile[threadIdx.x][r];
    }
}

static void finish_problem(regot_ctx* ctx)
{
    if (ctx->prob.on_the_fly) std::memset(&ctx->prob.tmap, 0, sizeof(ctx->prob.tmap));  // the sweeps compute their tiles
    else build_tensor_map(ctx);
    ctx->prob.loaded = true;
    ctx->topk_prev_bin = -1;  // a threshold bin of the previous problem says nothing about this one
    make_sweep_plan(ctx);
    ensure_sweep_ws(ctx, ctx->ws_main);
    ensure_sweep_ws(ctx, ctx->ws_side);
}

static void check_shape(int64_t n, int64_t m, int64_t row_begin, int64_t row_count, double eta)
{
    // validate_problem (problem.h:30-50) shape and eta rules; the marginal and
    // finiteness rules are checked on the device by regot_b200_validate_problem
    if (n < 1 || m < 1) raise(REGOT_E_VALIDATION, "problem: n and m must be at least 1");
    if (row_begin < 0 || row_count < 1 || row_begin + row_count > n)
        raise(REGOT_E_VALIDATION, "problem: row block out of range");
    if (!(eta > 0.0) || !std::isfinite(eta)) raise(REGOT_E_VALIDATION, "problem: eta must be positive and finite");
    if (n >= (1LL << 30) || m >= (1LL << 30)) raise(REGOT_E_VALIDATION, "problem: dimension exceeds int32 index range");
}

void set_problem_host(regot_ctx* ctx, int64_t n, int64_t m, int64_t row_begin, int64_t row_count, const double* M,
                      int layout, int64_t ld, const double* a, const double* b, double eta)
{
    check_shape(n, m, row_begin, row_count, eta);
    if (!M || !a || !b) raise(REGOT_E_VALIDATION, "problem: null input");
    if (layout != REGOT_LAYOUT_COLMAJOR && layout != REGOT_LAYOUT_ROWMAJOR)
        raise(REGOT_E_VALIDATION, "problem: unknown cost-matrix layout");
    if ((layout == REGOT_LAYOUT_COLMAJOR && ld < n) || (layout == REGOT_LAYOUT_ROWMAJOR && ld < m))
        raise(REGOT_E_VALIDATION, "problem: cost matrix shape mismatch");
    RG_CUDA(cudaSetDevice(ctx->device));
    DeviceProblem& pr = ctx->prob;
    pr.loaded = false;
    pr.on_the_fly = false;
    pr.cloud_d = 0;
    pr.n = n;
    pr.m = m;
    pr.row_begin = row_begin;
    pr.nloc = row_count;
    pr.eta = eta;
    pr.ld = (m + 15) / 16 * 16;  // 128-byte row pitch
    pr.M_own.ensure((size_t)pr.nloc * (size_t)pr.ld);
    pr.a_own.ensure((size_t)pr.nloc);
    pr.b_own.ensure((size_t)m);
    pr.M = pr.M_own.p;
    pr.a = pr.a_own.p;
    pr.b = pr.b_own.p;
    cudaStream_t st = ctx->stream;
    RG_CUDA(cudaMemsetAsync(pr.M_own.p, 0, sizeof(double) * (size_t)pr.nloc * (size_t)pr.ld, st));
    if (layout == REGOT_LAYOUT_ROWMAJOR) {
        RG_CUDA(cudaMemcpy2DAsync(pr.M_own.p, (size_t)pr.ld * 8, M, (size_t)ld * 8, (size_t)m * 8, (size_t)pr.nloc,
                                  cudaMemcpyHostToDevice, st));
    } else {
        // column-major (Eigen) source: copy the row block of every column, transpose on the device
        DevBuf<double> stagebuf;
        stagebuf.ensure((size_t)pr.nloc * (size_t)m);
        RG_CUDA(cudaMemcpy2DAsync(stagebuf.p, (size_t)pr.nloc * 8, M + row_begin, (size_t)ld * 8, (size_t)pr.nloc * 8,
                                  (size_t)m, cudaMemcpyHostToDevice, st));
        const dim3 grid((unsigned)((pr.nloc + 31) / 32), (unsigned)((m + 31) / 32)), block(32, 8);
        k_transpose<<<grid, block, 0, st>>>((int)pr.nloc, (int)m, stagebuf.p, (long)pr.nloc, pr.M_own.p, (long)pr.ld);
        RG_CUDA(cudaGetLastError());
        ++ctx->launches;
        RG_CUDA(cudaStreamSynchronize(st));
    }
    RG_CUDA(cudaMemcpyAsync(pr.a_own.p, a + row_begin, sizeof(double) * (size_t)pr.nloc, cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaMemcpyAsync(pr.b_own.p, b, sizeof(double) * (size_t)m, cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaStreamSynchronize(st));
    finish_problem(ctx);
}

void set_problem_device(regot_ctx* ctx, int64_t n, int64_t m, int64_t row_begin, int64_t row_count,
                        const double* M_dev, int64_t ld, const double* a_dev, const double* b_dev, double eta)
{
    check_shape(n, m, row_begin, row_count, eta);
    if (!M_dev || !a_dev || !b_dev) raise(REGOT_E_VALIDATION, "problem: null input");
    if (ld < m) raise(REGOT_E_VALIDATION, "problem: cost matrix shape mismatch");
    RG_CUDA(cudaSetDevice(ctx->device));
    DeviceProblem& pr = ctx->prob;
    pr.loaded = false;
    pr.on_the_fly = false;
    pr.cloud_d = 0;
    pr.n = n;
    pr.m = m;
    pr.row_begin = row_begin;
    pr.nloc = row_count;
    pr.eta = eta;
    pr.ld = ld;
    pr.M = M_dev;
    pr.a = a_dev;
    pr.b = b_dev;
    finish_problem(ctx);
}

// ---- point-cloud problems ------------------------------------------------------------------------
// cost = |x_i - y_j|^2 / max (problem.h:53-61, 124-132), formed on the device with the arithmetic of
// cloud_sqdist (sweep.cuh) so it equals the host generators' matrix bit for bit.
constexpr int kCloudCols = 256;

// maximum of the un-normalised cost over this rank's rows: one partial per block
__global__ void __launch_bounds__(kCloudCols) k_cloud_max(int nloc, int m, const CloudGeom c, double* __restrict__ blockmax)
{
    __shared__ double wmax[kCloudCols / 32];
    const int j = blockIdx.x * kCloudCols + threadIdx.x;
    double mx = 0.0;
    if (j < m) {
        const double* yj = c.Y + (size_t)j * c.d;
        for (int i = blockIdx.y; i < nloc; i += gridDim.y) mx = fmax(mx, cloud_sqdist(c.X + (size_t)i * c.d, yj, c.d));
    }
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kCloudCols / 32; ++w) mx = fmax(mx, wmax[w]);
        blockmax[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = mx;
    }
}

// does cloud_div_fast reproduce true division on every entry of the block?  flag |= 1 if not
__global__ void __launch_bounds__(kCloudCols) k_cloud_verify_div(int nloc, int m, const CloudGeom c, unsigned int* flag)
{
    const int j = blockIdx.x * kCloudCols + threadIdx.x;
    bool bad = false;
    if (j < m) {
        const double* yj = c.Y + (size_t)j * c.d;
        for (int i = blockIdx.y; i < nloc; i += gridDim.y) {
            const double s = cloud_sqdist(c.X + (size_t)i * c.d, yj, c.d);
            const double q = cloud_div_fast(s, c.cmax, c.inv_cmax), e = __ddiv_rn(s, c.cmax);
            bad |= __double_as_longlong(q) != __double_as_longlong(e);
        }
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

__global__ void __launch_bounds__(kCloudCols) k_cloud_materialize(int nloc, int m, long ld, const CloudGeom c,
                                                                  double* __restrict__ M)
{
    const int j = blockIdx.x * kCloudCols + threadIdx.x;
    if (j >= m) return;
    const double* yj = c.Y + (size_t)j * c.d;
    for (int i = blockIdx.y; i < nloc; i += gridDim.y)
        M[(size_t)i * ld + j] = cloud_div(cloud_sqdist(c.X + (size_t)i * c.d, yj, c.d), c);
}

void set_pointcloud(regot_ctx* ctx, int64_t n, int64_t m, int64_t row_begin, int64_t row_count, int d, const double* X,
                    const double* Y, const double* a, const double* b, double eta, bool on_the_fly)
{
    check_shape(n, m, row_begin, row_count, eta);
    if (!X || !Y || !a || !b) raise(REGOT_E_VALIDATION, "problem: null input");
    if (d < 1 || d > 4096) raise(REGOT_E_VALIDATION, "set_pointcloud: need 1 <= d <= 4096");
    if (on_the_fly && d > kCloudMaxD)
        raise(REGOT_E_UNSUPPORTED, "set_pointcloud: on-the-fly cost supports d <= " + std::to_string(kCloudMaxD) +
                                       " (a panel of target points must fit in shared memory); materialise instead");
    for (int64_t q = row_begin * d; q < (row_begin + row_count) * d; ++q)
        if (!std::isfinite(X[q])) raise(REGOT_E_VALIDATION, "problem: non-finite entries");
    for (int64_t q = 0; q < m * d; ++q)
        if (!std::isfinite(Y[q])) raise(REGOT_E_VALIDATION, "problem: non-finite entries");
    RG_CUDA(cudaSetDevice(ctx->device));
    DeviceProblem& pr = ctx->prob;
    pr.loaded = false;
    pr.n = n;
    pr.m = m;
    pr.row_begin = row_begin;
    pr.nloc = row_count;
    pr.eta = eta;
    pr.cloud_d = d;
    pr.on_the_fly = on_the_fly;
    pr.X_own.ensure((size_t)pr.nloc * (size_t)d);
    pr.Y_own.ensure((size_t)m * (size_t)d);
    pr.a_own.ensure((size_t)pr.nloc);
    pr.b_own.ensure((size_t)m);
    pr.a = pr.a_own.p;
    pr.b = pr.b_own.p;
    cudaStream_t st = ctx->stream;
    RG_CUDA(cudaMemcpyAsync(pr.X_own.p, X + row_begin * d, sizeof(double) * (size_t)pr.nloc * (size_t)d, cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaMemcpyAsync(pr.Y_own.p, Y, sizeof(double) * (size_t)m * (size_t)d, cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaMemcpyAsync(pr.a_own.p, a + row_begin, sizeof(double) * (size_t)pr.nloc, cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaMemcpyAsync(pr.b_own.p, b, sizeof(double) * (size_t)m, cudaMemcpyHostToDevice, st));

    // exact maximum of the un-normalised cost (normalize_cost, problem.h:53-61), over all ranks
    CloudGeom c;
    c.X = pr.X_own.p;
    c.Y = pr.Y_own.p;
    c.d = d;
    c.cmax = 1.0;
    c.inv_cmax = 1.0;
    c.fast_div = 0;
    const dim3 grid((unsigned)((m + kCloudCols - 1) / kCloudCols),
                    (unsigned)std::max<int64_t>(1, std::min<int64_t>(pr.nloc, 8L * ctx->sm_count)));
    DevBuf<double> bm;
    const size_t nb = (size_t)grid.x * grid.y;
    bm.ensure(nb + 1);
    k_cloud_max<<<grid, kCloudCols, 0, st>>>((int)pr.nloc, (int)m, c, bm.p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
    std::vector<double> hb(nb);
    RG_CUDA(cudaMemcpyAsync(hb.data(), bm.p, sizeof(double) * nb, cudaMemcpyDeviceToHost, st));
    RG_CUDA(cudaStreamSynchronize(st));
    double cmax = 0.0;
    for (double v : hb) cmax = std::max(cmax, v);
    if (ctx->sharded) {
        RG_CUDA(cudaMemcpyAsync(bm.p, &cmax, sizeof(double), cudaMemcpyHostToDevice, st));
        allreduce_max(ctx, ctx->comm, bm.p, 1, st);
        RG_CUDA(cudaMemcpyAsync(&cmax, bm.p, sizeof(double), cudaMemcpyDeviceToHost, st));
        RG_CUDA(cudaStreamSynchronize(st));
    }
    if (!(cmax > 0.0)) raise(REGOT_E_DEGENERATE_COST, "normalize_cost: no strictly positive entry");
    pr.cloud_max = cmax;
    c.cmax = cmax;
    c.inv_cmax = 1.0 / cmax;
    c.fast_div = 0;
    {   // the fast division is used only if it equals true division on every entry of this block
        DevBuf<unsigned int> flag;
        flag.ensure(1);
        RG_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(unsigned int), st));
        k_cloud_verify_div<<<grid, kCloudCols, 0, st>>>((int)pr.nloc, (int)m, c, flag.p);
        RG_CUDA(cudaGetLastError());
        ++ctx->launches;
        unsigned int bad = 1;
        RG_CUDA(cudaMemcpyAsync(&bad, flag.p, sizeof(bad), cudaMemcpyDeviceToHost, st));
        RG_CUDA(cudaStreamSynchronize(st));
        pr.cloud_fast_div = (bad == 0) && std::getenv("REGOT_B200_CLOUD_EXACT_DIV") == nullptr;
        c.fast_div = pr.cloud_fast_div ? 1 : 0;
    }
    if (on_the_fly) {
        pr.M_own.release();
        pr.M = nullptr;
        pr.ld = 0;
    } else {
        pr.ld = (m + 15) / 16 * 16;
        pr.M_own.ensure((size_t)pr.nloc * (size_t)pr.ld);
        pr.M = pr.M_own.p;
        RG_CUDA(cudaMemsetAsync(pr.M_own.p, 0, sizeof(double) * (size_t)pr.nloc * (size_t)pr.ld, st));
        k_cloud_materialize<<<grid, kCloudCols, 0, st>>>((int)pr.nloc, (int)m, (long)pr.ld, c, pr.M_own.p);
        RG_CUDA(cudaGetLastError());
        ++ctx->launches;
        RG_CUDA(cudaStreamSynchronize(st));
    }
    finish_problem(ctx);
}

// the cost block of this rank, row-major nloc x m, to the host (formed on the fly if it is not resident)
void get_cost_host(regot_ctx* ctx, double* out)
{
    const DeviceProblem& pr = ctx->prob;
    cudaStream_t st = ctx->stream;
    if (!pr.on_the_fly) {
        RG_CUDA(cudaMemcpy2DAsync(out, (size_t)pr.m * 8, pr.M, (size_t)pr.ld * 8, (size_t)pr.m * 8, (size_t)pr.nloc,
                                  cudaMemcpyDeviceToHost, st));
        RG_CUDA(cudaStreamSynchronize(st));
        return;
    }
    DevBuf<double> tmp;
    tmp.ensure((size_t)pr.nloc * (size_t)pr.m);
    const dim3 grid((unsigned)((pr.m + kCloudCols - 1) / kCloudCols),
                    (unsigned)std::max<int64_t>(1, std::min<int64_t>(pr.nloc, 8L * ctx->sm_count)));
    k_cloud_materialize<<<grid, kCloudCols, 0, st>>>((int)pr.nloc, (int)pr.m, (long)pr.m, cloud_geom(ctx), tmp.p);
    RG_CUDA(cudaGetLastError());
    ++ctx->launches;
    RG_CUDA(cudaMemcpyAsync(out, tmp.p, sizeof(double) * (size_t)pr.nloc * (size_t)pr.m, cudaMemcpyDeviceToHost, st));
    RG_CUDA(cudaStreamSynchronize(st));
}

// ---- host <-> device vectors ---------------------------------------------------------------------
void upload_dual(regot_ctx* ctx, const double* alpha_host, const double* beta_host, DVec& x, bool check_gauge,
                 const char* who)
{
    const DeviceProblem& pr = ctx->prob;
    if (!alpha_host || !beta_host) raise(REGOT_E_VALIDATION, std::string(who) + ": null dual point");
    // dual.h:72-78: the gauge is part of every entry point's contract
    if (check_gauge && beta_host[pr.m - 1] != 0.0)
        raise(REGOT_E_VALIDATION, std::string(who) + ": gauge violated, beta[m-1] must be 0");
    x.ensure(pr.nloc, pr.m);
    RG_CUDA(cudaMemcpyAsync(x.a.p, alpha_host + pr.row_begin, sizeof(double) * (size_t)pr.nloc, cudaMemcpyHostToDevice,
                            ctx->stream));
    RG_CUDA(cudaMemcpyAsync(x.b.p, beta_host, sizeof(double) * (size_t)pr.m, cudaMemcpyHostToDevice, ctx->stream));
}

}  // namespace rg

// ---- validate_problem (problem.h:30-50) on the resident instance -----------------------------------
namespace rg {

__global__ void k_count_nonfinite(int nloc, int m, long ld, const double* __restrict__ M, unsigned int* flag)
{
    const long total = (long)nloc * m;
    unsigned int bad = 0;
    for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (long)gridDim.x * blockDim.x) {
        const double v = M[(size_t)(q / m) * ld + (q % m)];
        bad |= isfinite(v) ? 0u : 1u;
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

void validate_problem_device(regot_ctx* ctx)
{
    const DeviceProblem& pr = ctx->prob;
    std::vector<double> a((size_t)pr.nloc), b((size_t)pr.m);
    RG_CUDA(cudaMemcpy(a.data(), pr.a, sizeof(double) * a.size(), cudaMemcpyDeviceToHost));
    RG_CUDA(cudaMemcpy(b.data(), pr.b, sizeof(double) * b.size(), cudaMemcpyDeviceToHost));
    DevBuf<unsigned int> flag;
    flag.ensure(1);
    RG_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(unsigned int), ctx->stream));
    if (!pr.on_the_fly) {  // point clouds were checked at upload
        k_count_nonfinite<<<4 * ctx->sm_count, 256, 0, ctx->stream>>>((int)pr.nloc, (int)pr.m, (long)pr.ld, pr.M, flag.p);
        RG_CUDA(cudaGetLastError());
        ++ctx->launches;
    }
    unsigned int bad = 0;
    RG_CUDA(cudaMemcpyAsync(&bad, flag.p, sizeof(bad), cudaMemcpyDeviceToHost, ctx->stream));
    RG_CUDA(cudaStreamSynchronize(ctx->stream));
    double sa = 0.0, sb = 0.0, mina = INFINITY, minb = INFINITY;
    bool fin = bad == 0;
    for (double v : a) { fin &= std::isfinite(v); sa += v; mina = std::min(mina, v); }
    for (double v : b) { fin &= std::isfinite(v); sb += v; minb = std::min(minb, v); }
    if (!fin) raise(REGOT_E_VALIDATION, "problem: non-finite entries");
    if (!(mina > 0.0)) raise(REGOT_E_VALIDATION, "problem: a must be elementwise positive");
    if (!(minb > 0.0)) raise(REGOT_E_VALIDATION, "problem: b must be elementwise positive");
    if (ctx->sharded) {
        // the row block only holds part of a: sum the pieces
        DevBuf<double> s;
        s.ensure(1);
        RG_CUDA(cudaMemcpy(s.p, &sa, sizeof(double), cudaMemcpyHostToDevice));
        allreduce_sum(ctx, ctx->comm, s.p, 1, ctx->stream);
        RG_CUDA(cudaMemcpyAsync(&sa, s.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        RG_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    if (std::fabs(sa - 1.0) > 1e-12) raise(REGOT_E_VALIDATION, "problem: a must sum to 1 within 1e-12");
    if (std::fabs(sb - 1.0) > 1e-12) raise(REGOT_E_VALIDATION, "problem: b must sum to 1 within 1e-12");
}

}  // namespace rg
