// dsmem_probe.cu -- checks the exchange primitive of the block-resident PCG kernel in isolation: remote shared-memory
// stores that complete on the receiver's mbarrier (st.async ... mbarrier::complete_tx::bytes) inside a thread-block
// cluster, including completions that land before the receiver has armed the barrier, over many rounds.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_probe dsmem_probe.cu && ./dsmem_probe [cluster=8] [rounds=1000] [vec=1]
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t map_rank(uint32_t a, int r)
{
    uint32_t d;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(r));
    return d;
}

template <int kVec>
__global__ void __launch_bounds__(128) k_probe(int rounds, double* out, long long* cycles)
{
    __shared__ __align__(16) double inbox[16 * 128 * 2];
    __shared__ uint64_t mbar;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank(), n = (int)cl.num_blocks(), tid = threadIdx.x;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    cl.sync();
    uint32_t parity = 0;
    double acc = 0.0;
    const long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
        // everybody sends (r, rank, tid) to everybody
        for (int dst = 0; dst < n; ++dst) {
            const uint32_t ra = map_rank(smem_u32(inbox + (rank * 128 + tid) * 2), dst), rm = map_rank(smem_u32(&mbar), dst);
            const double a = (double)(r + rank + tid), b = (double)(r * 2 + tid);
            if (kVec)
                asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(ra),
                             "l"(__double_as_longlong(a)), "l"(__double_as_longlong(b)), "r"(rm) : "memory");
            else {
                asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra),
                             "l"(__double_as_longlong(a)), "r"(rm) : "memory");
                asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra + 8),
                             "l"(__double_as_longlong(b)), "r"(rm) : "memory");
            }
        }
        if ((r & 3) == rank % 4) __nanosleep(2000);  // some receivers arm late: completions arrive first
        if (tid == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(n * 128 * 16) : "memory");
        uint32_t ok;
        do {
            asm volatile("{ .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok) : "r"(smem_u32(&mbar)), "r"(parity) : "memory");
        } while (!ok);
        parity ^= 1u;
        for (int s = 0; s < n; ++s) acc += inbox[(s * 128 + tid) * 2] + inbox[(s * 128 + tid) * 2 + 1];
        // nobody may overwrite my inbox for round r + 1 before I have read round r
        cl.sync();
    }
    const long long t1 = clock64();
    cl.sync();
    out[(size_t)blockIdx.x * 128 + tid] = acc;
    if (tid == 0) cycles[blockIdx.x] = t1 - t0;
}

int main(int argc, char** argv)
{
    const int csize = argc > 1 ? atoi(argv[1]) : 8, rounds = argc > 2 ? atoi(argv[2]) : 1000, vec = argc > 3 ? atoi(argv[3]) : 1;
    double* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(double) * csize * 128);
    cudaMalloc(&cyc, sizeof(long long) * csize);
    const void* fn = vec ? (const void*)k_probe<1> : (const void*)k_probe<0>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(csize);
    cfg.blockDim = dim3(128);
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = argc > 4 ? atoi(argv[4]) : 2;  // 1: without the cooperative attribute
    int r = rounds;
    void* args[] = {&r, &out, &cyc};
    cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
    printf("launch: %s\n", cudaGetErrorString(e));
    e = cudaDeviceSynchronize();
    printf("sync: %s\n", cudaGetErrorString(e));
    double h[16 * 128];
    long long hc[16];
    cudaMemcpy(h, out, sizeof(double) * csize * 128, cudaMemcpyDeviceToHost);
    cudaMemcpy(hc, cyc, sizeof(long long) * csize, cudaMemcpyDeviceToHost);
    // expected: sum over r, s of (r + s + tid) + (2 r + tid)
    int bad = 0;
    for (int b = 0; b < csize; ++b)
        for (int t = 0; t < 128; ++t) {
            double want = 0.0;
            for (int rr = 0; rr < rounds; ++rr)
                for (int s = 0; s < csize; ++s) want += (double)(rr + s + t) + (double)(rr * 2 + t);
            if (h[b * 128 + t] != want) ++bad;
        }
    printf("cluster %d, %d rounds, vec %d: %d wrong sums, %.0f cycles per round (incl. a cluster barrier)\n", csize, rounds, vec, bad,
           (double)hc[0] / rounds);
    return bad != 0;
}
