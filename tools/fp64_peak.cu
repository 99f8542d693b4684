// fp64_peak.cu -- measures the vector fp64 FMA throughput and latency of the
// device (the second ceiling of the fused gradient pass).  Not in
// MEASURED_PEAKS.json, so measured here.  Build: see tools/Makefile.
#include <cuda_runtime.h>
#include <cstdio>

template <int ILP>
__global__ void k_dfma(double* out, int iters, double a, double b)
{
    double v[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) v[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < ILP; ++k) v[k] = fma(v[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += v[k];
    if (s == 123.456) out[0] = s;
}

__global__ void k_latency(double* out, long long* cycles, int iters, double a, double b)
{
    double v = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) v = fma(v, a, b);
    long long t1 = clock64();
    if (threadIdx.x == 0) cycles[0] = t1 - t0;
    if (v == 123.456) out[0] = v;
}

int main()
{
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    double* out;
    long long* cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int warps : {4, 8, 16, 32}) {
        const int blocks = p.multiProcessorCount * (warps >= 32 ? 2 : 1);
        const int threads = (warps >= 32 ? 16 : warps) * 32;
        k_dfma<8><<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        k_dfma<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fma_count = (double)blocks * threads * 8.0 * iters;
        std::printf("warps/SM %2d ILP 8: %.2f TFLOP/s fp64 (%.1f DFMA/clk/SM at %d MHz nominal)\n", warps,
                    2.0 * fma_count / ms * 1e-9, fma_count / (ms * 1e-3) / p.multiProcessorCount / (p.clockRate * 1e3),
                    p.clockRate / 1000);
    }
    k_latency<<<1, 32>>>(out, cyc, 10000, 1.0000001, 1e-9);
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    std::printf("DFMA dependent-chain latency: %.2f cycles\n", (double)c / 10000);
    std::printf("device %s, %d SMs\n", p.name, p.multiProcessorCount);
    return 0;
}
