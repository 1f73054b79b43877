// fp64_probe.cu -- latency of a dependent fp64 add / multiply chain and the per-SM throughput of
// independent ones on this GPU (the LOD classifier is a dependent fp64 chain: which of the two bounds it?)
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double *out, int iters, int mode)
{
    double x = threadIdx.x * 1e-3 + 1.0, y = 0.999;
    const long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (mode == 0) x = __dadd_rn(x, y);
        else x = __dmul_rn(x, y);
    }
    const long long c1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(c1 - c0) / iters;
    if (x == 12345.678) out[1] = x;
}

// 8 independent chains per thread, `warps` warps per SM
__global__ void k_tput(double *out, int iters)
{
    double x[8];
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    const long long c0 = clock64();
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __dadd_rn(x[k], 0.999);
    const long long c1 = clock64();
    double s = 0;
    for (int k = 0; k < 8; ++k) s += x[k];
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(c1 - c0);
    if (s == 12345.678) out[1] = s;
}

int main()
{
    double *out, h[2];
    cudaMalloc(&out, 16);
    for (int mode = 0; mode < 2; ++mode) {
        k_lat<<<1, 32>>>(out, 4096, mode);
        cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
        printf("dependent %s chain: %.1f clk per op\n", mode ? "DMUL" : "DADD", h[0]);
    }
    for (int threads : {32, 128, 256, 512, 1024}) {
        const int iters = 2048;
        k_tput<<<148, threads>>>(out, iters);
        cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
        const double ops = (double)threads * 8 * iters; // per SM
        printf("%4d threads/SM, 8 independent DADD chains each: %.1f fp64 ops per clk per SM\n", threads, ops / h[0]);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
