// gridsync_probe2.cu -- how cheap can a device-wide barrier of 296 co-resident CTAs be?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gridsync_probe2 benchmarks/gridsync_probe2.cu
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned *bar, unsigned *sink)
{
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
}

// monotonic counter, no reset: arrive = one atomic, wait = poll until count >= target
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release(unsigned *p)
{
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}

__global__ void k_mono(int iters, unsigned *bar, unsigned *sink)
{
    unsigned target = 0;
    for (int i = 0; i < iters; ++i) {
        target += gridDim.x;
        __syncthreads();
        if (threadIdx.x == 0) {
            red_release(bar);
            while (ld_acquire(bar) < target) { }
        }
        __syncthreads();
    }
}

// every warp polls itself: no second CTA barrier
__global__ void k_mono_warp(int iters, unsigned *bar, unsigned *sink)
{
    unsigned target = 0;
    for (int i = 0; i < iters; ++i) {
        target += gridDim.x;
        __syncthreads();
        if (threadIdx.x == 0) red_release(bar);
        if ((threadIdx.x & 31) == 0)
            while (ld_acquire(bar) < target) { }
        __syncwarp();
    }
}

// arrivals spread over 8 counters (one per 37 CTAs), a last-arriver of each bumps a top counter
__global__ void k_tree(int iters, unsigned *bar, unsigned *sink)
{
    unsigned target_leaf = 0, target_top = 0;
    const unsigned groups = 8, per = (gridDim.x + groups - 1) / groups;
    const unsigned g = blockIdx.x / per;
    const unsigned in_group = (g == groups - 1) ? gridDim.x - per * (groups - 1) : per;
    for (int i = 0; i < iters; ++i) {
        target_leaf += in_group;
        target_top += groups;
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned old = atomicAdd(bar + 32 * (1 + g), 1u);
            if (old + 1 == target_leaf) {
                __threadfence();
                red_release(bar);
            }
            while (ld_acquire(bar) < target_top) { }
        }
        __syncthreads();
    }
}

template <typename K>
void run(const char *name, K kernel, int grid, unsigned *bar, unsigned *sink)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float t[2];
    int its[2] = {1, 1001};
    for (int k = 0; k < 2; ++k) {
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaMemset(bar, 0, 4096);
            int iters = its[k];
            void *args[] = {&iters, &bar, &sink};
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void *)kernel, dim3(grid), dim3(256), args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        t[k] = best;
    }
    printf("%-28s grid %4d: %6.3f us per barrier\n", name, grid, (t[1] - t[0]) * 1e3 / 1000);
}

int main()
{
    unsigned *sink, *bar;
    cudaMalloc(&sink, 4);
    cudaMalloc(&bar, 4096);
    for (int per_sm : {1, 2, 4}) {
        const int grid = 148 * per_sm;
        run("cooperative_groups", k_cg, grid, bar, sink);
        run("monotonic counter", k_mono, grid, bar, sink);
        run("monotonic, warps poll", k_mono_warp, grid, bar, sink);
        run("two-level tree", k_tree, grid, bar, sink);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
