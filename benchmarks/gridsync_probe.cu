// gridsync_probe.cu -- cost of a cooperative-groups grid barrier on this GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gridsync_probe benchmarks/gridsync_probe.cu
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_sync(int iters, unsigned* sink)
{
    cg::grid_group g = cg::this_grid();
    unsigned acc = 0;
    for (int i = 0; i < iters; ++i) {
        acc += i;
        g.sync();
    }
    if (acc == 0xdeadbeef) *sink = acc;
}

// hand-rolled sense-reversing barrier: one arrive per CTA, spin on a generation word
__device__ __forceinline__ void grid_barrier(unsigned* count, volatile unsigned* gen, unsigned nblocks)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned my_gen = *gen;
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *count = 0;
            __threadfence();
            atomicAdd((unsigned*)gen, 1u);
        } else {
            while (*gen == my_gen) { }
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void k_sync_manual(int iters, unsigned* bar, unsigned* sink)
{
    unsigned acc = 0;
    for (int i = 0; i < iters; ++i) {
        acc += i;
        grid_barrier(bar, bar + 32, gridDim.x);
    }
    if (acc == 0xdeadbeef) *sink = acc;
}

int main()
{
    unsigned *sink, *bar;
    cudaMalloc(&sink, 4); cudaMalloc(&bar, 256); cudaMemset(bar, 0, 256);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int per_sm : {1, 2, 4}) {
        for (int iters : {1, 101}) {
            int grid = 148 * per_sm;
            void* args[] = {&iters, &sink};
            float best = 1e9;
            for (int r = 0; r < 5; ++r) {
                cudaEventRecord(a);
                cudaLaunchCooperativeKernel((void*)k_sync, dim3(grid), dim3(256), args, 0, 0);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
            }
            printf("cg   grid %4d iters %4d : %8.2f us total\n", grid, iters, best * 1e3);
            void* args2[] = {&iters, &bar, &sink};
            best = 1e9;
            for (int r = 0; r < 5; ++r) {
                cudaEventRecord(a);
                cudaLaunchCooperativeKernel((void*)k_sync_manual, dim3(grid), dim3(256), args2, 0, 0);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
            }
            printf("manual grid %4d iters %4d : %8.2f us total\n", grid, iters, best * 1e3);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
