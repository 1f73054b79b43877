// gridsync_probe3.cu -- a device-wide barrier through thread-block clusters: the CTAs of a cluster meet in
// the hardware cluster barrier, ONE thread per cluster arrives at / polls the global counter (37 .. 148
// arrivals instead of 296), then the cluster barrier releases the others.  Against cooperative_groups'
// grid.sync() at the frame kernel's shape (296 CTAs x 256 threads, 2 per SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gridsync_probe3 benchmarks/gridsync_probe3.cu
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release(unsigned *p)
{
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}

__global__ void __launch_bounds__(256, 2) k_cg(int iters, unsigned *bar)
{
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
}

// monotonic counter; clusters of any size (1 = plain CTAs)
__global__ void __launch_bounds__(256, 2) k_cluster(int iters, unsigned *bar, unsigned n_clusters)
{
    cg::cluster_group cl = cg::this_cluster();
    const bool leader = cl.block_rank() == 0 && threadIdx.x == 0;
    unsigned target = 0;
    for (int i = 0; i < iters; ++i) {
        target += n_clusters;
        cl.sync(); // everybody of the cluster has arrived (release / acquire at cluster scope)
        if (leader) {
            __threadfence();
            red_release(bar);
            while (ld_acquire(bar) < target) { }
            __threadfence();
        }
        cl.sync();
    }
}

template <typename... Args>
float launch(void *kernel, int grid, int cluster, Args... a)
{
    void *args[] = {(void *)&a...};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = cluster;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = cluster > 1 ? 2 : 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t rc = cudaLaunchKernelExC(&cfg, kernel, args);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = -1;
    if (rc == cudaSuccess && cudaGetLastError() == cudaSuccess) cudaEventElapsedTime(&ms, e0, e1);
    else printf("   launch failed: %s\n", cudaGetErrorString(rc));
    return ms;
}

int main()
{
    unsigned *bar;
    cudaMalloc(&bar, 4096);
    const int its[2] = {1, 2001};
    float t[2];
    for (int k = 0; k < 2; ++k) {
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            int iters = its[k];
            float ms = launch((void *)k_cg, 296, 1, iters, bar);
            best = ms < best ? ms : best;
        }
        t[k] = best;
    }
    printf("cooperative_groups grid.sync, 296 CTAs:      %6.3f us per barrier\n", (t[1] - t[0]) * 1e3 / 2000);
    for (int cluster : {1, 2, 4, 8}) {
        int grid = 296;
        // how many clusters of this size are co-resident?
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(256);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cluster;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int max_clusters = 0;
        if (cluster > 1) {
            cudaOccupancyMaxActiveClusters(&max_clusters, (void *)k_cluster, &cfg);
            if (max_clusters * cluster < grid) grid = max_clusters * cluster;
        }
        for (int k = 0; k < 2; ++k) {
            float best = 1e9;
            for (int r = 0; r < 5; ++r) {
                cudaMemset(bar, 0, 4096);
                int iters = its[k];
                unsigned n_clusters = grid / cluster;
                float ms = launch((void *)k_cluster, grid, cluster, iters, bar, n_clusters);
                if (ms < 0) { best = -1; break; }
                best = ms < best ? ms : best;
            }
            t[k] = best;
        }
        printf("cluster barrier + counter, clusters of %d, %3d CTAs (max co-resident clusters %d): %6.3f us per barrier\n",
               cluster, grid, max_clusters, (t[1] - t[0]) * 1e3 / 2000);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
