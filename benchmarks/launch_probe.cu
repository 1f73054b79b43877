// launch_probe.cu -- what one frame's launch path costs on this system, by mechanism.
// A stand-in for the frame kernel (296 CTAs x 256 threads, six grid barriers, ~36 us of
// spinning, result written into host-mapped memory) is launched K times; after each launch
// the host polls the result word.  Reported: time per iteration minus the kernel's own
// duration = launch call + start latency + completion signalling.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/launch_probe benchmarks/launch_probe.cu
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

struct BigArgs { double prm[23]; void *p[40]; long long seq; int spin_ns; int coop; };

__device__ __forceinline__ unsigned long long gns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(256) k_frame(const BigArgs a, volatile long long *ring, volatile long long *out)
{
    const unsigned long long t0 = gns();
    long long seq = a.seq;
    if (seq < 0) seq = ring[0];                // graph mode: the request number comes from mapped host memory
    if (a.coop) {
        cg::grid_group g = cg::this_grid();
        for (int i = 0; i < 6; ++i) {
            while (gns() - t0 < (unsigned long long)a.spin_ns * (i + 1) / 6) { }
            g.sync();
        }
    } else {
        while (gns() - t0 < (unsigned long long)a.spin_ns) { }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        out[1] = (long long)(gns() - t0);
        __threadfence_system();
        out[0] = seq;
    }
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

int main()
{
    long long *h;
    CK(cudaHostAlloc(&h, 4096, cudaHostAllocMapped));
    volatile long long *out = h, *ring = h + 64;
    out[0] = 0;
    const int K = 2000, grid = 296;
    BigArgs a = {};
    a.spin_ns = 36000;
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    auto run = [&](const char *name, int mode) -> int {
        double kernel_us = 0;
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        if (mode == 3 || mode == 4) {
            BigArgs g = a;
            g.seq = -1;
            g.coop = mode == 3;
            CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
            if (g.coop) {
                void *args[] = {&g, (void *)&ring, (void *)&out};
                CK(cudaLaunchCooperativeKernel((const void *)k_frame, dim3(grid), dim3(256), args, 0, st));
            } else {
                k_frame<<<grid, 256, 0, st>>>(g, ring, out);
            }
            CK(cudaStreamEndCapture(st, &graph));
            CK(cudaGraphInstantiate(&exec, graph, 0));
        }
        long long base = out[0];
        auto t0 = std::chrono::steady_clock::now();
        double call_us = 0;
        for (int i = 1; i <= K; ++i) {
            a.seq = base + i;
            auto c0 = std::chrono::steady_clock::now();
            if (mode == 0) {
                a.coop = 1;
                void *args[] = {&a, (void *)&ring, (void *)&out};
                CK(cudaLaunchCooperativeKernel((const void *)k_frame, dim3(grid), dim3(256), args, 0, st));
            } else if (mode == 1) {
                a.coop = 0;
                k_frame<<<grid, 256, 0, st>>>(a, ring, out);
            } else if (mode == 2) {
                a.coop = 1;
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(grid), cfg.blockDim = dim3(256), cfg.stream = st;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeCooperative;
                at[0].val.cooperative = 1;
                cfg.attrs = at, cfg.numAttrs = 1;
                CK(cudaLaunchKernelEx(&cfg, k_frame, a, ring, out));
            } else {
                ring[0] = base + i;
                CK(cudaGraphLaunch(exec, st));
            }
            auto c1 = std::chrono::steady_clock::now();
            call_us += std::chrono::duration<double, std::micro>(c1 - c0).count();
            while (out[0] < base + i) { }
            kernel_us += out[1] / 1e3;
        }
        auto t1 = std::chrono::steady_clock::now();
        CK(cudaStreamSynchronize(st));
        const double per = std::chrono::duration<double, std::micro>(t1 - t0).count() / K;
        printf("%-44s %6.1f us/iter, kernel %5.1f us, overhead %5.1f us (launch call %4.1f us)\n", name, per,
               kernel_us / K, per - kernel_us / K, call_us / K);
        return 0;
    };
    // the same launch call while the previous kernel is still running (queued, no host wait)
    for (int coop = 0; coop < 2; ++coop) {
        a.coop = coop;
        a.spin_ns = 36000;
        CK(cudaStreamSynchronize(st));
        double call_us = 0;
        const int Q = 64;
        for (int i = 0; i < Q; ++i) {
            a.seq = 1;
            auto c0 = std::chrono::steady_clock::now();
            if (coop) {
                void *args[] = {&a, (void *)&ring, (void *)&out};
                CK(cudaLaunchCooperativeKernel((const void *)k_frame, dim3(grid), dim3(256), args, 0, st));
            } else {
                k_frame<<<grid, 256, 0, st>>>(a, ring, out);
            }
            call_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - c0).count();
        }
        CK(cudaStreamSynchronize(st));
        printf("%-44s launch call %4.1f us while the previous kernel runs (%d queued)\n",
               coop ? "cudaLaunchCooperativeKernel, queued" : "plain <<<>>>, queued", call_us / Q, Q);
    }
    for (int rep = 0; rep < 1; ++rep) {
        if (run("cudaLaunchCooperativeKernel", 0)) return 1;
        if (run("plain <<<>>> (no grid barriers)", 1)) return 1;
        if (run("cudaLaunchKernelEx + cooperative attribute", 2)) return 1;
        if (run("graph launch, cooperative node, mapped ring", 3)) return 1;
        if (run("graph launch, plain node, mapped ring", 4)) return 1;
    }
    return 0;
}
