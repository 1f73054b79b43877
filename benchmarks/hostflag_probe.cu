// hostflag_probe.cu -- round trip host -> GPU -> host through pinned, device-mapped memory: the host
// writes a flag that a spinning GPU thread polls, the GPU answers into another host word that the host
// polls.  This is the signalling path of the lingering frame kernel (cbtm_update_linger).
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k(volatile int64_t *req, volatile int64_t *ack, int iters)
{
    for (int i = 1; i <= iters; ++i) {
        while (*req < i) { }
        *ack = i;
        __threadfence_system();
    }
}

int main()
{
    int64_t *h;
    cudaHostAlloc(&h, 4096, cudaHostAllocMapped);
    volatile int64_t *req = h, *ack = h + 64;
    *req = 0; *ack = 0;
    const int iters = 20000;
    k<<<1, 1>>>(req, ack, iters);
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 1; i <= iters; ++i) {
        *req = i;
        while (*ack < i) { }
    }
    auto t1 = std::chrono::steady_clock::now();
    cudaDeviceSynchronize();
    printf("host -> GPU (polling mapped host memory) -> host: %.2f us per round trip\n",
           std::chrono::duration<double, std::micro>(t1 - t0).count() / iters);
    // launch + completion of an empty kernel for comparison
    auto t2 = std::chrono::steady_clock::now();
    for (int i = 0; i < 2000; ++i) { k<<<1, 1>>>(req, ack, 0); cudaStreamSynchronize(0); }
    auto t3 = std::chrono::steady_clock::now();
    printf("launch + stream synchronise of an empty kernel: %.2f us\n", std::chrono::duration<double, std::micro>(t3 - t2).count() / 2000);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
