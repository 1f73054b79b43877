// icache_probe2.cu -- cost of a short branchy routine (a 4-step warp descent over a counter heap)
// when its code is cold (evicted by 192 KB of other code in between) versus warm.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define OP x = x * 1664525u + y; y ^= x >> 3;
#define R4(a) a a a a
#define R16(a) R4(R4(a))
#define R64(a) R4(R16(a))
#define R256(a) R4(R64(a))
#define R1024(a) R4(R256(a))
__device__ __noinline__ uint32_t evict(uint32_t x, uint32_t y) { R1024(OP) R1024(OP) R1024(OP) return x ^ y; }

__device__ __noinline__ uint32_t descent(const uint32_t *counters, int lc, uint32_t rank)
{
    const int lane = threadIdx.x & 31;
    uint32_t idx = 0;
    int l = 0;
    while (l < lc) {
        const int s = lc - l < 5 ? lc - l : 5;
        const uint32_t fan = 1u << s;
        uint32_t z = 0;
        if ((uint32_t)lane < fan) z = counters[(1u << (l + s)) + (idx << s) + lane];
        uint32_t incl = z;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        const unsigned hit = __ballot_sync(0xffffffffu, (uint32_t)lane < fan && incl > rank);
        const int child = hit ? __ffs(hit) - 1 : (int)fan - 1;
        rank -= __shfl_sync(0xffffffffu, incl - z, child);
        idx = (idx << s) + child;
        l += s;
    }
    return idx;
}

__global__ void k(const uint32_t *counters, int lc, int do_evict, unsigned long long *out, uint32_t *sink)
{
    if (threadIdx.x >= 32) return;
    uint32_t acc = threadIdx.x;
    unsigned long long total = 0;
    for (int r = 0; r < 16; ++r) {
        if (do_evict) acc = evict(acc, r);
        const long long c0 = clock64();
        acc += descent(counters, lc, 12345u + 977u * r + (acc & 1u));
        const long long c1 = clock64();
        if (r >= 4) total += (unsigned long long)(c1 - c0);
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = total / 12;
    if (acc == 0xdeadbeef) *sink = acc;
}

int main()
{
    const int lc = 16;
    std::vector<uint32_t> heap(2u << lc, 0);
    for (uint32_t i = 0; i < (1u << lc); ++i) heap[(1u << lc) + i] = 512;
    for (uint32_t i = (1u << lc) - 1; i >= 1; --i) heap[i] = heap[2 * i] + heap[2 * i + 1];
    uint32_t *d, *sink;
    unsigned long long *out, h;
    cudaMalloc(&d, heap.size() * 4); cudaMalloc(&sink, 4); cudaMalloc(&out, 8);
    cudaMemcpy(d, heap.data(), heap.size() * 4, cudaMemcpyHostToDevice);
    for (int grid : {1, 296}) for (int ev : {0, 1}) {
        k<<<grid, 256>>>(d, lc, ev, out, sink);
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        printf("grid %3d  %s code: descent %6llu clk\n", grid, ev ? "COLD" : "warm", h);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
