// latency_probe.cu -- what one dependent step costs on this GPU: the numbers the frame
// kernel's phase budget is made of.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/latency_probe benchmarks/latency_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// mode 0: plain ld, 1: ld.relaxed.gpu, 2: atomicOr(.,0) returning, 3: ld.global.cg
__global__ void k_chase(uint32_t *buf, int hops, int mode, unsigned long long *out, uint32_t *sink)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint32_t p = 0;
    const long long c0 = clock64();
    const unsigned long long t0 = gns();
    for (int i = 0; i < hops; ++i) {
        if (mode == 0) p = buf[p];
        else if (mode == 1) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(p) : "l"(buf + p) : "memory");
        else if (mode == 2) p = atomicOr(buf + p, 0u);
        else p = __ldcg(buf + p);
    }
    const unsigned long long t1 = gns();
    const long long c1 = clock64();
    out[0] = t1 - t0;
    out[1] = (unsigned long long)(c1 - c0);
    *sink = p;
}

// block scan of 256 threads, repeated
__global__ void k_scan(int iters, unsigned long long *out, uint32_t *sink)
{
    __shared__ uint32_t wt[32];
    uint32_t v = threadIdx.x;
    const unsigned long long t0 = gns();
    for (int i = 0; i < iters; ++i) {
        uint32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t u = __shfl_up_sync(0xffffffffu, x, o);
            if ((threadIdx.x & 31) >= o) x += u;
        }
        if ((threadIdx.x & 31) == 31) wt[threadIdx.x >> 5] = x;
        __syncthreads();
        if (threadIdx.x < 32) {
            uint32_t w = threadIdx.x < 8 ? wt[threadIdx.x] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t u = __shfl_up_sync(0xffffffffu, w, o);
                if (threadIdx.x >= o) w += u;
            }
            wt[threadIdx.x] = w;
        }
        __syncthreads();
        v = x + (threadIdx.x >= 32 ? wt[(threadIdx.x >> 5) - 1] : 0);
        __syncthreads();
    }
    const unsigned long long t1 = gns();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    if (v == 0xdeadbeef) *sink = v;
}

// producer/consumer flag ping-pong between two CTAs (store -> remote poll sees it -> store back)
__global__ void k_pingpong(volatile uint32_t *flags, int iters, unsigned long long *out)
{
    if (threadIdx.x != 0) return;
    const int me = blockIdx.x;
    const unsigned long long t0 = gns();
    for (int i = 1; i <= iters; ++i) {
        if (me == 0) {
            flags[0] = i;
            while (flags[32] != (uint32_t)i) { }
        } else if (me == gridDim.x - 1) {
            while (flags[0] != (uint32_t)i) { }
            flags[32] = i;
        }
    }
    const unsigned long long t1 = gns();
    if (me == 0) out[0] = t1 - t0;
}

// cost of reading %globaltimer (dependent reads) and of the warp-level tree descent used by the frame kernel
__global__ void k_timer(int iters, unsigned long long *out)
{
    if (threadIdx.x != 0) return;
    const long long c0 = clock64();
    unsigned long long acc = 0;
    for (int i = 0; i < iters; ++i) acc += gns();
    const long long c1 = clock64();
    out[0] = (unsigned long long)(c1 - c0);
    out[1] = acc;
}

__global__ void k_descent(const uint32_t *counters, int lc, uint32_t rank0, int reps, unsigned long long *out, uint32_t *sink)
{
    const int lane = threadIdx.x & 31;
    if (threadIdx.x >= 32) return;
    uint32_t acc = 0;
    const long long c0 = clock64();
    for (int r = 0; r < reps; ++r) {
        uint32_t rank = rank0 + 977u * r + (acc & 1u), idx = 0;
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
        acc += idx;
    }
    const long long c1 = clock64();
    if (lane == 0) out[0] = (unsigned long long)(c1 - c0);
    if (acc == 0xdeadbeef) *sink = acc;
}

int main()
{
    const size_t small_n = 1u << 20, big_n = 1u << 28; // 4 MB, 1 GB of u32
    uint32_t *small, *big, *sink;
    unsigned long long *out;
    cudaMalloc(&small, small_n * 4); cudaMalloc(&big, big_n * 4); cudaMalloc(&sink, 4); cudaMalloc(&out, 64);
    auto fill = [&](uint32_t *d, size_t n, size_t stride) {
        std::vector<uint32_t> h(n);
        // a permutation cycle with a large odd stride: every hop lands on another line / page
        for (size_t i = 0; i < n; ++i) h[i] = (uint32_t)((i + stride) % n);
        cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
    };
    fill(small, small_n, 40503);           // 4 MB: L2 resident
    fill(big, big_n, 40503 * 1031 + 64);   // 1 GB: DRAM + TLB misses
    const char *names[] = {"ld", "ld.relaxed.gpu", "atom.or (returning)", "ld.cg"};
    unsigned long long h[2];
    for (int which = 0; which < 2; ++which) {
        for (int mode = 0; mode < 4; ++mode) {
            const int hops = 2000;
            for (int r = 0; r < 2; ++r) k_chase<<<1, 32>>>(which ? big : small, hops, mode, out, sink);
            cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
            printf("%-5s %-22s %7.1f ns/hop  %7.1f clk/hop\n", which ? "1GB" : "4MB", names[mode], (double)h[0] / hops,
                   (double)h[1] / hops);
        }
    }
    for (int r = 0; r < 2; ++r) k_scan<<<1, 256>>>(1000, out, sink);
    cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
    printf("block scan (256 thr, 3 barriers) %7.1f ns\n", (double)h[0] / 1000);
    k_timer<<<1, 32>>>(1000, out);
    cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
    printf("%%globaltimer read: %7.1f clk each\n", (double)h[0] / 1000);
    {
        const int lc = 16;
        std::vector<uint32_t> heap(2u << lc, 0);
        for (uint32_t i = 0; i < (1u << lc); ++i) heap[(1u << lc) + i] = 512;
        for (uint32_t i = (1u << lc) - 1; i >= 1; --i) heap[i] = heap[2 * i] + heap[2 * i + 1];
        uint32_t *d;
        cudaMalloc(&d, heap.size() * 4);
        cudaMemcpy(d, heap.data(), heap.size() * 4, cudaMemcpyHostToDevice);
        for (int r = 0; r < 2; ++r) k_descent<<<1, 32>>>(d, lc, 12345u, 200, out, sink);
        cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
        printf("warp descent (16 levels, 4 steps): %7.1f clk each\n", (double)h[0] / 200);
    }
    uint32_t *flags;
    cudaMalloc(&flags, 256); cudaMemset(flags, 0, 256);
    for (int grid : {2, 148, 296}) {
        cudaMemset(flags, 0, 256);
        k_pingpong<<<grid, 32>>>(flags, 1000, out);
        cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
        printf("flag ping-pong CTA0 <-> CTA%d: %7.1f ns per round trip (2 one-way signals)\n", grid - 1, (double)h[0] / 1000);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
