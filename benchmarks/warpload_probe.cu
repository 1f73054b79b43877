// warpload_probe.cu -- latency of ONE warp-wide load of 32 consecutive 64-bit words (a look-back
// window) for the different load flavours: are strong / volatile accesses coalesced?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE> __device__ __forceinline__ uint64_t ld(const uint64_t *p)
{
    uint64_t v;
    if (MODE == 0) v = *p;
    else if (MODE == 1) asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else if (MODE == 2) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else if (MODE == 3) asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

template <int MODE>
__global__ void k(const uint64_t *buf, int iters, unsigned long long *out, uint64_t *sink)
{
    const int lane = threadIdx.x;
    uint64_t acc = 0;
    uint32_t pos = 1u << 16;
    const long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const uint64_t f = ld<MODE>(buf + pos - 1 - lane + (acc & 1));
        acc += f;
        // the next address depends on the loaded data (as in a look-back walk)
        acc = __shfl_xor_sync(0xffffffffu, acc, 1) + acc;
        pos -= 32;
    }
    const long long c1 = clock64();
    if (lane == 0) out[0] = (unsigned long long)(c1 - c0);
    if (acc == 0xdeadbeef) *sink = acc;
}

int main()
{
    uint64_t *buf, *sink;
    unsigned long long *out, h;
    cudaMalloc(&buf, 8 << 17); cudaMemset(buf, 0, 8 << 17); cudaMalloc(&sink, 8); cudaMalloc(&out, 8);
    const char *names[] = {"ld (weak)", "ld.cg", "ld.relaxed.gpu", "ld.volatile", "ld.acquire.gpu"};
    const int iters = 1000;
#define RUN(M) for (int r = 0; r < 2; ++r) k<M><<<1, 32>>>(buf, iters, out, sink); cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost); \
    printf("%-16s %7.1f clk per dependent warp-wide load (32 x u64)\n", names[M], (double)h / iters);
    RUN(0) RUN(1) RUN(2) RUN(3) RUN(4)
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
