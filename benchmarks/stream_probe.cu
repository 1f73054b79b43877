// stream_probe.cu -- calibration: what does a pure HBM *read* stream reach on this
// GPU for 128 MiB .. 1 GiB, and how much of a short kernel is fixed cost?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stream_probe benchmarks/stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void k_read(const uint4* __restrict__ p, size_t n, unsigned long long* out)
{
    unsigned acc = 0;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
        uint4 a, b, c, d;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(p + i));
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(p + i + stride));
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(c.x), "=r"(c.y), "=r"(c.z), "=r"(c.w) : "l"(p + i + 2 * stride));
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(d.x), "=r"(d.y), "=r"(d.z), "=r"(d.w) : "l"(p + i + 3 * stride));
        acc += a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
    }
    for (; i < n; i += stride) { uint4 a = p[i]; acc += a.x ^ a.y ^ a.z ^ a.w; }
    if (acc == 0x12345678u) atomicAdd(out, 1ull);
}
__global__ void k_touch(const uint4* __restrict__ p, size_t n, unsigned long long* out)
{
    unsigned acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) { uint4 a = p[i]; acc += a.x; }
    if (acc == 0x12345678u) atomicAdd(out, 1ull);
}
__global__ void k_write(uint4* __restrict__ p, size_t n)
{
    const uint4 v = make_uint4(1, 2, 3, 4);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void k_empty(unsigned long long* out) { if (threadIdx.x == 9999) *out = 1; }

int main()
{
    const size_t flush_bytes = 512ull << 20;
    uint4 *buf, *flush; unsigned long long* out;
    cudaMalloc(&buf, 1ull << 30); cudaMalloc(&flush, flush_bytes); cudaMalloc(&out, 8);
    cudaMemset(buf, 1, 1ull << 30); cudaMemset(flush, 2, flush_bytes);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char* name, size_t bytes, int grid, int block) {
        std::vector<float> ts;
        for (int r = 0; r < 12; ++r) {
            k_touch<<<1184, 256>>>(flush, flush_bytes / 16, out);   // clean L2 flush (reads)
            cudaEventRecord(a);
            if (bytes) k_read<<<grid, block>>>(buf, bytes / 16, out); else k_empty<<<1, 32>>>(out);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (r >= 2) ts.push_back(ms);
        }
        std::sort(ts.begin(), ts.end());
        const float med = ts[ts.size() / 2], mn = ts[0];
        printf("%-10s %7.1f MiB grid %5d x %4d : med %8.2f us  min %8.2f us  -> %7.1f GB/s (med)\n", name, bytes / 1048576.0, grid, block, med * 1e3, mn * 1e3, bytes ? bytes / (med * 1e-3) / 1e9 : 0.0);
    };
    run("empty", 0, 1, 32);
    for (size_t mb : {8, 32, 128, 512, 1024})
        for (int grid : {592, 1184, 2368, 4736})
            run("read", mb << 20, grid, 256);
    // pure WRITE streams: the ceiling for decode-all (4N bytes written, N/8 read)
    for (size_t mb : {256, 1024}) {
        for (int grid : {1184, 4736}) {
            std::vector<float> ts;
            for (int r = 0; r < 8; ++r) {
                k_touch<<<1184, 256>>>(flush, flush_bytes / 16, out);
                cudaEventRecord(a);
                k_write<<<grid, 256>>>(buf, (mb << 20) / 16);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b); if (r >= 2) ts.push_back(ms);
            }
            std::sort(ts.begin(), ts.end());
            printf("write      %7.1f MiB grid %5d x  256 : med %8.2f us -> %7.1f GB/s\n", (double)mb, grid, ts[ts.size() / 2] * 1e3, (mb << 20) / (ts[ts.size() / 2] * 1e-3) / 1e9);
        }
        std::vector<float> ts;
        for (int r = 0; r < 8; ++r) {
            k_touch<<<1184, 256>>>(flush, flush_bytes / 16, out);
            cudaEventRecord(a);
            cudaMemsetAsync(buf, 3, mb << 20);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (r >= 2) ts.push_back(ms);
        }
        std::sort(ts.begin(), ts.end());
        printf("memset     %7.1f MiB                   : med %8.2f us -> %7.1f GB/s\n", (double)mb, ts[ts.size() / 2] * 1e3, (mb << 20) / (ts[ts.size() / 2] * 1e-3) / 1e9);
    }
    run("read512t", 128ull << 20, 1184, 512);
    run("read1024t", 128ull << 20, 592, 1024);
    return 0;
}
