// tile_load_probe.cu -- how long does it take to get one 16 KB tile per CTA from L2 (warm) or DRAM
// (cold) into the SM, for every tile of a 2 / 8 / 32 MB bitfield at once (one CTA per tile, like
// k_sum_reduce at up to 2^26 leaves)?  Three ways to fetch:
//   tma   one cp.async.bulk of 16 KB per CTA + mbarrier, then 4 LDS.128 per thread
//   ldg   4 coalesced LDG.128 per thread (thread t reads 16-byte words t, t+256, t+512, t+768)
//   ldg64 4 LDG.128 per thread over 64 contiguous bytes (the layout k_sum_reduce's tree wants)
//   l256  2 LDG.256 per thread over 64 contiguous bytes
//   l256c 2 coalesced LDG.256 per thread (lane l reads 32 bytes at 32 * (256 j + t))
//   pf+l256  one bulk prefetch into L2 per CTA, a 2 us spin, then l256 (timed from the end of the spin:
//            does the prefetch make the loads L2 hits?)   spin+l256: the same without the prefetch
// Reported: us from the first CTA's entry to the latest "tile counted" stamp (%globaltimer), and
// the median CTA's entry -> counted time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tile_load_probe benchmarks/tile_load_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long now()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t popc128(uint4 v) { return __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w); }

__device__ __forceinline__ void ldg256(const void *p, uint32_t *v)
{
    asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "l"(p)
                 : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(256) k_load(const uint8_t *bits, uint32_t *out, unsigned long long *stamps)
{
    __shared__ __align__(128) uint8_t tile[16384];
    __shared__ __align__(8) uint64_t bar;
    const int t = threadIdx.x;
    const uint8_t *src = bits + (size_t)blockIdx.x * 16384;
    if (MODE >= 5) { // prefetch (5) or not (6), spin 2 us, then the timed part
        if (MODE == 5 && t == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(16384) : "memory");
        const unsigned long long t0 = now();
        while (now() - t0 < 2000) { }
        __syncthreads();
    }
    if (t == 0) stamps[2 * blockIdx.x] = now();
    uint32_t c = 0;
    if (MODE == 0) {
        if (t == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(16384) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             smem_u32(tile)), "l"(src), "r"(16384), "r"(smem_u32(&bar)) : "memory");
        }
        __syncthreads();
        asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@p bra D;\nbra W;\nD:\n}\n" ::"r"(smem_u32(&bar)) : "memory");
        const uint4 *mine = reinterpret_cast<const uint4 *>(tile) + t * 4;
#pragma unroll
        for (int j = 0; j < 4; ++j) c += popc128(mine[(j + ((t & 31) >> 1)) & 3]);
    } else if (MODE == 1) {
        const uint4 *p = reinterpret_cast<const uint4 *>(src);
        uint4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = __ldcg(p + j * 256 + t);
#pragma unroll
        for (int j = 0; j < 4; ++j) c += popc128(v[j]);
    } else if (MODE == 2) {
        const uint4 *p = reinterpret_cast<const uint4 *>(src) + t * 4;
        uint4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = __ldcg(p + j);
#pragma unroll
        for (int j = 0; j < 4; ++j) c += popc128(v[j]);
    } else if (MODE == 4) {
        uint32_t w[16];
        ldg256(src + t * 32, w);
        ldg256(src + 8192 + t * 32, w + 8);
#pragma unroll
        for (int j = 0; j < 16; ++j) c += __popc(w[j]);
    } else {
        uint32_t w[16];
        ldg256(src + t * 64, w);
        ldg256(src + t * 64 + 32, w + 8);
#pragma unroll
        for (int j = 0; j < 16; ++j) c += __popc(w[j]);
    }
    c += __shfl_xor_sync(0xffffffffu, c, 1);
    if ((t & 1) == 0) out[blockIdx.x * 128 + (t >> 1)] = c;
    __syncthreads();
    if (t == 0) stamps[2 * blockIdx.x + 1] = now();
}

__global__ void k_flush(uint4 *p, size_t n)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(1, 2, 3, 4);
}

int main()
{
    const size_t max_bytes = 32u << 20;
    uint8_t *bits;
    uint32_t *out;
    unsigned long long *stamps;
    uint4 *flush;
    const size_t flush_n = (512u << 20) / 16;
    cudaMalloc(&bits, max_bytes);
    cudaMemset(bits, 0x5a, max_bytes);
    cudaMalloc(&out, max_bytes / 128 * 4);
    cudaMalloc(&stamps, sizeof(unsigned long long) * 2 * 2048);
    cudaMalloc(&flush, flush_n * 16);
    std::vector<unsigned long long> h(2 * 2048);
    const char *names[7] = {"tma  ", "ldg  ", "ldg64", "l256 ", "l256c", "pf+l256", "spin+l256"};
    for (size_t mb : {2, 8, 32}) {
        const unsigned tiles = (unsigned)((mb << 20) / 16384);
        for (int warm = 1; warm >= 0; --warm)
            for (int mode = 0; mode < 7; ++mode) {
                std::vector<double> span, med;
                for (int rep = 0; rep < 7; ++rep) {
                    if (!warm) k_flush<<<1184, 256>>>(flush, flush_n);
                    else k_load<1><<<tiles, 256>>>(bits, out, stamps); // pull the bitfield into L2
                    cudaDeviceSynchronize();
                    if (mode == 0) k_load<0><<<tiles, 256>>>(bits, out, stamps);
                    else if (mode == 1) k_load<1><<<tiles, 256>>>(bits, out, stamps);
                    else if (mode == 2) k_load<2><<<tiles, 256>>>(bits, out, stamps);
                    else if (mode == 3) k_load<3><<<tiles, 256>>>(bits, out, stamps);
                    else if (mode == 4) k_load<4><<<tiles, 256>>>(bits, out, stamps);
                    else if (mode == 5) k_load<5><<<tiles, 256>>>(bits, out, stamps);
                    else k_load<6><<<tiles, 256>>>(bits, out, stamps);
                    cudaDeviceSynchronize();
                    cudaMemcpy(h.data(), stamps, sizeof(unsigned long long) * 2 * tiles, cudaMemcpyDeviceToHost);
                    unsigned long long t0 = ~0ull, t1 = 0;
                    std::vector<double> per;
                    for (unsigned b = 0; b < tiles; ++b) {
                        t0 = std::min(t0, h[2 * b]);
                        t1 = std::max(t1, h[2 * b + 1]);
                        per.push_back((double)(h[2 * b + 1] - h[2 * b]) / 1e3);
                    }
                    std::sort(per.begin(), per.end());
                    if (rep >= 2) span.push_back((double)(t1 - t0) / 1e3), med.push_back(per[per.size() / 2]);
                }
                std::sort(span.begin(), span.end());
                std::sort(med.begin(), med.end());
                printf("%2zu MB %s %s: first entry -> last counted %.2f us (%.2f TB/s), median CTA %.2f us\n", mb,
                       warm ? "L2  " : "DRAM", names[mode], span[span.size() / 2], (double)(mb << 20) / span[span.size() / 2] / 1e6,
                       med[med.size() / 2]);
            }
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
    return 0;
}
