// cbtm_common.cuh -- shared device helpers and the storage geometry of the CBT.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/cbtm.h"

namespace cbtm {

constexpr unsigned FULL_MASK = 0xffffffffu;
constexpr int LEAF_LOG2 = CBTM_LEAF_BLOCK_LOG2;  // 1024 slots = one 128-byte line
constexpr int CHUNK = 256;                       // live ranks per frame-kernel CTA pass

// Storage geometry of a depth-D tree (see include/cbtm.h).
struct Geo {
    int depth;        // D
    int lc;           // deepest counter level: max(D - 10, 0)
    uint32_t nblocks; // leaf blocks = 1 << lc
    uint32_t span;    // slots per leaf block = min(N, 1024)
    uint64_t n;       // N = 2^D
};

__host__ __device__ inline Geo make_geo(int depth)
{
    Geo g;
    g.depth = depth;
    g.lc = depth > LEAF_LOG2 ? depth - LEAF_LOG2 : 0;
    g.nblocks = 1u << g.lc;
    g.n = (uint64_t)1 << depth;
    g.span = depth > LEAF_LOG2 ? (1u << LEAF_LOG2) : (uint32_t)g.n;
    return g;
}

__host__ __device__ inline size_t bitfield_words(int depth)
{
    const size_t w = ((size_t)1 << depth) / 64;
    return w < 16 ? 16 : w;
}

__host__ __device__ inline size_t counter_words(int depth)
{
    const int lc = depth > LEAF_LOG2 ? depth - LEAF_LOG2 : 0;
    return (size_t)2 << lc;
}

// ---- warp primitives ------------------------------------------------------

__device__ __forceinline__ uint32_t warp_sum(uint32_t v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
    return v;
}

__device__ __forceinline__ uint32_t warp_inclusive_scan(uint32_t v)
{
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t up = __shfl_up_sync(FULL_MASK, v, o);
        if (lane >= o) v += up;
    }
    return v;
}

// Inclusive scan across a CTA of NT threads (NT multiple of 32, <= 1024).
// `warp_totals` is shared scratch of >= 32 entries.  Returns the inclusive
// prefix of v; *block_total receives the CTA-wide sum.
template <int NT>
__device__ __forceinline__ uint32_t block_inclusive_scan(uint32_t v, uint32_t *warp_totals,
                                                         uint32_t *block_total)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = warp_inclusive_scan(v);
    if (lane == 31) warp_totals[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < NT / 32 ? warp_totals[lane] : 0;
        w = warp_inclusive_scan(w);
        warp_totals[lane] = w;
    }
    __syncthreads();
    if (warp > 0) incl += warp_totals[warp - 1];
    *block_total = warp_totals[NT / 32 - 1];
    __syncthreads(); // scratch may be reused by the caller right away
    return incl;
}

// ---- bit tricks -------------------------------------------------------------

// position of the k-th (0-based) set bit of x; requires k < popc(x)
__device__ __forceinline__ int select32(uint32_t x, int k)
{
    int pos = 0;
#pragma unroll
    for (int width = 16; width > 0; width >>= 1) {
        const uint32_t low = x & ((1u << width) - 1u);
        const int c = __popc(low);
        if (k >= c) {
            k -= c;
            x >>= width;
            pos += width;
        } else {
            x = low;
        }
    }
    return pos;
}

__device__ __forceinline__ int select64(uint64_t x, int k)
{
    const uint32_t lo = (uint32_t)x;
    const int c = __popc(lo);
    if (k < c) return select32(lo, k);
    return 32 + select32((uint32_t)(x >> 32), k - c);
}

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ int bit_length64(uint64_t x) { return 64 - __clzll((long long)x); }

// bisector.py:91-97
__device__ __forceinline__ int depth_of(uint64_t id, int rank) { return bit_length64(id) - 1 - rank; }

__device__ __forceinline__ int popc128(const uint4 &v)
{
    return __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
}

} // namespace cbtm
