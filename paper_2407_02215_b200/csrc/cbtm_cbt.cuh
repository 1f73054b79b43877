// cbtm_cbt.cuh -- the concurrent binary tree on a packed bitfield:
// sum reduction, ranked decode (k-th set / unset bit) and stream-compacted
// indexation.  Reference semantics: pkg/src/cbtmesh/cbt.py.
#pragma once

#include "cbtm_common.cuh"

namespace cbtm {

// ---------------------------------------------------------------------------
// Sum reduction (Cbt.sum_reduce, cbt.py:61-68; pipeline stage 9).
//
// One CTA reduces a tile of 2^17 slots (16 KB of bitfield = 128 leaf blocks):
// four independent 128-bit loads per thread, popcount, 8-lane shuffle to a
// leaf-block count, then seven tree levels in shared memory.  The 255 tile
// nodes are written level by level (coalesced).  The last CTA to finish
// (ticket) builds the levels above the tile roots in shared memory.
// HBM traffic: N/8 bytes read + 4 * (2 << Lc) = N/128 bytes written.
// ---------------------------------------------------------------------------
constexpr int RED_THREADS = 256;
constexpr int RED_LOADS = 4;
constexpr int RED_TILE_VEC = RED_THREADS * RED_LOADS; // uint4 per tile
constexpr int RED_TILE_BLOCKS = RED_TILE_VEC / 8;     // leaf blocks per tile = 128
constexpr int RED_TILE_LOG2 = 7;
constexpr int RED_UPPER_MAX = 4096; // tile roots handled in shared memory

__global__ void __launch_bounds__(RED_THREADS)
k_sum_reduce(const uint4 *__restrict__ bits, uint32_t *__restrict__ counters, int lc,
             uint32_t n_vec, unsigned *ticket, int64_t *live_after)
{
    __shared__ uint32_t tree[2 * RED_TILE_BLOCKS];
    __shared__ uint32_t upper[2 * RED_UPPER_MAX];
    __shared__ bool is_last;

    const int t = threadIdx.x;
    const uint32_t tile = blockIdx.x;

    uint4 v[RED_LOADS];
#pragma unroll
    for (int j = 0; j < RED_LOADS; ++j) {
        const uint32_t idx = tile * RED_TILE_VEC + j * RED_THREADS + t;
        v[j] = idx < n_vec ? ld_stream(bits + idx) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < RED_LOADS; ++j) {
        uint32_t c = popc128(v[j]);
        c += __shfl_xor_sync(FULL_MASK, c, 1);
        c += __shfl_xor_sync(FULL_MASK, c, 2);
        c += __shfl_xor_sync(FULL_MASK, c, 4);
        if ((t & 7) == 0) tree[RED_TILE_BLOCKS + j * (RED_THREADS / 8) + (t >> 3)] = c;
    }
    __syncthreads();
#pragma unroll
    for (int w = RED_TILE_BLOCKS / 2; w >= 1; w >>= 1) {
        if (t < w) tree[w + t] = tree[2 * (w + t)] + tree[2 * (w + t) + 1];
        __syncthreads();
    }
    // local heap node t (level ll, position pos) is global level lc - 7 + ll
    if (t >= 1) {
        const int ll = 31 - __clz(t);
        const uint32_t pos = t - (1u << ll);
        const int gl = lc - RED_TILE_LOG2 + ll;
        if (gl >= 0 && (gridDim.x > 1 || pos < (1u << gl))) {
            counters[(1u << gl) + tile * (1u << ll) + pos] = tree[t];
            if (gl == 0 && live_after) *live_after = tree[t];
        }
    }
    if (gridDim.x == 1) return;

    // ---- levels above the tile roots: last CTA standing ----
    __threadfence();
    __syncthreads();
    if (t == 0) is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!is_last) return;
    __threadfence();

    uint32_t cnt = gridDim.x; // nodes on the tile-root level, a power of two
    while (cnt > RED_UPPER_MAX) {
        const uint32_t half = cnt >> 1;
        for (uint32_t i = t; i < half; i += RED_THREADS)
            counters[half + i] = __ldcg(&counters[cnt + 2 * i]) + __ldcg(&counters[cnt + 2 * i + 1]);
        __syncthreads();
        cnt = half;
    }
    for (uint32_t i = t; i < cnt; i += RED_THREADS) upper[cnt + i] = __ldcg(&counters[cnt + i]);
    __syncthreads();
    for (uint32_t w = cnt >> 1; w >= 1; w >>= 1) {
        for (uint32_t i = t; i < w; i += RED_THREADS)
            upper[w + i] = upper[2 * (w + i)] + upper[2 * (w + i) + 1];
        __syncthreads();
    }
    for (uint32_t i = 1 + t; i < cnt; i += RED_THREADS) counters[i] = upper[i];
    if (t == 0) {
        *ticket = 0;
        if (live_after) *live_after = upper[1];
    }
}

// ---------------------------------------------------------------------------
// Ranked decode (one_to_bit_id / zero_to_bit_id, cbt.py:75-107 and 127-150):
// descent over the counter heap, then popcount select inside the 128-byte leaf
// block.
// ---------------------------------------------------------------------------
template <bool ONES>
__device__ __forceinline__ int32_t cbt_find(const uint64_t *__restrict__ bits,
                                            const uint32_t *__restrict__ counters,
                                            const Geo &g, uint32_t rank)
{
    uint32_t node = 1;
    uint32_t half = (uint32_t)(g.n >> 1); // slots under a child of the current node
    for (int l = 0; l < g.lc; ++l) {
        node <<= 1;
        const uint32_t ones = __ldg(&counters[node]);
        const uint32_t left = ONES ? ones : half - ones;
        if (rank >= left) {
            rank -= left;
            node += 1;
        }
        half >>= 1;
    }
    const uint32_t block = node - g.nblocks;
    const uint64_t *line = bits + (size_t)block * 16;
    const int words = g.span >= 64 ? (int)(g.span >> 6) : 1;
    for (int w = 0; w < words; ++w) {
        uint64_t x = __ldg(&line[w]);
        if (!ONES) {
            x = ~x;
            if (g.span < 64) x &= (((uint64_t)1 << g.span) - 1);
        }
        const uint32_t c = __popcll(x);
        if (rank < c) return (int32_t)(block * g.span + w * 64 + select64(x, (int)rank));
        rank -= c;
    }
    return -1; // rank out of range
}

template <bool ONES>
__global__ void __launch_bounds__(256)
k_decode(const uint64_t *__restrict__ bits, const uint32_t *__restrict__ counters, int depth,
         const int64_t *__restrict__ ranks, int64_t K, int32_t *__restrict__ out)
{
    const Geo g = make_geo(depth);
    const uint32_t ones = counters[1];
    const uint64_t limit = ONES ? (uint64_t)ones : g.n - ones;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < K;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = ranks ? ranks[i] : i;
        out[i] = (r < 0 || (uint64_t)r >= limit) ? -1 : cbt_find<ONES>(bits, counters, g, (uint32_t)r);
    }
}

// ---------------------------------------------------------------------------
// Indexation (pipeline stage 2, k_cache_pointers kernels.py:244-252) as a
// stream compaction.  One warp per 1024-slot leaf block:
//   * its rank offset comes from the counter heap (sum of the left siblings on
//     the root path -- all addresses known up front, one load per lane),
//   * the block's slots are expanded into a 4 KB shared staging area (set bits
//     from the front, unset bits behind them) and copied out coalesced.
// Blocks with no set bit are skipped without touching the bitfield when the
// free list is not requested.
// ---------------------------------------------------------------------------
constexpr int IDX_WARPS = 8;

__global__ void __launch_bounds__(IDX_WARPS * 32)
k_index(const uint32_t *__restrict__ bits32, const uint32_t *__restrict__ counters, int depth,
        int32_t *__restrict__ cache_live, int32_t *__restrict__ cache_free,
        uint32_t *__restrict__ dispatch)
{
    __shared__ int32_t stage[IDX_WARPS][1024];
    const Geo g = make_geo(depth);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t gwarp = blockIdx.x * IDX_WARPS + warp;
    const uint32_t nwarps = gridDim.x * IDX_WARPS;

    if (dispatch && blockIdx.x == 0 && threadIdx.x == 0) {
        const uint32_t n = counters[1];
        dispatch[0] = (n + CHUNK - 1) / CHUNK;
        dispatch[1] = 1;
        dispatch[2] = 1;
        dispatch[3] = n;
    }

    int32_t *st = stage[warp];
    for (uint32_t b = gwarp; b < g.nblocks; b += nwarps) {
        const uint32_t cnt = __ldg(&counters[g.nblocks + b]);
        if (cnt == 0 && !cache_free) continue;

        // ones before this block: left siblings along the root path
        uint32_t part = 0;
        if (lane >= 1 && lane <= g.lc) {
            const uint32_t idx = b >> (g.lc - lane);
            if (idx & 1) part = __ldg(&counters[(1u << lane) + idx - 1]);
        }
        const uint32_t ones_before = warp_sum(part);
        const uint32_t zeros_before = b * g.span - ones_before;
        const int32_t base = (int32_t)(b * g.span);
        const uint32_t zcnt = g.span - cnt;

        if (cnt == 0) { // all free
            for (uint32_t i = lane; i < g.span; i += 32) cache_free[zeros_before + i] = base + (int32_t)i;
            continue;
        }
        if (cnt == g.span) { // all live
            for (uint32_t i = lane; i < g.span; i += 32) cache_live[ones_before + i] = base + (int32_t)i;
            continue;
        }

        const uint32_t valid = g.span >= 1024 ? 32u
                             : (lane * 32u >= g.span ? 0u : (g.span - lane * 32u >= 32u ? 32u : g.span - lane * 32u));
        uint32_t w = valid ? bits32[(size_t)b * 32 + lane] : 0u;
        const uint32_t vmask = valid == 32 ? 0xffffffffu : ((1u << valid) - 1u);
        w &= vmask;
        const uint32_t c = __popc(w);
        const uint32_t incl = warp_inclusive_scan(c);
        uint32_t o1 = incl - c;                     // set bits before this lane
        uint32_t o0 = cnt + (lane * 32u > g.span ? g.span : lane * 32u) - o1; // staged after the ones
        const int32_t lane_base = base + lane * 32;
        uint32_t ones = w;
        while (ones) {
            const int k = __ffs(ones) - 1;
            ones &= ones - 1;
            st[o1++] = lane_base + k;
        }
        if (cache_free) {
            uint32_t zeros = ~w & vmask;
            while (zeros) {
                const int k = __ffs(zeros) - 1;
                zeros &= zeros - 1;
                st[o0++] = lane_base + k;
            }
        }
        __syncwarp();
        for (uint32_t i = lane; i < cnt; i += 32) cache_live[ones_before + i] = st[i];
        if (cache_free)
            for (uint32_t i = lane; i < zcnt; i += 32) cache_free[zeros_before + i] = st[cnt + i];
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Parity views of the reference heap layout (Cbt.nodes / Cbt.leaves).
// ---------------------------------------------------------------------------
__global__ void k_import_leaves(uint32_t *__restrict__ bits32, int depth,
                                const uint32_t *__restrict__ leaves)
{
    const uint64_t n = (uint64_t)1 << depth;
    const uint64_t nwords32 = bitfield_words(depth) * 2;
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords32;
         w += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t x = 0;
        for (int k = 0; k < 32; ++k) {
            const uint64_t s = w * 32 + k;
            if (s < n && leaves[s]) x |= 1u << k;
        }
        bits32[w] = x;
    }
}

__global__ void k_export_nodes(const uint64_t *__restrict__ bits,
                               const uint32_t *__restrict__ counters, int depth,
                               uint32_t *__restrict__ nodes)
{
    const Geo g = make_geo(depth);
    const uint64_t total = 2 * g.n;
    for (uint64_t h = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; h < total;
         h += (uint64_t)gridDim.x * blockDim.x) {
        if (h == 0) {
            nodes[0] = 0;
            continue;
        }
        const int l = 63 - __clzll((long long)h);
        const uint64_t i = h - ((uint64_t)1 << l);
        if (l <= g.lc) {
            nodes[h] = counters[h];
            continue;
        }
        const uint64_t span = (uint64_t)1 << (depth - l); // < 1024 slots
        const uint64_t first = i * span;
        uint32_t c = 0;
        if (span >= 64) {
            for (uint64_t w = 0; w < span / 64; ++w) c += __popcll(bits[first / 64 + w]);
        } else {
            const uint64_t x = bits[first / 64] >> (first % 64);
            c = __popcll(x & (((uint64_t)1 << span) - 1));
        }
        nodes[h] = c;
    }
}

} // namespace cbtm
