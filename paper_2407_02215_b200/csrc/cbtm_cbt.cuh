// cbtm_cbt.cuh -- the concurrent binary tree on a packed bitfield:
// sum reduction, ranked decode (k-th set / unset bit) and stream-compacted
// indexation.  Reference semantics: pkg/src/cbtmesh/cbt.py.
#pragma once

#include "cbtm_common.cuh"

namespace cbtm {

// ---------------------------------------------------------------------------
// Sum reduction (Cbt.sum_reduce, cbt.py:61-68; pipeline stage 9).
//
// A tile is 2^17 slots = 16 KB of bitfield = 128 leaf blocks = ONE CTA of 256 threads (32 registers:
// eight CTAs, 128 KB of loads in flight per SM; the hardware CTA scheduler is the load balancer --
// SMs that stream faster simply retire more tiles).  No ring, no shared-memory staging:
//   * a thread fetches its 64 contiguous bytes with two 256-bit loads (every lane a whole sector)
//     straight into registers, and a warp starts counting when ITS 2 KB have arrived;
//   * before griddepcontrol.wait (programmatic dependent launch: the CTAs are scheduled while the
//     previous kernel of the stream drains) the CTA's tile is pulled into L2 by one TMA bulk
//     prefetch, so that in a back-to-back series the loads behind the wait are L2 hits;
//   * the 16 words of a thread go through a carry-save adder tree (Harley-Seal: 30 logic operations
//     on the ALU pipe) that leaves five words to count instead of 16 -- POPC issues at 16 lanes per
//     clock and SM, and with every tile of a small pool landing within a microsecond it was the
//     kernel's tail;
//   * a leaf block is a lane pair and the warp's five tree levels (16+8+4+2+1 nodes) fall out of five
//     shuffle butterflies; disjoint lanes hold one node each and write all 31 with a single store
//     instruction; one CTA barrier joins the eight warps (3 more levels);
//   * levels above the tile roots: every tile adds the CHANGE of its root to its ancestors with
//     atomics (see TREE_STAMP); only a tree that was never built goes through a last-CTA rebuild.
// HBM traffic: N/8 bytes read + 4 * (2 << Lc) = N/128 bytes written.
// (Earlier versions streamed tiles through a ring of TMA bulk copies + mbarriers, 3 CTAs per SM: 0.27 / 0.53
// / 0.73 of the copy peak at 2^26 / 2^28 / 2^30 where this kernel reaches 0.38 / 0.75 / 0.95.)
// ---------------------------------------------------------------------------
constexpr int RED_THREADS = 256;
constexpr int RED_TILE_BYTES = 16384;
constexpr int RED_TILE_BLOCKS = 128; // leaf blocks per tile
constexpr uint32_t RED_HEAP_ROOTS = 2048; // rebuild path: tile roots the shared-memory heap holds (16 KB)

// end-of-frame bookkeeping (publish_frame)
struct ReducePublish {
    int64_t *ctl_stats;  // Control::stats
    int64_t *pool_stats; // cbtm_pool::stats
    int64_t *stats_seq;  // per-frame rows of a sequence run
    uint32_t *seq_frame; // Control::seq_frame
    const unsigned long long *phase_t; // this frame's Control::phase_t row (persistent kernel) or NULL
};

__device__ __forceinline__ unsigned long long global_ns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void publish_frame(const ReducePublish &pub, uint32_t live_after, int tid)
{
    if (!pub.ctl_stats) return;
    if (tid < CBTM_STATS_WORDS) { // one warp
        int64_t v = pub.ctl_stats[tid];
        if (tid == CBTM_STAT_LIVE_AFTER) v = live_after;
        if (tid == CBTM_STAT_FRAME) {
            v += 1;
            pub.ctl_stats[tid] = v;
        }
        const int64_t frame = __shfl_sync(FULL_MASK, v, CBTM_STAT_FRAME);
        if (tid == CBTM_STAT_SEQ || tid == CBTM_STAT_DONE) v = frame;
        if (tid >= CBTM_STAT_PHASE_NS && tid < CBTM_STAT_PHASE_NS + CBTM_STAT_PHASES) {
            v = 0;
            if (pub.phase_t) { // stamp k = start of phase k; the frame ends now
                const int k = tid - CBTM_STAT_PHASE_NS;
                const unsigned long long t0 = pub.phase_t[k];
                const unsigned long long t1 = k + 1 < CBTM_STAT_PHASES ? pub.phase_t[k + 1] : global_ns();
                v = t1 > t0 ? (int64_t)(t1 - t0) : 0;
            }
        }
        if (pub.stats_seq) pub.stats_seq[(size_t)CBTM_STATS_WORDS * (*pub.seq_frame) + tid] = v;
        // pool stats may live in host-mapped memory: counters first, fence, sequence word last
        if (pub.pool_stats) { // warp-uniform
            if (tid != CBTM_STAT_SEQ && tid != CBTM_STAT_DONE) pub.pool_stats[tid] = v;
            __threadfence_system();
            __syncwarp();
            if (tid == CBTM_STAT_SEQ || tid == CBTM_STAT_DONE) *(volatile int64_t *)&pub.pool_stats[tid] = v;
        }
        // the per-frame counters start the next frame at zero
        if (tid < CBTM_STAT_PHASE_NS && tid != CBTM_STAT_FRAME) pub.ctl_stats[tid] = 0;
    }
    __syncwarp();
    if (tid == 0) *pub.seq_frame += 1;
}

// The counters of a frame as soon as they are DECIDED: after the agreement phase every command
// is final (admission, split masks, merge agreement, allocation counts), so splits / merges applied,
// slots allocated and -- from them, pipeline.py:316-322 asserts exactly that identity -- the live
// count after the frame are known three phases before the frame has been applied and reduced.
// Written to pool->stats (host-mapped memory in ParallelEngine.update, which returns on the sequence
// word).  Not in this early row: the poison count of stage 6 (diagnostic, 0 by construction) and the
// times of the phases that have not run yet.  The frame's bookkeeping (per-frame rows, counter
// reset, the complete row, CBTM_STAT_DONE) stays with publish_frame at the end of the frame.  One warp.
__device__ __forceinline__ void publish_early(const int64_t *ctl_stats, int64_t *pool_stats,
                                              const unsigned long long *phase_t, int tid)
{
    if (tid >= CBTM_STATS_WORDS) return;
    int64_t v = ctl_stats[tid];
    const bool alloc = tid == CBTM_STAT_SPLIT_ALLOC || tid == CBTM_STAT_MERGE_ALLOC;
    const bool freed = tid == CBTM_STAT_SPLIT_FREED || tid == CBTM_STAT_MERGE_FREED;
    int64_t live_after = (tid == CBTM_STAT_LIVE_BEFORE || alloc) ? v : freed ? -v : 0;
    int64_t allocated = alloc ? v : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        live_after += __shfl_xor_sync(FULL_MASK, live_after, o);
        allocated += __shfl_xor_sync(FULL_MASK, allocated, o);
    }
    if (tid == CBTM_STAT_LIVE_AFTER) v = live_after;
    if (tid == CBTM_STAT_ALLOCATED) v = allocated;
    // (word CBTM_STAT_POISON: whatever earlier frames left unreported -- see retire_frame)
    if (tid == CBTM_STAT_FRAME) v += 1;
    const int64_t frame = __shfl_sync(FULL_MASK, v, CBTM_STAT_FRAME);
    if (tid >= CBTM_STAT_PHASE_NS && tid < CBTM_STAT_PHASE_NS + CBTM_STAT_PHASES) {
        const int k = tid - CBTM_STAT_PHASE_NS;
        v = 0;
        if (phase_t && k < 3) { // index, classify, agree have run
            const unsigned long long t0 = phase_t[k];
            const unsigned long long t1 = k < 2 ? phase_t[k + 1] : global_ns();
            v = t1 > t0 ? (int64_t)(t1 - t0) : 0;
        }
    }
    if (tid != CBTM_STAT_SEQ && tid != CBTM_STAT_DONE) pool_stats[tid] = v;
    __threadfence_system();
    __syncwarp();
    if (tid == CBTM_STAT_SEQ) *(volatile int64_t *)&pool_stats[tid] = frame;
}

// End-of-frame bookkeeping of a single-frame launch that publishes only the early row: frame
// counter, per-frame counters back to zero.  Runs right behind the barrier that ends the apply
// phase (every counter is final then), next to the reduction, so that the kernel can end with
// its reduction work -- no device-wide barrier and no host write on its tail.  The poison count
// is NOT reset: nobody has reported it yet, the next frame's row will.  One warp.
__device__ __forceinline__ void retire_frame(int64_t *ctl_stats, uint32_t *seq_frame, int tid)
{
    if (tid < CBTM_STAT_PHASE_NS) {
        if (tid == CBTM_STAT_FRAME) ctl_stats[tid] += 1;
        else if (tid != CBTM_STAT_POISON) ctl_stats[tid] = 0;
    }
    if (tid == 0) *seq_frame += 1;
}

// counters[0] is padding in the heap layout; the library keeps a stamp there that says "every
// counter above the tile roots equals the sum of its children" (true after any full build and
// kept true by the in-frame reducer).  With the stamp present a full reduction does not rebuild
// those levels: each tile adds the CHANGE of its root to its ancestors with fire-and-forget
// atomics, so the kernel has no last-CTA pass, no ticket and no fence.  Without it (fresh or
// foreign counters) the last CTA to finish rebuilds them and sets the stamp.
constexpr uint32_t TREE_STAMP = 0x31544243u; // "CBT1"

// Programmatic dependent launch: the CTAs of the next PDL-launched kernel on the stream may be
// scheduled (and run their prologue up to griddep_wait) while this grid is still running.
__device__ __forceinline__ void griddep_launch_dependents()
{
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// TMA bulk prefetch of `bytes` (a multiple of 16) into L2.  L2 is the device's point of coherence, so
// unlike a load this may be issued for memory an earlier kernel is still writing.
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Levels above `cnt` subtree roots (counters[cnt .. 2 cnt), cnt a power of two >= 2),
// built by the last CTA to arrive (ticket; only thread 0 fences -- the fence is
// cumulative over the preceding barrier).  Binary heap in shared memory (`heap`,
// 2 * cnt words): coalesced L2 loads of the roots issued eight at a time per
// thread so they overlap, log2(cnt) levels in shared memory, one coalesced
// copy-out of all internal nodes (walking the levels through L2 instead costs a
// round trip per level).  All nb CTAs must call it.
__device__ __forceinline__ void finish_upper_tree(uint32_t *counters, uint32_t cnt, unsigned *ticket,
                                                  uint32_t *heap, bool *is_last, uint32_t nb, uint32_t heap_cap = ~0u)
{
    const int t = threadIdx.x;
    __syncthreads();
    if (t == 0) {
        __threadfence();
        *is_last = atomicAdd(ticket, 1u) == nb - 1;
    }
    __syncthreads();
    if (!*is_last) return;
    __threadfence();
    // more roots than the shared-memory heap holds (heap_cap of them): the first levels go through L2
    for (; cnt > heap_cap; cnt >>= 1) {
        const uint32_t w = cnt >> 1;
        for (uint32_t i = t; i < w; i += RED_THREADS) {
            const uint2 kids = __ldcg(reinterpret_cast<const uint2 *>(counters + 2 * (w + i)));
            counters[w + i] = kids.x + kids.y;
        }
        __syncthreads();
    }
    for (uint32_t base = 0; base < cnt; base += 8 * RED_THREADS) {
        uint32_t r[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t i = base + u * RED_THREADS + t;
            r[u] = i < cnt ? __ldcg(&counters[cnt + i]) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t i = base + u * RED_THREADS + t;
            if (i < cnt) heap[cnt + i] = r[u];
        }
    }
    __syncthreads();
    for (uint32_t w = cnt >> 1; w >= 1; w >>= 1) {
        for (uint32_t i = t; i < w; i += RED_THREADS) heap[w + i] = heap[2 * (w + i)] + heap[2 * (w + i) + 1];
        __syncthreads();
    }
    for (uint32_t i = 1 + t; i < cnt; i += RED_THREADS) counters[i] = heap[i];
    if (t == 0) {
        *ticket = 0;
        counters[0] = TREE_STAMP;
    }
    __syncthreads();
}

// The subtree of one tile (128 leaf blocks, 8 levels), shared by the two reduction kernels.  A thread
// holds the count `c` of its 64 contiguous bytes: a leaf block is a lane pair, five butterflies give the
// warp's 16+8+4+2+1 nodes, disjoint lanes each hold one node and write all 31 with one store
// instruction.  Returns the warp's root (16 leaf blocks).
__device__ __forceinline__ uint32_t tile_tree_warp(uint32_t c, uint32_t tile, int lc, uint32_t *counters, int lane,
                                                   int warp)
{
    // butterflies: l0 leaf block (lane pair) ... l4 all 16 leaf blocks of the warp
    const uint32_t l0 = c + __shfl_xor_sync(FULL_MASK, c, 1);
    const uint32_t l1 = l0 + __shfl_xor_sync(FULL_MASK, l0, 2);
    const uint32_t l2 = l1 + __shfl_xor_sync(FULL_MASK, l1, 4);
    const uint32_t l3 = l2 + __shfl_xor_sync(FULL_MASK, l2, 8);
    const uint32_t l4 = l3 + __shfl_xor_sync(FULL_MASK, l3, 16);

    uint32_t val = 0, pos = 0;
    int lvl = -1;
    if ((lane & 1) == 0) {
        val = l0, lvl = lc, pos = tile * 128 + warp * 16 + (lane >> 1);
    } else if ((lane & 3) == 1) {
        val = l1, lvl = lc - 1, pos = tile * 64 + warp * 8 + (lane >> 2);
    } else if ((lane & 7) == 3) {
        val = l2, lvl = lc - 2, pos = tile * 32 + warp * 4 + (lane >> 3);
    } else if ((lane & 15) == 7) {
        val = l3, lvl = lc - 3, pos = tile * 16 + warp * 2 + (lane >> 4);
    } else if (lane == 15) {
        val = l4, lvl = lc - 4, pos = tile * 8 + warp;
    }
    if (lvl >= 0 && pos < (1u << lvl)) counters[(1u << lvl) + pos] = val;
    return l4;
}

// Warp 0, from the eight warp roots `w` (shared memory): levels lc-5 (4 nodes), lc-6 (2), lc-7 (the
// tile root); then, on a stamped tree, the levels above: lane l adds the change of the tile root
// (old_root: the root as the levels above still see it, held by lane 6) to the ancestor on level l.
__device__ __forceinline__ void tile_tree_top(const uint32_t *w, uint32_t tile, int lc, uint32_t *counters, int lane,
                                              bool delta_mode, uint32_t old_root)
{
    const int top = lc - 7; // level of the tile roots
    uint32_t v2 = 0, p2 = 0;
    int l5 = -1;
    if (lane < 4) {
        v2 = w[2 * lane] + w[2 * lane + 1], l5 = lc - 5, p2 = tile * 4 + lane;
    } else if (lane < 6) {
        const int q = (lane - 4) * 4;
        v2 = w[q] + w[q + 1] + w[q + 2] + w[q + 3], l5 = lc - 6, p2 = tile * 2 + (lane - 4);
    } else if (lane == 6) {
        v2 = w[0] + w[1] + w[2] + w[3] + w[4] + w[5] + w[6] + w[7], l5 = lc - 7, p2 = tile;
    }
    if (l5 >= 0 && p2 < (1u << l5)) counters[(1u << l5) + p2] = v2;
    if (delta_mode) {
        const uint32_t delta = __shfl_sync(FULL_MASK, v2 - old_root, 6);
        if (delta != 0 && lane < top) atomicAdd(&counters[(1u << lane) + (tile >> (top - lane))], delta);
    }
}

#ifdef CBTM_DEBUG_TIMING
// per CTA: kernel entry, released by griddepcontrol.wait, first tile landed, last tile counted, SM id;
// four slots of 2048 CTAs, chosen by the 256-byte unit the ticket pointer sits in (so that the launches
// of a back-to-back series can be told apart: benchmarks/reduce_chain_probe.cu)
__device__ unsigned long long g_reduce_stamps[4 * 2048 * 5];
#define RED_STAMP_ROW() (g_reduce_stamps + ((((uintptr_t)ticket >> 8) & 3) * 2048 + blockIdx.x) * 5)
#define RED_STAMP(slot)                                                                                           \
    do {                                                                                                          \
        if (threadIdx.x == 0 && blockIdx.x < 2048) RED_STAMP_ROW()[slot] = global_ns();                           \
    } while (0)
#else
#define RED_STAMP(slot)
#endif

__device__ __forceinline__ void csa(uint32_t a, uint32_t b, uint32_t c, uint32_t &sum, uint32_t &carry)
{
    sum = a ^ b ^ c;
    carry = (a & b) | (c & (a ^ b));
}

// number of set bits in 16 words
__device__ __forceinline__ uint32_t popc_16words(const uint32_t (&w)[16])
{
#ifdef CBTM_REDUCE_PLAIN_POPC
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) c += __popc(w[j]);
    return c;
#else
    uint32_t s0, s1, s2, s3, s4, s5, s6, c0, c1, c2, c3, c4, c5, c6;
    csa(w[0], w[1], w[2], s0, c0);
    csa(w[3], w[4], w[5], s1, c1);
    csa(w[6], w[7], w[8], s2, c2);
    csa(w[9], w[10], w[11], s3, c3);
    csa(w[12], w[13], w[14], s4, c4);
    csa(s0, s1, s2, s5, c5);
    csa(s3, s4, w[15], s6, c6);
    const uint32_t ones = s5 ^ s6, c7 = s5 & s6;
    uint32_t t0, t1, t2, d0, d1, d2;
    csa(c0, c1, c2, t0, d0);
    csa(c3, c4, c5, t1, d1);
    csa(c6, c7, t0, t2, d2);
    const uint32_t twos = t1 ^ t2, d3 = t1 & t2;
    uint32_t f0, e0;
    csa(d0, d1, d2, f0, e0);
    const uint32_t fours = f0 ^ d3, e1 = f0 & d3;
    const uint32_t eights = e0 ^ e1, sixteens = e0 & e1;
    return __popc(ones) + 2 * __popc(twos) + 4 * __popc(fours) + 8 * __popc(eights) + 16 * __popc(sixteens);
#endif
}

__device__ __forceinline__ void ldg256(const void *p, uint32_t *v)
{
    asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" // L2 only: streamed once, never stale
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "l"(p)
                 : "memory");
}

// One full sum reduction by the grid (Cbt.sum_reduce, initialize, BASELINE config 4): gridDim.x = n_tiles.
// WIDE: the bitfield is 32-byte aligned (256-bit loads); otherwise four 128-bit loads per thread (the ABI
// asks for 16-byte alignment only).
template <bool WIDE>
__global__ void __launch_bounds__(RED_THREADS)
k_sum_reduce(const uint8_t *bits, uint32_t *counters, int lc, uint64_t total_bytes, uint32_t n_tiles,
             unsigned *ticket, int prefetch)
{
    extern __shared__ __align__(16) uint32_t heap[]; // 2 * min(n_tiles, RED_HEAP_ROOTS) words: rebuild path only
    __shared__ uint32_t wroot[RED_THREADS / 32];
    __shared__ bool is_last, s_delta;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t tile = blockIdx.x;
    const uint64_t left = total_bytes - (uint64_t)tile * RED_TILE_BYTES;
    const uint32_t bytes = left < RED_TILE_BYTES ? (uint32_t)left : (uint32_t)RED_TILE_BYTES;
    const uint8_t *src = bits + (size_t)tile * RED_TILE_BYTES;

    RED_STAMP(0);
    // nothing is READ before the wait: the address comes from the launch parameters, and a line
    // prefetched into L2 cannot go stale (L2 is where the previous kernel's writes land)
    if (t == 0 && prefetch) bulk_prefetch_l2(src, bytes);
    // (prefetching the two counter words of the delta path as well was measured and rejected: the stamp is
    // one line for the whole grid, and 8192 prefetches of it cost more than its one cold read)
    griddep_wait();
    RED_STAMP(1);
#ifdef CBTM_DEBUG_TIMING
    if (t == 0 && tile < 2048) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        RED_STAMP_ROW()[4] = smid;
    }
#endif
    uint32_t w[16];
    const bool mine = (uint32_t)t * 64u < bytes; // (partial tile of a tiny pool; bytes is a multiple of 128)
    if (mine && WIDE) {
        ldg256(src + t * 64, w);
        ldg256(src + t * 64 + 32, w + 8);
    } else if (mine) {
        const uint4 *q = reinterpret_cast<const uint4 *>(src + t * 64);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint4 v = __ldcg(q + j);
            w[4 * j] = v.x, w[4 * j + 1] = v.y, w[4 * j + 2] = v.z, w[4 * j + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) w[j] = 0;
    }
    // The next grid of the stream may be set up from here on -- not earlier: a CTA that waits in
    // griddepcontrol.wait holds its slot, and in a long series of reductions the grids two and three ahead
    // (each released as soon as all CTAs of the one before it were running) piled up on the SMs, left the
    // current grid a CTA or two per SM and made a launch 4.3 us long (benchmarks/reduce_chain_probe.py with
    // CHAIN=16: 1..7 CTAs of one grid per SM).  Triggered behind the wait, only ONE grid is ever waiting.
    griddep_launch_dependents();
    const int top = lc - 7; // level of the tile roots (n_tiles > 1)
    uint32_t old_root = 0;
    // The stamp is the same word for every CTA of the grid (only the rebuild path writes it, after the
    // last ticket).  ONE lane per CTA reads it: a load by every warp put 8 requests per CTA on a single
    // L2 sector -- 4096 at 2^26, served one per clock by its slice: a microsecond at the head of the launch.
    bool delta_mode = false;
    if (t == 6 && n_tiles > 1) {
        old_root = __ldcg(counters + (1u << top) + tile);
        delta_mode = __ldcg(&counters[0]) == TREE_STAMP;
    }

    const uint32_t c = popc_16words(w);
    RED_STAMP(2);
    const uint32_t l4 = tile_tree_warp(c, tile, lc, counters, lane, warp);
    if (lane == 0) wroot[warp] = l4;
    if (t == 6) s_delta = delta_mode;
    __syncthreads();
    if (warp == 0) tile_tree_top(wroot, tile, lc, counters, lane, s_delta, old_root);
    RED_STAMP(3);
    if (n_tiles == 1) { // the single tile's subtree is the whole tree
        if (t == 0) counters[0] = TREE_STAMP;
        return;
    }
    if (s_delta) return;
    finish_upper_tree(counters, n_tiles, ticket, heap, &is_last, gridDim.x, RED_HEAP_ROOTS);
}

// ---------------------------------------------------------------------------
// Incremental sum reduction (pipeline stage 9 inside a frame).  phase_apply
// marks the leaf block of every bit it flips in a byte map (plain stores: no
// read-modify-write, any number of writers); here the marked blocks recount
// their 128-byte line and every level above the leaf blocks is rebuilt:
// N/1024 counters + N/1024 marks in, as many counters out, plus 128 bytes per
// touched block, instead of a pass over the whole bitfield (D = 26: ~0.4 MB
// instead of 8 MB; the cost no longer grows with the bitfield).  A tile is 1024
// leaf counters: a thread owns four (one 128-bit load) and with them two nodes
// of level Lc-1 and one of Lc-2; five shuffle butterflies and one CTA barrier
// give the other eight levels of the tile, as in reduce_phase.  The levels above
// the tile roots (6 at D = 26) are not rebuilt: each tile adds the change of its
// root to its ancestors with atomics, so there is no last-CTA pass, no ticket
// and no fence on the frame's critical path.  Untouched tiles write nothing.
// ---------------------------------------------------------------------------
constexpr int UP_TILE = 1024;

__device__ __forceinline__ uint32_t recount_block(const uint64_t *bits, uint32_t block)
{
    const uint4 *line = reinterpret_cast<const uint4 *>(bits) + (size_t)block * 8;
    uint4 x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = line[j];
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) c += popc128(x[j]);
    return c;
}

__device__ __forceinline__ void upper_reduce_phase(const uint64_t *bits, uint8_t *dirty, uint32_t *counters,
                                                   int lc, uint32_t *tile_vals /* UP_TILE words of shared memory */,
                                                   uint32_t (*wroot)[RED_THREADS / 32], uint32_t bid, uint32_t nb)
{
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t nblocks = 1u << lc;
    const uint32_t n_tiles = nblocks > (uint32_t)UP_TILE ? nblocks / UP_TILE : 1u;
    const int top = lc > 10 ? lc - 10 : 0; // level of the tile roots
    auto put = [&](int lvl, uint32_t pos, uint32_t val) {
        if (lvl >= 0 && pos < (1u << lvl)) counters[(1u << lvl) + pos] = val;
    };
    uint32_t k = 0;
    for (uint32_t tile = bid; tile < n_tiles; tile += nb, ++k) {
        // Recount: a frame's fresh slots fall into a run of CONSECUTIVE leaf blocks, so for this step a
        // thread owns the blocks t, t + 256, t + 512, t + 768 of the tile (a dense run of marks then
        // spreads over different threads and their recounts run in parallel, one round trip), and the
        // values change hands through shared memory for the tree, where a thread owns four siblings.
        const uint32_t base = tile * UP_TILE;
        uint32_t c[4] = {0, 0, 0, 0};
        uint32_t d[4] = {0, 0, 0, 0};
        uint32_t old_root = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t b = base + t + q * RED_THREADS;
            if (b < nblocks) {
                c[q] = counters[nblocks + b];
                d[q] = dirty[b];
            }
        }
        // the tile root as the levels above still see it (rewritten below by this same thread)
        if (n_tiles > 1 && t == 0) old_root = counters[(1u << top) + tile];
        // a tile without a touched block keeps all its counters
        if (!__syncthreads_or((d[0] | d[1] | d[2] | d[3]) != 0)) continue;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t b = base + t + q * RED_THREADS;
            if (d[q]) {
                c[q] = recount_block(bits, b);
                counters[nblocks + b] = c[q];
                dirty[b] = 0;
            }
            tile_vals[t + q * RED_THREADS] = c[q];
        }
        __syncthreads();
        const uint4 v = *reinterpret_cast<const uint4 *>(tile_vals + 4 * t);
        const uint32_t a0 = v.x + v.y, a1 = v.z + v.w, cc = a0 + a1;
        put(lc - 1, tile * 512 + 2 * t, a0);
        put(lc - 1, tile * 512 + 2 * t + 1, a1);
        put(lc - 2, tile * 256 + t, cc);
        const uint32_t l1 = cc + __shfl_xor_sync(FULL_MASK, cc, 1);
        const uint32_t l2 = l1 + __shfl_xor_sync(FULL_MASK, l1, 2);
        const uint32_t l3 = l2 + __shfl_xor_sync(FULL_MASK, l2, 4);
        const uint32_t l4 = l3 + __shfl_xor_sync(FULL_MASK, l3, 8);
        const uint32_t l5 = l4 + __shfl_xor_sync(FULL_MASK, l4, 16);
        if ((lane & 1) == 0) put(lc - 3, tile * 128 + warp * 16 + (lane >> 1), l1);
        else if ((lane & 3) == 1) put(lc - 4, tile * 64 + warp * 8 + (lane >> 2), l2);
        else if ((lane & 7) == 3) put(lc - 5, tile * 32 + warp * 4 + (lane >> 3), l3);
        else if ((lane & 15) == 7) put(lc - 6, tile * 16 + warp * 2 + (lane >> 4), l4);
        else if (lane == 15) put(lc - 7, tile * 8 + warp, l5);
        if (lane == 0) wroot[k & 1][warp] = l5;
        __syncthreads(); // (also: tile_vals may be refilled by the next tile)
        if (warp == 0 && lane < 7) {
            const uint32_t *w = wroot[k & 1];
            if (lane < 4) put(lc - 8, tile * 4 + lane, w[2 * lane] + w[2 * lane + 1]);
            else if (lane < 6) {
                const int q = (lane - 4) * 4;
                put(lc - 9, tile * 2 + (lane - 4), w[q] + w[q + 1] + w[q + 2] + w[q + 3]);
            } else
                put(lc - 10, tile, w[0] + w[1] + w[2] + w[3] + w[4] + w[5] + w[6] + w[7]);
        }
        if (n_tiles > 1 && t == 0) { // the levels above the tile roots take the tile's delta
            const uint32_t *w = wroot[k & 1];
            const uint32_t delta = w[0] + w[1] + w[2] + w[3] + w[4] + w[5] + w[6] + w[7] - old_root;
            if (delta) {
                uint32_t idx = tile >> 1;
                for (int l = top - 1; l >= 0; --l, idx >>= 1) atomicAdd(&counters[(1u << l) + idx], delta);
            }
        }
    }
}

__global__ void __launch_bounds__(RED_THREADS)
k_upper_reduce(const uint64_t *bits, uint8_t *dirty, uint32_t *counters, int lc)
{
    __shared__ __align__(16) uint32_t tile_vals[UP_TILE];
    __shared__ uint32_t wroot[2][RED_THREADS / 32];
    upper_reduce_phase(bits, dirty, counters, lc, tile_vals, wroot, blockIdx.x, gridDim.x);
}

// ---------------------------------------------------------------------------
// Ranked decode (one_to_bit_id / zero_to_bit_id, cbt.py:75-107 and 127-150):
// descent over the counter heap, then popcount select inside the 128-byte leaf
// block.
// ---------------------------------------------------------------------------
template <bool ONES, bool WIDE = false>
__device__ __forceinline__ int32_t cbt_find(const uint64_t *bits, const uint32_t *counters,
                                            const Geo &g, uint32_t rank)
{
    uint32_t node = 1;
    int l = 0;
    // Three levels per step: the eight descendants of a node three levels down are contiguous in the
    // heap (one aligned 32-byte load), and which of them holds the rank is a chain of compares -- one
    // dependent load per three levels instead of three.
    for (; l + 3 <= g.lc; l += 3) {
        const uint32_t base = node << 3;
        uint32_t c[8];
        if (WIDE) { // 32-byte aligned counters: the eight siblings with one load instruction
            asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3]), "=r"(c[4]), "=r"(c[5]), "=r"(c[6]), "=r"(c[7])
                         : "l"(counters + base)
                         : "memory");
        } else {
            const uint4 lo = *reinterpret_cast<const uint4 *>(counters + base);
            const uint4 hi = *reinterpret_cast<const uint4 *>(counters + base + 4);
            c[0] = lo.x, c[1] = lo.y, c[2] = lo.z, c[3] = lo.w, c[4] = hi.x, c[5] = hi.y, c[6] = hi.z, c[7] = hi.w;
        }
        const uint32_t span = (uint32_t)(g.n >> (l + 3)); // slots under each of the eight
        uint32_t k = 0;
#pragma unroll
        for (int q = 0; q < 7; ++q) {
            const uint32_t v = ONES ? c[q] : span - c[q];
            const bool beyond = k == (uint32_t)q && rank >= v; // still walking right, and not in child q
            rank -= beyond ? v : 0u;
            k += beyond ? 1u : 0u;
        }
        node = base + k;
    }
    uint32_t half = (uint32_t)(g.n >> (l + 1)); // slots under a child of the current node
    for (; l < g.lc; ++l) {
        node <<= 1;
        const uint32_t ones = counters[node];
        const uint32_t left = ONES ? ones : half - ones;
        if (rank >= left) {
            rank -= left;
            node += 1;
        }
        half >>= 1;
    }
    const uint32_t block = node - g.nblocks;
    const uint64_t *line = bits + (size_t)block * 16;
    if (WIDE && g.span == 1024u) {
        // A 32-byte sector per step with one 256-bit load (the bitfield is 32-byte aligned): with
        // random ranks every lane of a load touches its own line, so the L1 pays per INSTRUCTION and
        // lane -- a word per step meant 8 loads for the average rank, a sector per step means 2.5
        // for the same sectors from L2.
        for (int sct = 0; sct < 4; ++sct) {
            uint32_t w[8];
            asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                         : "l"(line + 4 * sct)
                         : "memory");
            if (!ONES) {
#pragma unroll
                for (int j = 0; j < 8; ++j) w[j] = ~w[j];
            }
            uint32_t c[8], total = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                c[j] = __popc(w[j]);
                total += c[j];
            }
            if (rank >= total) {
                rank -= total;
                continue;
            }
            uint32_t word = 0, at = 0; // the 32-bit word holding the rank, found without branching
            bool found = false;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const bool here = !found && rank < c[j];
                if (here) word = w[j], at = (uint32_t)j;
                found |= here;
                if (!found) rank -= c[j];
            }
            return (int32_t)(block * 1024u + (uint32_t)sct * 256u + at * 32u + (uint32_t)select32(word, (int)rank));
        }
        return -1; // rank out of range
    }
    // (words are fetched one by one with an early exit: fetching the whole 128-byte line at once costs
    // four times the L2 sectors and made random decodes 1.5x slower)
    const int words = g.span >= 64 ? (int)(g.span >> 6) : 1;
    for (int w = 0; w < words; ++w) {
        uint64_t x = line[w];
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

// WIDE: bitfield and counters are 32-byte aligned (256-bit loads in the descent and in the leaf search)
template <bool ONES, bool WIDE>
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
        out[i] = (r < 0 || (uint64_t)r >= limit) ? -1 : cbt_find<ONES, WIDE>(bits, counters, g, (uint32_t)r);
    }
}

// ---------------------------------------------------------------------------
// Indexation (pipeline stage 2, k_cache_pointers kernels.py:244-252) as a
// stream compaction.  One warp per 1024-slot leaf block:
//   * its rank offset comes from the counter heap (sum of the left siblings on
//     the root path -- all addresses known up front, one load per lane);
//   * lane l owns word l of the block.  Live list only (the frame's index phase, sparse pools): the
//     warp walks the non-empty words, each broadcast with one shuffle, and lane l handles BIT l of the
//     current word -- its rank inside the word is a popcount under a lane mask.  Both lists
//     (decode-all): every lane expands ITS OWN word, 32 steps of test-bit / select / store / count
//     from the staging indices a five-step scan of the words' popcounts gives it.  Slots go to a
//     shared staging area (set bits first, unset bits behind them), each list placed so that its
//     staging index is congruent to its global index modulo 32;
//   * the copy-out therefore moves 128-byte-aligned lines with 128-bit shared
//     loads and 128-bit global stores (scalar stores only on the two edge
//     vectors of a list).
// ncu on the first versions showed decode-all bound by instruction issue (71-78 % issue slots busy):
// hence the instruction diet; the own-word expansion is bound by the shared-memory data path instead
// (its scattered staging stores take ~4 bank conflicts each).
// Blocks with no set bit are skipped from their counter without touching the
// bitfield when the free list is not requested; so are empty words.
// Plain (coherent) loads only: inside the persistent frame kernel the bitfield
// and the counters were written earlier in the same launch.
// ---------------------------------------------------------------------------
constexpr int IDX_WARPS = 8;
constexpr int IDX_STAGE_WORDS = 1152; // 1024 slots + alignment slack of both lists

// out[gbase + off .. gbase + off + count) = st[off .. off + count); gbase is a multiple of 32
// entries (128 bytes) and st is 16-byte aligned, so interior vectors move as int4.
__device__ __forceinline__ void copy_out_lines(int32_t *out, uint32_t gbase, uint32_t off, uint32_t count,
                                               const int32_t *st, int lane)
{
    const uint32_t total = off + count;
    for (uint32_t e0 = 4u * lane; e0 < total; e0 += 128u) {
        if (e0 + 4u <= off) continue;
        const int4 x = *reinterpret_cast<const int4 *>(st + e0);
        if (e0 >= off && e0 + 4u <= total) {
            *reinterpret_cast<int4 *>(out + gbase + e0) = x;
        } else {
            if (e0 >= off && e0 < total) out[gbase + e0] = x.x;
            if (e0 + 1 >= off && e0 + 1 < total) out[gbase + e0 + 1] = x.y;
            if (e0 + 2 >= off && e0 + 2 < total) out[gbase + e0 + 2] = x.z;
            if (e0 + 3 >= off && e0 + 3 < total) out[gbase + e0 + 3] = x.w;
        }
    }
}

// The same copy by the TMA: the 16-byte aligned interior of the run as ONE bulk copy shared -> global
// (cp.async.bulk.global.shared::cta, issued by lane 0), at most three head and three tail entries by
// scalar stores.  The staging stores must have been made visible to the async proxy
// (fence.proxy.async + __syncwarp) before the call; the staging area may be rewritten only after
// cp.async.bulk.wait_group.read says the copy has read it.  Takes the 128-bit shared loads and global stores of the copy-out off the
// LSU / shared-memory path, which is what bounds decode-all.
__device__ __forceinline__ void bulk_copy_out(int32_t *out, uint32_t gbase, uint32_t off, uint32_t count,
                                              const int32_t *st, int lane)
{
    const uint32_t end = off + count;
    const uint32_t a0 = (off + 3u) & ~3u, a1 = end & ~3u; // aligned interior [a0, a1)
    if (a1 > a0) {
        if (lane == 0)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + gbase + a0),
                         "r"((uint32_t)__cvta_generic_to_shared(st + a0)), "r"(4u * (a1 - a0))
                         : "memory");
        // head [off, a0) and tail [a1, end): lanes 1..3 and 4..6
        if (lane >= 1 && lane <= 3 && off + (uint32_t)(lane - 1) < a0) out[gbase + off + (lane - 1)] = st[off + (lane - 1)];
        if (lane >= 4 && lane <= 6 && a1 + (uint32_t)(lane - 4) < end) out[gbase + a1 + (lane - 4)] = st[a1 + (lane - 4)];
    } else if ((uint32_t)lane < count) { // fewer than four aligned entries: at most six in all
        out[gbase + off + lane] = st[off + lane];
    }
}
__device__ __forceinline__ void bulk_copy_out_commit(int lane)
{
    if (lane == 0) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// out[first .. first + count) = slot0, slot0 + 1, ... (a block that is entirely live or free)
__device__ __forceinline__ void fill_run_lines(int32_t *out, uint32_t first, uint32_t count, int32_t slot0,
                                               int lane)
{
    const uint32_t off = first & 31u, gbase = first - off, total = off + count;
    for (uint32_t e0 = 4u * lane; e0 < total; e0 += 128u) {
        if (e0 + 4u <= off) continue;
        const int32_t v = slot0 + (int32_t)e0 - (int32_t)off;
        if (e0 >= off && e0 + 4u <= total) {
            *reinterpret_cast<int4 *>(out + gbase + e0) = make_int4(v, v + 1, v + 2, v + 3);
        } else {
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k)
                if (e0 + k >= off && e0 + k < total) out[gbase + e0 + k] = v + (int32_t)k;
        }
    }
}

// BULK (k_index_all): the copy-out of decode-all goes through TMA bulk stores out of TWO staging areas per
// warp (stage[2 * warp], stage[2 * warp + 1]), so that the store of one block overlaps the expansion of the
// next.  Standalone kernel only: the stores are awaited when the warp is done, nothing orders them against
// a later phase of a persistent kernel.
template <bool RESET, bool BULK = false>
__device__ __forceinline__ void index_phase(const uint32_t *bits32, const uint32_t *counters, int depth,
                                            int32_t *cache_live, int32_t *cache_free, uint32_t *dispatch,
                                            uint32_t *reset_cmds, int32_t (*stage)[IDX_STAGE_WORDS],
                                            uint32_t bid, uint32_t nb)
{
    const Geo g = make_geo(depth);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t gwarp = bid * IDX_WARPS + warp;
    const uint32_t nwarps = nb * IDX_WARPS;
    const uint32_t lane_lt = (1u << lane) - 1u;
    const bool want_free = cache_free != nullptr;
    int32_t *st = stage[BULK ? 2 * warp : warp];
    uint32_t bulk_turn = 0; // BULK: staging area of the next block

    if (dispatch && bid == 0 && threadIdx.x == 0) {
        const uint32_t n = counters[1];
        dispatch[0] = (n + CHUNK - 1) / CHUNK;
        dispatch[1] = 1;
        dispatch[2] = 1;
        dispatch[3] = n;
    }

    // this warp owns leaf blocks gwarp + k * nwarps; lane k fetches the count of the
    // k-th of them, so one round trip tells the warp which of its next 32 blocks
    // hold anything (a sparse pool skips almost all of them)
    for (uint32_t k0 = 0; gwarp + (uint64_t)k0 * nwarps < g.nblocks; k0 += 32) {
        const uint64_t mine = gwarp + (uint64_t)(k0 + lane) * nwarps;
        const uint32_t my_cnt = mine < g.nblocks ? counters[g.nblocks + mine] : 0u;
        unsigned todo = __ballot_sync(FULL_MASK, mine < g.nblocks && (my_cnt != 0 || want_free));
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            const uint32_t b = gwarp + (k0 + src) * nwarps;
            const uint32_t cnt = __shfl_sync(FULL_MASK, my_cnt, src);

            // the block's bits travel together with the root path (one round trip, not two)
            // (issuing them one block ahead was measured and rejected: more registers, decode-all 4 % slower)
            const uint32_t own_full = (g.span == 1024u && cnt != 0 && cnt != g.span) ? bits32[(size_t)b * 32 + lane] : 0u;
            // ones before this block: left siblings along the root path
            uint32_t part = 0;
            if (lane >= 1 && lane <= g.lc) {
                const uint32_t idx = b >> (g.lc - lane);
                if (idx & 1) part = counters[(1u << lane) + idx - 1];
            }
            const uint32_t ones_before = warp_sum(part);
            const uint32_t zeros_before = b * g.span - ones_before;
            const int32_t base = (int32_t)(b * g.span);

            if (cnt == 0 || cnt == g.span) { // uniform block: no expansion needed
                fill_run_lines(cnt ? cache_live : cache_free, cnt ? ones_before : zeros_before, g.span, base, lane);
                if (RESET && cnt)
                    for (uint32_t e = lane; e < g.span; e += 32) reset_cmds[(uint32_t)base + e] = 0u;
                continue;
            }

            // staging: ones at [o1, o1 + cnt), zeros at [z0, z0 + zcnt); both congruent to their
            // global index modulo 32
            const uint32_t zcnt = g.span - cnt;
            const uint32_t o1 = ones_before & 31u;
            const uint32_t zline = (o1 + cnt + 31u) & ~31u;
            const uint32_t z0 = zline + (zeros_before & 31u);
            uint32_t p1 = o1, p0 = z0;
            if (g.span == 1024u && want_free) { // decode-all: every slot goes to exactly one of the two lists
                // Lane w expands ITS OWN word: one POPC and a five-step scan per block give every word's
                // first staging index in both lists; then 32 steps of test-bit / select / store / count --
                // no shuffle and no POPC inside the loop.  (Earlier versions took a word per step across the
                // lanes -- shuffle, two POPCs on the quarter-rate pipe, twelve instructions per 32 slots --
                // and were bound by instruction issue: 2^30 leaves 916 us.  Now 864 us; the lanes' staging
                // addresses are unrelated, so a store takes ~4 bank conflicts and the kernel is bound by
                // the shared-memory data path: ncu l1tex 91 % of peak, profiles/r2b_index_own_word_d28_ncu.txt.)
                const uint32_t own = own_full;
                const uint32_t c = __popc(own);
                uint32_t incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t up = __shfl_up_sync(FULL_MASK, incl, o);
                    if (lane >= o) incl += up;
                }
                const uint32_t e1 = incl - c; // ones in the words before mine
                uint32_t q1 = p1 + e1;                                       // next set bit of my word goes here
                const uint32_t q01 = (p0 + 32u * (uint32_t)lane - e1) + q1;  // a clear bit k goes to q01 + k - q1
                const int32_t v = base + 32 * lane;
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    const bool bit = (own >> k) & 1u;
                    st[bit ? q1 : q01 + (uint32_t)k - q1] = v + k;
                    if (RESET && bit) reset_cmds[v + k] = 0u;
                    q1 += bit;
                }
            } else if (g.span == 1024u) { // every word fully valid (all pools with D >= 10)
                const uint32_t own = own_full;
#pragma unroll 8
                for (int w = 0; w < 32; ++w) {
                    const uint32_t word = __shfl_sync(FULL_MASK, own, w);
                    if (word == 0u) continue;
                    const uint32_t r1 = __popc(word & lane_lt);
                    const int32_t slot = base + w * 32 + lane;
                    // (two predicated stores: one `if` around both made the compiler emit a divergent
                    // branch with a reconvergence barrier per word)
                    const bool bit = (word >> lane) & 1u;
                    if (bit) st[p1 + r1] = slot;
                    if (RESET && bit) reset_cmds[slot] = 0u; // stage 3 (kernels.py:256-259)
                    p1 += __popc(word);
                }
            } else { // tiny pool: a single partial block
                const uint32_t nwords = (g.span + 31u) / 32u;
                const uint32_t own = (uint32_t)lane < nwords ? bits32[(size_t)b * 32 + lane] : 0u;
                for (uint32_t w = 0; w < nwords; ++w) {
                    const uint32_t valid = g.span - w * 32u >= 32u ? 32u : g.span - w * 32u;
                    const uint32_t vmask = valid == 32u ? 0xffffffffu : (1u << valid) - 1u;
                    const uint32_t word = __shfl_sync(FULL_MASK, own, (int)w) & vmask;
                    const uint32_t r1 = __popc(word & lane_lt);
                    const int32_t slot = base + (int32_t)(w * 32u) + lane;
                    if ((uint32_t)lane < valid) {
                        if ((word >> lane) & 1u) {
                            st[p1 + r1] = slot;
                            if (RESET) reset_cmds[slot] = 0u;
                        } else if (want_free)
                            st[p0 + (uint32_t)lane - r1] = slot;
                    }
                    const uint32_t c = __popc(word);
                    p1 += c;
                    p0 += valid - c;
                }
            }
            if (BULK && want_free && g.span == 1024u) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); // my staging stores -> async proxy
                __syncwarp();
                bulk_copy_out(cache_live, ones_before - o1, o1, cnt, st, lane);
                bulk_copy_out(cache_free, zeros_before - (zeros_before & 31u), zeros_before & 31u, zcnt, st + zline, lane);
                bulk_copy_out_commit(lane);
                // the next block expands into the other staging area, once the store issued from it two
                // blocks ago has read it (at most one group -- this block's -- stays pending)
                bulk_turn ^= 1u;
                st = stage[2 * warp + bulk_turn];
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                __syncwarp();
                continue;
            }
            __syncwarp();
            copy_out_lines(cache_live, ones_before - o1, o1, cnt, st, lane);
            if (want_free) copy_out_lines(cache_free, zeros_before - (zeros_before & 31u), zeros_before & 31u, zcnt,
                                          st + zline, lane);
            __syncwarp();
        }
    }
    if (BULK && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); // writes done before the warp exits
}

template <bool RESET>
__global__ void __launch_bounds__(IDX_WARPS * 32)
k_index(const uint32_t *bits32, const uint32_t *counters, int depth, int32_t *cache_live,
        int32_t *cache_free, uint32_t *dispatch, uint32_t *reset_cmds)
{
    __shared__ __align__(16) int32_t stage[IDX_WARPS][IDX_STAGE_WORDS];
    griddep_wait(); // (no-ops unless launched with programmatic stream serialization: cbtm_export_live_triangles)
    griddep_launch_dependents();
    index_phase<RESET>(bits32, counters, depth, cache_live, cache_free, dispatch, reset_cmds, stage, blockIdx.x,
                       gridDim.x);
}

// decode-all (both lists, pools of >= 1024 slots): two staging areas per warp, copy-out by TMA bulk
// stores that overlap the expansion of the warp's next block
constexpr size_t IDX_ALL_SMEM = sizeof(int32_t) * 2 * IDX_WARPS * IDX_STAGE_WORDS;
__global__ void __launch_bounds__(IDX_WARPS * 32)
k_index_all(const uint32_t *bits32, const uint32_t *counters, int depth, int32_t *cache_live, int32_t *cache_free,
            uint32_t *dispatch)
{
    extern __shared__ __align__(128) int32_t stage_dyn[];
    index_phase<false, true>(bits32, counters, depth, cache_live, cache_free, dispatch, nullptr,
                             reinterpret_cast<int32_t(*)[IDX_STAGE_WORDS]>(stage_dyn), blockIdx.x, gridDim.x);
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
