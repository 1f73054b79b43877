// cbtm.cu -- C ABI of libcbtm.so (see include/cbtm.h).  Host-side launch logic
// only; the kernels live in the .cuh files next to this one.
//
// Build (see paper_2407_02215_b200/build.py):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false
//        --shared -Xcompiler -fPIC -o libcbtm.so cbtm.cu
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "cbtm_frame.cuh"
#include "cbtm_mesh.cuh"

using namespace cbtm;

namespace {

// Per-device properties, cached per device ordinal (a process may drive several GPUs).
constexpr int MAX_DEVICES = 64;
struct DeviceInfo {
    std::atomic<int> sm_count{0};
    std::atomic<int> index_all_smem_opt_in{0};
    std::atomic<int> frame_ctas_per_sm[2] = {{0}, {0}};
    std::atomic<int> batch_ctas_per_sm{0};
};
DeviceInfo g_devices[MAX_DEVICES];

inline DeviceInfo &device_info()
{
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= MAX_DEVICES) dev = 0;
    return g_devices[dev];
}

inline int sm_count()
{
    DeviceInfo &d = device_info();
    int n = d.sm_count.load(std::memory_order_relaxed);
    if (n == 0) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
            n = 148; // B200
        d.sm_count.store(n, std::memory_order_relaxed); // (racing threads store the same value)
    }
    return n;
}

inline int status(cudaError_t e) { return e == cudaSuccess ? 0 : -(int)e; }
inline int launch_status() { return status(cudaGetLastError()); }
inline bool bad_depth(int d) { return d < CBTM_MIN_DEPTH || d > CBTM_MAX_DEPTH; }
inline cudaStream_t as_stream(uintptr_t s) { return reinterpret_cast<cudaStream_t>(s); }

// grid for kernels that stride over up to `units` work items of `per_cta` each
inline unsigned strided_grid(uint64_t units, uint64_t per_cta, int ctas_per_sm)
{
    uint64_t want = (units + per_cta - 1) / per_cta;
    const uint64_t cap = (uint64_t)sm_count() * ctas_per_sm;
    if (want > cap) want = cap;
    return want ? (unsigned)want : 1u;
}

int reduce_launch(const uint64_t *bits, uint32_t *counters, int depth, unsigned *ticket, cudaStream_t st)
{
    const Geo g = make_geo(depth);
    const unsigned tiles = g.nblocks > (unsigned)RED_TILE_BLOCKS ? g.nblocks / RED_TILE_BLOCKS : 1u;
    const uint64_t total_bytes = (uint64_t)bitfield_words(depth) * 8;
    // one CTA per 16 KB tile (8192 at the ABI's largest pool); the shared-memory heap is only touched
    // by the last CTA of a tree that was never built
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(tiles);
    cfg.blockDim = dim3(RED_THREADS);
    cfg.dynamicSmemBytes = (size_t)(tiles < RED_HEAP_ROOTS ? tiles : RED_HEAP_ROOTS) * 8;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    // programmatic dependent launch: this grid's CTAs may be scheduled while the previous kernel
    // of the stream drains; the kernel prefetches its tiles into L2 and waits (griddepcontrol.wait)
    // before it reads memory
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    static const bool no_pdl = getenv("CBTM_REDUCE_NO_PDL") != nullptr;           // measurement hooks
    static const bool no_prefetch = getenv("CBTM_REDUCE_NO_PREFETCH") != nullptr;
    cfg.attrs = attr;
    cfg.numAttrs = no_pdl ? 0 : 1;
    const bool wide = ((uintptr_t)bits & 31) == 0; // 256-bit loads need 32-byte alignment, the ABI asks for 16
    return status(cudaLaunchKernelEx(&cfg, wide ? k_sum_reduce<true> : k_sum_reduce<false>,
                                     reinterpret_cast<const uint8_t *>(bits), counters, g.lc, total_bytes, tiles, ticket,
                                     no_pdl || no_prefetch ? 0 : 1));
}

int check_pool(const cbtm_pool *p, bool need_ws)
{
    if (!p) return CBTM_E_NULL;
    if (bad_depth(p->depth)) return CBTM_E_DEPTH;
    if (!p->ids || !p->nexts || !p->prevs || !p->twins || !p->commands || !p->reserved ||
        !p->cache_live || !p->cache_free || !p->counter || !p->bits || !p->counters)
        return CBTM_E_NULL;
    if (need_ws) {
        if (!p->workspace) return CBTM_E_NULL;
        if (p->workspace_bytes < carve_workspace(nullptr, p->depth, nullptr)) return CBTM_E_WORKSPACE;
    }
    if (p->rank < 1 || p->rank > 62 || p->max_depth < 0) return CBTM_E_RANGE;
    // 128-bit accesses: reserved rows, index lists, bitfield lines
    // (counters: the ranked descent reads eight sibling counters as two 128-bit loads)
    if (((uintptr_t)p->reserved | (uintptr_t)p->cache_live | (uintptr_t)p->cache_free | (uintptr_t)p->bits |
         (uintptr_t)p->counters) & 15)
        return CBTM_E_ALIGN;
    return 0;
}

int fill_args(const cbtm_pool *pool, const cbtm_verdict *v, FrameArgs *a)
{
    a->pool = *pool;
    carve_workspace(pool->workspace, pool->depth, &a->ws);
    a->use_prm_seq = 0;
    a->pad_ = 0;
    a->vexplicit = nullptr;
    a->root_tris = nullptr;
    a->vmode = CBTM_VERDICT_CONST;
    a->vvalue = 0;
    for (int k = 0; k < CBTM_PRM_WORDS; ++k) a->prm[k] = 0.0;
    if (!v) return 0;
    if (v->mode < CBTM_VERDICT_CONST || v->mode > CBTM_VERDICT_EXPLICIT) return CBTM_E_MODE;
    a->vmode = v->mode;
    a->vvalue = v->value;
    if (v->mode == CBTM_VERDICT_CONST && (v->value < 0 || v->value > 2)) return CBTM_E_MODE;
    if (v->mode == CBTM_VERDICT_EXPLICIT) {
        if (!v->explicit_verdicts) return CBTM_E_NULL;
        a->vexplicit = v->explicit_verdicts;
    }
    if (v->mode == CBTM_VERDICT_LOD) {
        if (!v->root_tris) return CBTM_E_NULL;
        a->root_tris = v->root_tris;
        for (int k = 0; k < CBTM_PRM_WORDS; ++k) a->prm[k] = v->prm[k];
    }
    return 0;
}

unsigned frame_grid(int depth)
{
    return strided_grid((uint64_t)1 << depth, CHUNK, 8);
}

int index_launch(const cbtm_pool *pool, bool reset_commands, cudaStream_t st)
{
    const Geo g = make_geo(pool->depth);
    int32_t *freep = (pool->flags & CBTM_POOL_FULL_FREE_CACHE) ? pool->cache_free : nullptr;
    const unsigned grid = strided_grid(g.nblocks, IDX_WARPS, 6);
    if (reset_commands)
        k_index<true><<<grid, IDX_WARPS * 32, 0, st>>>(reinterpret_cast<const uint32_t *>(pool->bits), pool->counters,
                                                       pool->depth, pool->cache_live, freep, pool->dispatch,
                                                       pool->commands);
    else
        k_index<false><<<grid, IDX_WARPS * 32, 0, st>>>(reinterpret_cast<const uint32_t *>(pool->bits), pool->counters,
                                                        pool->depth, pool->cache_live, freep, pool->dispatch, nullptr);
    return launch_status();
}

int upper_reduce_launch(const FrameArgs &a, int64_t *stats_seq, cudaStream_t st)
{
    const Geo g = make_geo(a.pool.depth);
    const unsigned tiles = g.nblocks > (unsigned)UP_TILE ? g.nblocks / UP_TILE : 1u;
    const unsigned cap = (unsigned)sm_count() * 2;
    k_upper_reduce<<<tiles < cap ? tiles : cap, RED_THREADS, 0, st>>>(a.pool.bits, a.ws.dirty, a.pool.counters, g.lc);
    k_publish<<<1, CHUNK, 0, st>>>(a, stats_seq);
    return launch_status();
}

// stages 3-9, one kernel per phase (staged path).  with_reset: stage 3 was not
// folded into the index kernel (cbtm_update_finish).
int finish_staged(const FrameArgs &a, int64_t *stats_seq, bool with_reset, cudaStream_t st)
{
    const int d = a.pool.depth;
    if (with_reset) k_reset<<<frame_grid(d), CHUNK, 0, st>>>(a);
    k_classify_frame<<<frame_grid(d), CHUNK, 0, st>>>(a);
    k_admit<<<1, CHUNK, 0, st>>>(a);
    k_scatter<<<frame_grid(d), CHUNK, 0, st>>>(a);
    k_agree<<<frame_grid(d), CHUNK, 0, st>>>(a);
    k_reserve<<<frame_grid(d), CHUNK, 0, st>>>(a);
    k_apply<<<frame_grid(d), CHUNK, 0, st>>>(a);
    const int rc = launch_status();
    if (rc) return rc;
    return upper_reduce_launch(a, stats_seq, st);
}

// Co-resident grid of the persistent frame kernel (0: cooperative launch unavailable); wide = 4 CTAs per SM
unsigned persistent_grid(int depth, bool wide = false)
{
    // cached per device as value + 1 (0 = not probed yet); the probe is idempotent, so racing
    // threads store the same number
    std::atomic<int> &slot = device_info().frame_ctas_per_sm[wide ? 1 : 0];
    int cached = slot.load(std::memory_order_acquire) - 1;
    if (cached < 0) {
        const void *kernel = wide ? (const void *)k_frames<4> : (const void *)k_frames<2>;
        const int want_per_sm = wide ? 4 : 2;
        int dev = 0, coop = 0, per_sm = 0;
        cached = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev) == cudaSuccess && coop &&
            cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FRAMES_DYN_SMEM) ==
                cudaSuccess &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, CHUNK, FRAMES_DYN_SMEM) == cudaSuccess)
            cached = per_sm > want_per_sm ? want_per_sm : per_sm;
        (void)cudaGetLastError();
        slot.store(cached + 1, std::memory_order_release);
    }
    if (cached <= 0) return 0;
    const uint64_t want = (((uint64_t)1 << depth) + CHUNK - 1) / CHUNK; // tiny pools: fewer CTAs, cheaper barriers
    const uint64_t cap = (uint64_t)sm_count() * cached;
    return (unsigned)(want < cap ? want : cap);
}

inline bool wide(const cbtm_pool *pool) { return (pool->flags & CBTM_POOL_WIDE_GRID) != 0; }

#ifdef CBTM_DEBUG_TIMING
long long g_launch_ns = 0, g_launch_calls = 0;
#endif

// n_frames full updates (optionally without the index phase) in one cooperative launch; with a
// mailbox: one update, then the kernel lingers for further requests (cbtm_update_linger)
int frames_launch(FrameArgs &a, int n_frames, int64_t *stats_seq, int do_index, unsigned grid, cudaStream_t st,
                  const int64_t *mailbox = nullptr, long long linger_ns = 0, long long next_request = 0)
{
    void *args[] = {(void *)&a,       (void *)&n_frames,  (void *)&stats_seq,   (void *)&do_index,
                    (void *)&mailbox, (void *)&linger_ns, (void *)&next_request};
    const void *kernel = wide(&a.pool) ? (const void *)k_frames<4> : (const void *)k_frames<2>;
    // (cudaLaunchKernelExC with the cooperative attribute: ~1 us less host time per call than
    //  cudaLaunchCooperativeKernel, benchmarks/launch_probe.cu)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(CHUNK);
    cfg.dynamicSmemBytes = FRAMES_DYN_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
#ifdef CBTM_DEBUG_TIMING
    const auto t0 = std::chrono::steady_clock::now();
    const int rc = status(cudaLaunchKernelExC(&cfg, kernel, args));
    g_launch_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
    g_launch_calls += 1;
    return rc;
#else
    return status(cudaLaunchKernelExC(&cfg, kernel, args));
#endif
}

inline bool staged(const cbtm_pool *pool) { return (pool->flags & CBTM_POOL_STAGED_LAUNCHES) != 0; }

} // namespace

extern "C" {

int cbtm_abi_version(void) { return CBTM_ABI_VERSION; }

size_t cbtm_bitfield_words(int depth) { return bad_depth(depth) ? 0 : bitfield_words(depth); }

size_t cbtm_counter_words(int depth) { return bad_depth(depth) ? 0 : counter_words(depth); }

size_t cbtm_workspace_bytes(int depth)
{
    return bad_depth(depth) ? 0 : carve_workspace(nullptr, depth, nullptr);
}

size_t cbtm_cbt_workspace_bytes(int depth) { return bad_depth(depth) ? 0 : 256; }

int cbtm_sum_reduce(const uint64_t *bits, uint32_t *counters, int depth, void *workspace,
                    size_t workspace_bytes, uintptr_t stream)
{
    if (bad_depth(depth)) return CBTM_E_DEPTH;
    if (!bits || !counters || !workspace) return CBTM_E_NULL;
    if (((uintptr_t)bits | (uintptr_t)counters) & 15) return CBTM_E_ALIGN; // bulk prefetch, 128-bit loads
    if (workspace_bytes < 256) return CBTM_E_WORKSPACE;
    // word 0 of the workspace (also of a pool's frame workspace) is the ticket of the rebuild path;
    // it must be zero on entry and the kernel leaves it zero again
    return reduce_launch(bits, counters, depth, reinterpret_cast<unsigned *>(workspace), as_stream(stream));
}

#ifdef CBTM_DEBUG_TIMING
// debug builds only (benchmarks/reduce_probe.py): per-CTA stamps of the last k_sum_reduce launch
extern "C" long long cbtm_debug_launch_ns(int reset)
{
    const long long avg = g_launch_calls ? g_launch_ns / g_launch_calls : 0;
    if (reset) g_launch_ns = g_launch_calls = 0;
    return avg;
}
extern "C" int cbtm_debug_probes(unsigned long long *host_out, int reset)
{
    int rc = status(cudaMemcpyFromSymbol(host_out, g_probe, sizeof(g_probe)));
    if (rc == 0 && reset) {
        static unsigned long long zeros[PROBE_FRAMES][PROBE_SLOTS];
        rc = status(cudaMemcpyToSymbol(g_probe, zeros, sizeof(zeros)));
    }
    return rc;
}
extern "C" int cbtm_debug_reduce_stamps(unsigned long long *host_out, int n_ctas)
{
    return status(cudaMemcpyFromSymbol(host_out, g_reduce_stamps, sizeof(unsigned long long) * 5 * n_ctas));
}
#endif

int cbtm_decode_ones(const uint64_t *bits, const uint32_t *counters, int depth, const int64_t *ranks,
                     int64_t K, int32_t *out, uintptr_t stream)
{
    if (bad_depth(depth)) return CBTM_E_DEPTH;
    if (!bits || !counters || (K > 0 && !out)) return CBTM_E_NULL;
    if (K < 0) return CBTM_E_RANGE;
    if (((uintptr_t)bits | (uintptr_t)counters) & 15) return CBTM_E_ALIGN; // 128-bit loads of lines / sibling counters
    if (K == 0) return 0;
    const unsigned grid = strided_grid((uint64_t)K, 256, 8);
    if ((((uintptr_t)bits | (uintptr_t)counters) & 31) == 0) // 32-byte aligned: 256-bit loads
        k_decode<true, true><<<grid, 256, 0, as_stream(stream)>>>(bits, counters, depth, ranks, K, out);
    else
        k_decode<true, false><<<grid, 256, 0, as_stream(stream)>>>(bits, counters, depth, ranks, K, out);
    return launch_status();
}

int cbtm_decode_zeros(const uint64_t *bits, const uint32_t *counters, int depth, const int64_t *ranks,
                      int64_t K, int32_t *out, uintptr_t stream)
{
    if (bad_depth(depth)) return CBTM_E_DEPTH;
    if (!bits || !counters || (K > 0 && !out)) return CBTM_E_NULL;
    if (K < 0) return CBTM_E_RANGE;
    if (((uintptr_t)bits | (uintptr_t)counters) & 15) return CBTM_E_ALIGN; // 128-bit loads of lines / sibling counters
    if (K == 0) return 0;
    const unsigned grid = strided_grid((uint64_t)K, 256, 8);
    if ((((uintptr_t)bits | (uintptr_t)counters) & 31) == 0)
        k_decode<false, true><<<grid, 256, 0, as_stream(stream)>>>(bits, counters, depth, ranks, K, out);
    else
        k_decode<false, false><<<grid, 256, 0, as_stream(stream)>>>(bits, counters, depth, ranks, K, out);
    return launch_status();
}

int cbtm_index(const uint64_t *bits, const uint32_t *counters, int depth, int32_t *cache_live,
               int32_t *cache_free, uint32_t *dispatch, uintptr_t stream)
{
    if (bad_depth(depth)) return CBTM_E_DEPTH;
    if (!bits || !counters || !cache_live) return CBTM_E_NULL;
    if (((uintptr_t)bits | (uintptr_t)counters | (uintptr_t)cache_live | (uintptr_t)cache_free) & 15) return CBTM_E_ALIGN;
    const Geo g = make_geo(depth);
    if (cache_free && g.span == 1024u) { // decode-all: double-buffered staging, TMA bulk stores
        DeviceInfo &d = device_info();
        if (!d.index_all_smem_opt_in.load(std::memory_order_acquire)) {
            const cudaError_t e = cudaFuncSetAttribute(k_index_all, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       (int)IDX_ALL_SMEM);
            if (e != cudaSuccess) return status(e);
            d.index_all_smem_opt_in.store(1, std::memory_order_release);
        }
        k_index_all<<<strided_grid(g.nblocks, IDX_WARPS, 3), IDX_WARPS * 32, IDX_ALL_SMEM, as_stream(stream)>>>(
            reinterpret_cast<const uint32_t *>(bits), counters, depth, cache_live, cache_free, dispatch);
        return launch_status();
    }
    k_index<false><<<strided_grid(g.nblocks, IDX_WARPS, 6), IDX_WARPS * 32, 0, as_stream(stream)>>>(
        reinterpret_cast<const uint32_t *>(bits), counters, depth, cache_live, cache_free, dispatch, nullptr);
    return launch_status();
}

int cbtm_import_leaves(uint64_t *bits, int depth, const uint32_t *leaves, uintptr_t stream)
{
    if (bad_depth(depth)) return CBTM_E_DEPTH;
    if (!bits || !leaves) return CBTM_E_NULL;
    k_import_leaves<<<strided_grid(bitfield_words(depth) * 2, 256, 8), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<uint32_t *>(bits), depth, leaves);
    return launch_status();
}

int cbtm_export_nodes(const uint64_t *bits, const uint32_t *counters, int depth, uint32_t *nodes,
                      uintptr_t stream)
{
    if (bad_depth(depth)) return CBTM_E_DEPTH;
    if (!bits || !counters || !nodes) return CBTM_E_NULL;
    k_export_nodes<<<strided_grid((uint64_t)2 << depth, 256, 8), 256, 0, as_stream(stream)>>>(
        bits, counters, depth, nodes);
    return launch_status();
}

int cbtm_initialize(const cbtm_pool *pool, const int32_t *he_next, const int32_t *he_prev,
                    const int32_t *he_twin, int32_t n_halfedges, uintptr_t stream)
{
    int rc = check_pool(pool, true);
    if (rc) return rc;
    if (!he_next || !he_prev || !he_twin) return CBTM_E_NULL;
    if (n_halfedges < 1 || ((int64_t)n_halfedges > ((int64_t)1 << pool->depth))) return CBTM_E_RANGE;
    Workspace ws;
    carve_workspace(pool->workspace, pool->depth, &ws);
    cudaStream_t st = as_stream(stream);
    k_initialize<<<strided_grid((uint64_t)1 << pool->depth, 256, 8), 256, 0, st>>>(
        *pool, he_next, he_prev, he_twin, n_halfedges, ws);
    rc = launch_status();
    if (rc) return rc;
    return reduce_launch(pool->bits, pool->counters, pool->depth, ws.ticket, st);
}

int cbtm_root_triangles(const int32_t *he_next, const int32_t *he_vert, const double *positions,
                        int32_t n_halfedges, double *out, uintptr_t stream)
{
    if (!he_next || !he_vert || !positions || !out) return CBTM_E_NULL;
    if (n_halfedges < 1) return CBTM_E_RANGE;
    k_root_triangles<<<(n_halfedges + 127) / 128, 128, 0, as_stream(stream)>>>(he_next, he_vert, positions,
                                                                              n_halfedges, out);
    return launch_status();
}

int cbtm_classify(const cbtm_pool *pool, const cbtm_verdict *verdict, int8_t *verdicts, uintptr_t stream)
{
    int rc = check_pool(pool, true);
    if (rc) return rc;
    if (!verdict || !verdicts) return CBTM_E_NULL;
    FrameArgs a;
    rc = fill_args(pool, verdict, &a);
    if (rc) return rc;
    k_classify<<<frame_grid(pool->depth), CHUNK, 0, as_stream(stream)>>>(a, verdicts);
    return launch_status();
}

int cbtm_decode_triangles(const uint64_t *ids, int64_t K, int32_t rank, const double *root_tris,
                          double *out, uintptr_t stream)
{
    if (!ids || !root_tris || !out) return CBTM_E_NULL;
    if (K < 0 || rank < 1) return CBTM_E_RANGE;
    if (K == 0) return 0;
    k_decode_triangles<<<strided_grid((uint64_t)K, 256, 8), 256, 0, as_stream(stream)>>>(ids, K, rank,
                                                                                       root_tris, out);
    return launch_status();
}

int cbtm_export_live_triangles(const cbtm_pool *pool, const double *root_tris, double *out, int64_t out_capacity,
                               uint32_t *draw_args, uintptr_t stream)
{
    int rc = check_pool(pool, false);
    if (rc) return rc;
    if (!root_tris || !out) return CBTM_E_NULL;
    if (out_capacity < 0) return CBTM_E_RANGE;
    cudaStream_t st = as_stream(stream);
    // the active list of the CURRENT state (an update leaves the list of the state it started from)
    // both launches with programmatic stream serialization: each grid is set up while the kernel before it
    // on the stream (the frame kernel; the index pass) drains, and waits in griddepcontrol.wait
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(strided_grid(make_geo(pool->depth).nblocks, IDX_WARPS, 6));
    cfg.blockDim = dim3(IDX_WARPS * 32);
    rc = status(cudaLaunchKernelEx(&cfg, k_index<false>, reinterpret_cast<const uint32_t *>(pool->bits),
                                   (const uint32_t *)pool->counters, (int)pool->depth, pool->cache_live, (int32_t *)nullptr,
                                   pool->dispatch, (uint32_t *)nullptr));
    if (rc) return rc;
    const uint64_t cap = (uint64_t)out_capacity < ((uint64_t)1 << pool->depth) ? (uint64_t)out_capacity
                                                                               : ((uint64_t)1 << pool->depth);
    cfg.gridDim = dim3(strided_grid(cap ? cap : 1, 256, 8));
    cfg.blockDim = dim3(256);
    return status(cudaLaunchKernelEx(&cfg, k_export_live_triangles, (const uint64_t *)pool->ids,
                                     (const int32_t *)pool->cache_live, (const uint32_t *)pool->counters, (int)pool->rank,
                                     root_tris, out, (uint64_t)out_capacity, draw_args));
}

int cbtm_validate(const cbtm_pool *pool, int32_t n_halfedges, int64_t *out, uintptr_t stream)
{
    int rc = check_pool(pool, false);
    if (rc) return rc;
    if (!out) return CBTM_E_NULL;
    if (n_halfedges < 1) return CBTM_E_RANGE;
    cudaStream_t st = as_stream(stream);
    // words 0..5 and 7 start at 0, word 6 (first offending slot, taken with atomicMin) at ~0
    rc = status(cudaMemsetAsync(out, 0, sizeof(int64_t) * CBTM_VALIDATE_WORDS, st));
    if (rc) return rc;
    rc = status(cudaMemsetAsync(out + 6, 0xff, sizeof(int64_t), st));
    if (rc) return rc;
    k_validate<<<strided_grid((uint64_t)1 << pool->depth, 256, 8), 256, 0, st>>>(
        *pool, n_halfedges, reinterpret_cast<unsigned long long *>(out));
    return launch_status();
}

int cbtm_update_begin(const cbtm_pool *pool, uintptr_t stream)
{
    const int rc = check_pool(pool, true);
    if (rc) return rc;
    return index_launch(pool, false, as_stream(stream));
}

int cbtm_update_finish(const cbtm_pool *pool, const cbtm_verdict *verdict, uintptr_t stream)
{
    int rc = check_pool(pool, true);
    if (rc) return rc;
    if (!verdict) return CBTM_E_NULL;
    FrameArgs a;
    rc = fill_args(pool, verdict, &a);
    if (rc) return rc;
    const unsigned grid = staged(pool) ? 0 : persistent_grid(pool->depth, wide(pool));
    if (!grid) return finish_staged(a, nullptr, true, as_stream(stream));
    return frames_launch(a, 1, nullptr, 0, grid, as_stream(stream));
}

int cbtm_update(const cbtm_pool *pool, const cbtm_verdict *verdict, uintptr_t stream)
{
    int rc = check_pool(pool, true);
    if (rc) return rc;
    if (!verdict) return CBTM_E_NULL;
    FrameArgs a;
    rc = fill_args(pool, verdict, &a);
    if (rc) return rc;
    const unsigned grid = staged(pool) ? 0 : persistent_grid(pool->depth, wide(pool));
    if (!grid) {
        rc = index_launch(pool, true, as_stream(stream));
        return rc ? rc : finish_staged(a, nullptr, false, as_stream(stream));
    }
    return frames_launch(a, 1, nullptr, 1, grid, as_stream(stream));
}

size_t cbtm_mesh_workspace_bytes(int64_t n_halfedges)
{
    if (n_halfedges < 1 || n_halfedges > 0x7fffffff) return 0;
    return carve_mesh_scratch(nullptr, n_halfedges, nullptr);
}

int cbtm_mesh_from_polygons(const int32_t *face_offsets, const int32_t *face_verts, int32_t n_faces,
                            int32_t n_halfedges, int32_t n_vertices, int32_t *he_twin, int32_t *he_next,
                            int32_t *he_prev, int32_t *he_vert, int32_t *he_edge, int32_t *he_face,
                            int64_t *status_out, void *workspace, size_t workspace_bytes, uintptr_t stream)
{
    if (!face_offsets || !face_verts || !he_twin || !he_next || !he_prev || !he_vert || !he_edge || !he_face ||
        !status_out || !workspace)
        return CBTM_E_NULL;
    if (n_faces < 1 || n_halfedges < 1 || n_vertices < 1) return CBTM_E_RANGE;
    if (workspace_bytes < carve_mesh_scratch(nullptr, n_halfedges, nullptr)) return CBTM_E_WORKSPACE;
    cudaStream_t st = as_stream(stream);
    MeshScratch m;
    carve_mesh_scratch(workspace, n_halfedges, &m);
    unsigned long long *d_status = reinterpret_cast<unsigned long long *>(status_out);
    int rc = status(cudaMemsetAsync(status_out, 0, sizeof(int64_t) * CBTM_MESH_STATUS_WORDS, st));
    if (rc) return rc;
    rc = status(cudaMemsetAsync(status_out + MESH_FIRST_FACE, 0xff, 2 * sizeof(int64_t), st)); // atomicMin targets
    if (rc) return rc;
    k_mesh_faces<<<strided_grid((uint64_t)n_faces, 256, 8), 256, 0, st>>>(face_offsets, face_verts, n_faces, n_vertices,
                                                                        he_next, he_prev, he_vert, he_face, m.keys_a,
                                                                        m.vals_a, d_status);
    rc = launch_status();
    if (rc) return rc;
    int vbits = 1;
    while (vbits < 32 && ((int64_t)1 << vbits) < (int64_t)n_vertices) ++vbits;
    size_t tmp = m.cub_bytes;
    rc = status(cub::DeviceRadixSort::SortPairs(m.cub_tmp, tmp, m.keys_a, m.keys_b, m.vals_a, m.vals_b, n_halfedges, 0,
                                                32 + vbits, st));
    if (rc) return rc;
    k_mesh_run_starts<<<strided_grid((uint64_t)n_halfedges, 256, 8), 256, 0, st>>>(m.keys_b, n_halfedges, m.starts);
    tmp = m.cub_bytes;
    rc = status(cub::DeviceScan::ExclusiveSum(m.cub_tmp, tmp, m.starts, m.ranks, n_halfedges, st));
    if (rc) return rc;
    k_mesh_twins<<<strided_grid((uint64_t)n_halfedges, 256, 8), 256, 0, st>>>(m.keys_b, m.vals_b, m.starts, m.ranks,
                                                                            n_halfedges, he_vert, he_twin, he_edge,
                                                                            d_status);
    return launch_status();
}

static int wait_word(const int64_t *host_stats, int word, int64_t frame, uint64_t timeout_ns)
{
    if (!host_stats) return CBTM_E_NULL;
    const volatile int64_t *seq = host_stats + word;
    if (*seq >= frame) return 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (unsigned spins = 0;; ++spins) {
        if (*seq >= frame) break;
        if ((spins & 1023u) == 1023u &&
            (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count() >
                timeout_ns)
            return CBTM_E_TIMEOUT;
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    return 0;
}

int cbtm_wait_frame(const int64_t *host_stats, int64_t frame, uint64_t timeout_ns)
{
    return wait_word(host_stats, CBTM_STAT_SEQ, frame, timeout_ns);
}

int cbtm_wait_frame_done(const int64_t *host_stats, int64_t frame, uint64_t timeout_ns)
{
    return wait_word(host_stats, CBTM_STAT_DONE, frame, timeout_ns);
}

int cbtm_update_wait(const cbtm_pool *pool, const cbtm_verdict *verdict, const int64_t *host_stats,
                     uint64_t timeout_ns, uintptr_t stream)
{
    if (!host_stats) return CBTM_E_NULL;
    const int64_t frame = *(const volatile int64_t *)(host_stats + CBTM_STAT_SEQ) + 1;
    const int rc = cbtm_update(pool, verdict, stream);
    if (rc) return rc;
    return wait_word(host_stats, CBTM_STAT_SEQ, frame, timeout_ns);
}

int cbtm_run_epochs(const cbtm_pool *pool, const cbtm_verdict *verdict, int32_t n_frames, int64_t *stats_out,
                    uintptr_t stream)
{
    int rc = check_pool(pool, true);
    if (rc) return rc;
    if (!verdict) return CBTM_E_NULL;
    if (verdict->mode == CBTM_VERDICT_EXPLICIT) return CBTM_E_MODE; // explicit verdicts are per frame
    if (n_frames < 0) return CBTM_E_RANGE;
    cudaStream_t st = as_stream(stream);
    FrameArgs a;
    rc = fill_args(pool, verdict, &a);
    if (rc) return rc;
    const unsigned grid = staged(pool) ? 0 : persistent_grid(pool->depth, wide(pool));
    for (int32_t done = 0; done < n_frames;) {
        const int32_t batch = n_frames - done < MAX_SEQ_FRAMES ? n_frames - done : MAX_SEQ_FRAMES;
        rc = status(cudaMemsetAsync(&a.ws.ctl->seq_frame, 0, sizeof(uint32_t), st));
        if (rc) return rc;
        int64_t *so = stats_out ? stats_out + (size_t)CBTM_STATS_WORDS * done : nullptr;
        if (grid) {
            rc = frames_launch(a, batch, so, 1, grid, st);
            if (rc) return rc;
        } else {
            for (int32_t f = 0; f < batch; ++f) {
                rc = index_launch(pool, true, st);
                if (rc) return rc;
                rc = finish_staged(a, so, false, st);
                if (rc) return rc;
            }
        }
        done += batch;
    }
    return 0;
}

int cbtm_update_linger(const cbtm_pool *pool, const cbtm_verdict *verdict, const int64_t *mailbox, int64_t request,
                       int64_t linger_ns, uintptr_t stream)
{
    int rc = check_pool(pool, true);
    if (rc) return rc;
    if (!verdict || !mailbox) return CBTM_E_NULL;
    if (verdict->mode != CBTM_VERDICT_LOD) return CBTM_E_MODE; // later requests carry camera parameters only
    if (request < 1 || linger_ns < 0 || linger_ns > 100000000) return CBTM_E_RANGE; // at most 100 ms
    FrameArgs a;
    rc = fill_args(pool, verdict, &a);
    if (rc) return rc;
    const unsigned grid = staged(pool) ? 0 : persistent_grid(pool->depth, wide(pool));
    if (!grid) { // no cooperative launch: a plain update, nothing lingers
        rc = index_launch(pool, true, as_stream(stream));
        return rc ? rc : finish_staged(a, nullptr, false, as_stream(stream));
    }
    rc = status(cudaMemsetAsync(&a.ws.ctl->seq_frame, 0, sizeof(uint32_t), as_stream(stream)));
    if (rc) return rc;
    return frames_launch(a, 1, nullptr, 1, grid, as_stream(stream), mailbox, linger_ns, request + 1);
}

int cbtm_post_request(int64_t *mailbox_host, int64_t request, const double *prm)
{
    if (!mailbox_host || !prm) return CBTM_E_NULL;
    for (int k = 0; k < CBTM_PRM_WORDS; ++k) {
        int64_t bits;
        memcpy(&bits, &prm[k], sizeof bits);
        reinterpret_cast<volatile int64_t *>(mailbox_host)[8 + k] = bits;
    }
    std::atomic_thread_fence(std::memory_order_release);
    reinterpret_cast<volatile int64_t *>(mailbox_host)[0] = request;
    return 0;
}

int cbtm_run_lod_sequence(const cbtm_pool *pool, const double *root_tris, const double *prm_host,
                          int32_t n_frames, int64_t *stats_out, uintptr_t stream)
{
    int rc = check_pool(pool, true);
    if (rc) return rc;
    if (!root_tris || !prm_host) return CBTM_E_NULL;
    if (n_frames < 0) return CBTM_E_RANGE;
    cudaStream_t st = as_stream(stream);
    cbtm_verdict v;
    v.mode = CBTM_VERDICT_LOD;
    v.value = 0;
    v.explicit_verdicts = nullptr;
    v.root_tris = root_tris;
    for (int k = 0; k < CBTM_PRM_WORDS; ++k) v.prm[k] = 0.0;
    FrameArgs a;
    rc = fill_args(pool, &v, &a);
    if (rc) return rc;
    a.use_prm_seq = 1;
    const unsigned grid = staged(pool) ? 0 : persistent_grid(pool->depth, wide(pool));
    for (int32_t done = 0; done < n_frames;) {
        const int32_t batch = n_frames - done < MAX_SEQ_FRAMES ? n_frames - done : MAX_SEQ_FRAMES;
        rc = status(cudaMemcpyAsync(a.ws.prm_seq, prm_host + (size_t)CBTM_PRM_WORDS * done,
                                    sizeof(double) * CBTM_PRM_WORDS * batch, cudaMemcpyHostToDevice, st));
        if (rc) return rc;
        rc = status(cudaMemsetAsync(&a.ws.ctl->seq_frame, 0, sizeof(uint32_t), st));
        if (rc) return rc;
        int64_t *so = stats_out ? stats_out + (size_t)CBTM_STATS_WORDS * done : nullptr;
        if (grid) {
            rc = frames_launch(a, batch, so, 1, grid, st); // the whole batch in one launch
            if (rc) return rc;
        } else {
            for (int32_t f = 0; f < batch; ++f) {
                rc = index_launch(pool, true, st);
                if (rc) return rc;
                rc = finish_staged(a, so, false, st);
                if (rc) return rc;
            }
        }
        done += batch;
    }
    return 0;
}

int cbtm_run_lod_sequence_batch(const cbtm_pool *pools, int32_t n_pools, const double *const *root_tris,
                                const double *const *prm_host, int32_t n_frames, int64_t *const *stats_out,
                                uintptr_t stream)
{
    if (!pools || !root_tris || !prm_host) return CBTM_E_NULL;
    if (n_pools < 1 || n_pools > CBTM_MAX_BATCH || n_frames < 0 || n_frames > MAX_SEQ_FRAMES) return CBTM_E_RANGE;
    cudaStream_t st = as_stream(stream);
    BatchArgs b; // passed by value
    int max_depth = 0;
    bool any_staged = false;
    for (int q = 0; q < n_pools; ++q) {
        int rc = check_pool(&pools[q], true);
        if (rc) return rc;
        if (!root_tris[q] || !prm_host[q]) return CBTM_E_NULL;
        for (int r = 0; r < q; ++r)
            if (pools[r].workspace == pools[q].workspace || pools[r].bits == pools[q].bits) return CBTM_E_RANGE;
        cbtm_verdict v;
        v.mode = CBTM_VERDICT_LOD;
        v.value = 0;
        v.explicit_verdicts = nullptr;
        v.root_tris = root_tris[q];
        for (int k = 0; k < CBTM_PRM_WORDS; ++k) v.prm[k] = 0.0;
        rc = fill_args(&pools[q], &v, &b.a[q]);
        if (rc) return rc;
        b.a[q].use_prm_seq = 1;
        b.stats_seq[q] = stats_out ? stats_out[q] : nullptr;
        if (pools[q].depth > max_depth) max_depth = pools[q].depth;
        any_staged |= staged(&pools[q]);
    }
    if (n_frames == 0) return 0;
    // co-resident CTAs per SM of the batch kernel (0: no cooperative launch); per device, value + 1
    std::atomic<int> &batch_slot = device_info().batch_ctas_per_sm;
    int batch_per_sm = batch_slot.load(std::memory_order_acquire) - 1;
    if (batch_per_sm < 0) {
        int per_sm = 0;
        batch_per_sm = 0;
        if (persistent_grid(max_depth) != 0 &&
            cudaFuncSetAttribute(k_frames_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, FRAMES_DYN_SMEM) ==
                cudaSuccess &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_frames_batch, CHUNK, FRAMES_DYN_SMEM) ==
                cudaSuccess)
            batch_per_sm = per_sm > BATCH_CTAS_PER_SM ? BATCH_CTAS_PER_SM : per_sm;
        (void)cudaGetLastError();
        batch_slot.store(batch_per_sm + 1, std::memory_order_release);
    }
    const int batch_ok = batch_per_sm > 0;
    if (!batch_ok || any_staged || n_pools == 1) { // one pool after the other (same results)
        for (int q = 0; q < n_pools; ++q) {
            const int rc = cbtm_run_lod_sequence(&pools[q], root_tris[q], prm_host[q], n_frames,
                                                 stats_out ? stats_out[q] : nullptr, stream);
            if (rc) return rc;
        }
        return 0;
    }
    for (int q = 0; q < n_pools; ++q) {
        int rc = status(cudaMemcpyAsync(b.a[q].ws.prm_seq, prm_host[q], sizeof(double) * CBTM_PRM_WORDS * n_frames,
                                        cudaMemcpyHostToDevice, st));
        if (rc) return rc;
        rc = status(cudaMemsetAsync(&b.a[q].ws.ctl->seq_frame, 0, sizeof(uint32_t), st));
        if (rc) return rc;
    }
    uint64_t want = 0; // chunks of all pools if every slot were live: tiny pools get a small grid
    for (int q = 0; q < n_pools; ++q) want += (((uint64_t)1 << pools[q].depth) + CHUNK - 1) / CHUNK;
    const uint64_t cap = (uint64_t)sm_count() * batch_per_sm;
    const unsigned grid = (unsigned)(want < cap ? want : cap);
    void *args[] = {(void *)&b, (void *)&n_pools, (void *)&n_frames};
    return status(cudaLaunchCooperativeKernel((const void *)k_frames_batch, dim3(grid), dim3(CHUNK), args,
                                              FRAMES_DYN_SMEM, st));
}

} // extern "C"
