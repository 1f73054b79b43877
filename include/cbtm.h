/*
 * cbtm.h -- C ABI of libcbtm.so: the B200 (sm_100a) implementation of the
 * per-frame bisector update of arXiv 2407.02215.
 *
 * The reference (`cbtmesh`, pure Python + numba) has no FFI of its own; the
 * seam it offers is its Python API.  Each entry point below names the reference
 * interface it stands in for (paths relative to /root/reference/pkg/src/cbtmesh).
 * INTEGRATION.md shows the ctypes binding a maintainer would add.
 *
 * Conventions
 *   - extern "C", plain pointers and sizes only.  Unless stated otherwise every
 *     pointer is a DEVICE pointer owned by the caller; `stream` is a
 *     cudaStream_t passed as uintptr_t (0 = default stream).
 *   - Calls are asynchronous on `stream`, never synchronise the host, never
 *     allocate device memory (scratch is caller-provided, sized by
 *     cbtm_workspace_bytes) and never throw.
 *   - Return value: 0 ok; < 0 is -(cudaError_t); > 0 is a CBTM_E_* contract
 *     violation detected on the host before anything was launched.
 *   - There is no CPU fallback.  Without a CUDA device every compute entry
 *     point fails with a negative status.
 *
 * CBT storage: a packed bitfield, 1 bit per pool slot (bit s of
 * the field = slot s; little-endian inside 64-bit words), plus 32-bit counters
 * for every tree node that spans >= 1024 slots, laid out as a binary heap:
 * node i of level l (root = level 0) lives at counters[(1 << l) + i].  The
 * deepest counter level is Lc = max(D - 10, 0); below it a node is a 128-byte
 * line of the bitfield and is resolved with popcounts.
 */
#ifndef CBTM_H_
#define CBTM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CBTM_ABI_VERSION 2
#define CBTM_MIN_DEPTH 1
#define CBTM_MAX_DEPTH 30 /* slot indices are int32; counters are uint32 */
#define CBTM_LEAF_BLOCK_LOG2 10
#define CBTM_STATS_WORDS 32
#define CBTM_PRM_WORDS 23
#define CBTM_MAX_BATCH 8 /* pools per cbtm_run_lod_sequence_batch call */

/* contract violations */
#define CBTM_E_DEPTH 1     /* depth outside [CBTM_MIN_DEPTH, CBTM_MAX_DEPTH] */
#define CBTM_E_NULL 2      /* a required pointer is NULL */
#define CBTM_E_WORKSPACE 3 /* workspace smaller than cbtm_workspace_bytes */
#define CBTM_E_MODE 4      /* unknown verdict mode / flag */
#define CBTM_E_RANGE 5     /* count / size argument out of range */
#define CBTM_E_ALIGN 6     /* bits, counters, reserved, cache_live, cache_free must be 16-byte aligned
                              (32-byte aligned bits / counters select the 256-bit-load kernel variants) */
#define CBTM_E_TIMEOUT 7   /* cbtm_wait_frame gave up */

/* command-word bits (state.py:17-25) */
#define CBTM_CMD_SPLIT_T 1u
#define CBTM_CMD_SPLIT_N 2u
#define CBTM_CMD_SPLIT_P 4u
#define CBTM_CMD_SPLIT_MASK 7u
#define CBTM_CMD_MERGE 8u
#define CBTM_CMD_QUAD 16u
#define CBTM_CMD_OWNER 32u

/* cbtm_pool.flags */
#define CBTM_POOL_FULL_FREE_CACHE 1u /* materialise cache_free[0, F) every frame
                                        (whole-array parity with the reference);
                                        default: only the consumed window
                                        cache_free[T - A, T) is written */
#define CBTM_POOL_DESCEND_FREE_RANKS 4u /* resolve the frame's free ranks by tree descent (k-th unset
                                          bit per slot) instead of through the window table -- the path
                                          taken automatically when a frame's allocations span more than
                                          4096 leaf blocks; the flag exists so that tests can exercise it */
#define CBTM_POOL_WIDE_GRID 8u /* persistent frame kernel with 4 instead of 2 CTAs per SM: pays off from
                                 ~10^5 live bisectors on (each CTA then works through several chunks of
                                 256 ranks per phase); same results */
#define CBTM_POOL_FINAL_ROW 16u /* cbtm_update also writes the frame's COMPLETE stats row (poison count of this
                                  frame, times of all six phases) and CBTM_STAT_DONE to pool->stats when the
                                  frame has been reduced.  Default for a single-frame launch: only the early
                                  row (see CBTM_STAT_SEQ) -- the kernel then ends with its reduction, without a
                                  device-wide barrier and a host write behind it; a poison count (an error
                                  condition, 0 by construction) is carried over into the next frame's row */
#define CBTM_POOL_STAGED_LAUNCHES 2u /* one kernel launch per pipeline stage instead of
                                        the persistent cooperative frame kernel (per-stage
                                        profiling; automatic where cooperative launch is
                                        unavailable) */

/* stats layout written by cbtm_update to cbtm_pool.stats (int64) */
enum {
    CBTM_STAT_OOM_SPLITS = 0,  /* UpdateStats.splits_rejected_oom */
    CBTM_STAT_OOM_MERGES = 1,  /* UpdateStats.merges_rejected_oom */
    CBTM_STAT_SPLIT_FREED = 2, /* UpdateStats.splits_applied      */
    CBTM_STAT_MERGE_FREED = 3, /* UpdateStats.merges_applied      */
    CBTM_STAT_SPLIT_ALLOC = 4, /* UpdateStats.split_allocs        */
    CBTM_STAT_MERGE_ALLOC = 5, /* UpdateStats.merge_allocs        */
    CBTM_STAT_LIVE_BEFORE = 6,
    CBTM_STAT_LIVE_AFTER = 7,
    CBTM_STAT_RESERVED = 8,  /* T: slots reserved by admitted commands   */
    CBTM_STAT_ALLOCATED = 9, /* A: slots actually allocated              */
    CBTM_STAT_POISON = 10,   /* fresh pointers resolved to the poison -2 */
    CBTM_STAT_FRAME = 11,    /* frames applied to this pool so far       */
    CBTM_STAT_PEAK_DEPTH = 12, /* deepest live bisector at the start of the frame (the per-frame
                                * reduction cmd_animate does on the host, cli.py:232-237)   */
    CBTM_STAT_SEQ = 31,      /* = CBTM_STAT_FRAME, but stored LAST: the other words are written, then a
                              * system-scope fence, then this one -- so when cbtm_pool.stats points to
                              * host-mapped pinned memory the host may poll this word (cbtm_wait_frame)
                              * and then read the frame's counters without any stream synchronisation.
                              * cbtm_update publishes the counters of its frame EARLY: as soon as every
                              * command is final (after stage 5a: admission, split masks, merge agreement
                              * and allocation counts decide all of them; live_after = live_before -
                              * freed + allocated), while stages 5b-9 are still running on the stream --
                              * the host-side work between two frames overlaps with them and the next
                              * launch is queued behind a running kernel.  Not in that early copy: this
                              * frame's poison count and the times of phases 4-6 (words 19-21); with
                              * CBTM_POOL_FINAL_ROW (and in multi-frame launches) the complete row follows
                              * at the end of the frame: */
    CBTM_STAT_DONE = 30,     /* = CBTM_STAT_FRAME, stored after the frame's reduction and the complete
                              * row (cbtm_wait_frame_done; single-frame launches: needs CBTM_POOL_FINAL_ROW) */
    /* words 16..21: device time of each phase of the frame in ns (persistent
     * frame kernel only; 0 on the staged path): index (stages 1-3), classify +
     * admission + command scatter (stage 4), merge agreement (stage 5a), slot
     * hand-out (stage 5b), apply (stages 6-8), sum reduction + stats publish
     * (stage 9) -- cf. UpdateStats.stage_times_us */
    CBTM_STAT_PHASE_NS = 16,
    CBTM_STAT_PHASES = 6
};

/* One bisector pool == the reference's TriangulationState (state.py:32-55).
 * Array shapes, N = 2^depth:
 *   ids u64[N]; nexts/prevs/twins i32[N] (-1 = null); commands u32[N];
 *   reserved i32[N*4]; cache_live/cache_free i32[N]; counter i64[1];
 *   bits u64[cbtm_bitfield_words(depth)]; counters u32[cbtm_counter_words(depth)];
 *   stats i64[CBTM_STATS_WORDS]; dispatch u32[4] = {ceil(n/256), 1, 1, n}
 *   (indirect-dispatch arguments for the consumer of cache_live; may be NULL). */
typedef struct cbtm_pool {
    uint64_t *ids;
    int32_t *nexts;
    int32_t *prevs;
    int32_t *twins;
    uint32_t *commands;
    int32_t *reserved;
    int32_t *cache_live;
    int32_t *cache_free;
    int64_t *counter;
    uint64_t *bits;
    uint32_t *counters;
    int64_t *stats;
    uint32_t *dispatch;
    void *workspace;
    size_t workspace_bytes;
    int32_t depth;     /* D, pool capacity 2^D */
    int32_t rank;      /* R = max(1, ceil(log2 H)): root ids are 2^R + h */
    int32_t max_depth; /* split demotion limit (state.max_depth, 63 - R) */
    uint32_t flags;    /* CBTM_POOL_* */
} cbtm_pool;

/* Verdict source for stage 4 (pipeline.py:87-119, lod.py:272-312). */
enum {
    CBTM_VERDICT_CONST = 0,    /* KeepAll / SplitAll / MergeAll: value = 0/1/2 */
    CBTM_VERDICT_UNIFORM = 1,  /* UniformSplit: value = target depth           */
    CBTM_VERDICT_LOD = 2,      /* LodDecide: prm + root_tris                   */
    CBTM_VERDICT_EXPLICIT = 3  /* int8 verdicts[count] in cache_live order     */
};

typedef struct cbtm_verdict {
    int32_t mode;
    int32_t value;
    const int8_t *explicit_verdicts; /* device, mode EXPLICIT */
    const double *root_tris;         /* device f64[H*9] from cbtm_root_triangles */
    double prm[CBTM_PRM_WORDS];      /* HOST values, LodDecide._prm layout
                                        (lod.py:286-304), copied by value */
} cbtm_verdict;

/* ---- sizes ------------------------------------------------------------- */
int cbtm_abi_version(void);
/* number of u64 words of the bitfield (>= 16: one 128-byte line) */
size_t cbtm_bitfield_words(int depth);
/* number of u32 entries of the counter heap.  Index 0 is not a node: the library keeps a
 * stamp there ("the levels above the tile roots are mutually consistent", which lets a full
 * reduction update them by deltas instead of rebuilding them).  A caller that writes the
 * counter array by other means than these entry points must zero counters[0]. */
size_t cbtm_counter_words(int depth);
/* scratch bytes needed by cbtm_update / cbtm_sum_reduce for one pool */
size_t cbtm_workspace_bytes(int depth);
/* scratch bytes needed by the CBT-only calls (sum_reduce, index, decode) */
size_t cbtm_cbt_workspace_bytes(int depth);

/* ---- CBT: Cbt.sum_reduce / sum_reduce_array (cbt.py:61-68, 165-170) ------ */
int cbtm_sum_reduce(const uint64_t *bits, uint32_t *counters, int depth,
                    void *workspace, size_t workspace_bytes, uintptr_t stream);

/* ---- CBT: one_to_bit_id / zero_to_bit_id and their batch forms
 *      (cbt.py:75-107, 127-162).  ranks: device i64[K] or NULL for 0..K-1.
 *      out: device i32[K].  Ranks must be < count (ones) / < N - count (zeros);
 *      an out-of-range rank yields -1 in `out`. */
int cbtm_decode_ones(const uint64_t *bits, const uint32_t *counters, int depth,
                     const int64_t *ranks, int64_t K, int32_t *out, uintptr_t stream);
int cbtm_decode_zeros(const uint64_t *bits, const uint32_t *counters, int depth,
                      const int64_t *ranks, int64_t K, int32_t *out, uintptr_t stream);

/* ---- stage 2, k_cache_pointers (kernels.py:244-252) as a stream compaction:
 *      cache_live[i] = slot of the i-th set bit for i < n; if cache_free is not
 *      NULL, cache_free[i] = slot of the i-th unset bit for i < N - n.  Entries
 *      beyond are left untouched.  dispatch (may be NULL) receives the indirect
 *      dispatch arguments {ceil(n/256), 1, 1, n}. */
int cbtm_index(const uint64_t *bits, const uint32_t *counters, int depth,
               int32_t *cache_live, int32_t *cache_free, uint32_t *dispatch,
               uintptr_t stream);

/* ---- parity views of the reference heap layout (cbt.py:31, Cbt.nodes/leaves) */
/* leaves: device u32[N] of 0/1 -> packed bitfield (counters are NOT rebuilt) */
int cbtm_import_leaves(uint64_t *bits, int depth, const uint32_t *leaves, uintptr_t stream);
/* bitfield + counters -> device u32[2N] heap; every level is written, levels
 * below the counter heap are recomputed from the bitfield */
int cbtm_export_nodes(const uint64_t *bits, const uint32_t *counters, int depth,
                      uint32_t *nodes, uintptr_t stream);

/* ---- initialize (state.py:139-156): fills every pool array with the
 *      reference's initial values, seeds root bisectors at slots [0, H) and
 *      rebuilds the counters.  he_*: device i32[H]. */
int cbtm_initialize(const cbtm_pool *pool, const int32_t *he_next, const int32_t *he_prev,
                    const int32_t *he_twin, int32_t n_halfedges, uintptr_t stream);

/* ---- halfedge.from_polygons (halfedge.py:158-212) on the device, for input meshes too large for
 *      the python dictionaries of the reference (the paper's 21 399-halfedge asset and beyond).
 *      Input: polygon loops in CSR form, face_offsets i32[F+1] and face_verts i32[H] (device).
 *      Output (device i32[H] each): the six halfedge operators twin / next / prev / vert / edge /
 *      face exactly as the reference numbers them (halfedges in face order, edge = rank of the
 *      undirected vertex pair in sorted order, twin = -1 on a boundary).  status (device
 *      i64[CBTM_MESH_STATUS_WORDS]) = {degenerate faces (< 3 distinct vertices), corners with a
 *      vertex outside [0, V), zero-length edges, non-manifold edges (> 2 halfedges), edges whose
 *      two halfedges share a direction (inconsistent winding), lowest offending face or -1,
 *      lowest offending edge key (min << 32 | max) or -1, number of edges}: a mesh is valid iff
 *      the first five words are 0 -- the conditions under which the reference raises MeshError.
 *      workspace: cbtm_mesh_workspace_bytes(H) bytes of device scratch. */
#define CBTM_MESH_STATUS_WORDS 8
size_t cbtm_mesh_workspace_bytes(int64_t n_halfedges);
int cbtm_mesh_from_polygons(const int32_t *face_offsets, const int32_t *face_verts, int32_t n_faces,
                            int32_t n_halfedges, int32_t n_vertices, int32_t *he_twin,
                            int32_t *he_next, int32_t *he_prev, int32_t *he_vert, int32_t *he_edge,
                            int32_t *he_face, int64_t *status, void *workspace,
                            size_t workspace_bytes, uintptr_t stream);

/* ---- root bisector vertices per halfedge (bisector.py:154-173): v0, v1 and
 *      the face mean accumulated along `next`; out f64[H*9]. */
int cbtm_root_triangles(const int32_t *he_next, const int32_t *he_vert,
                        const double *positions, int32_t n_halfedges, double *out,
                        uintptr_t stream);

/* ---- verdict sources standalone (KernelDecide.fill, pipeline.py:87-119;
 *      _k_verdict_lod, lod.py:177-269): verdicts[i] for the current cache_live
 *      order, i < count (count read from the CBT root on device). */
int cbtm_classify(const cbtm_pool *pool, const cbtm_verdict *verdict, int8_t *verdicts,
                  uintptr_t stream);

/* ---- triangle export (state.decode_live / nb_decode_tris, bisector.py:186-189):
 *      out f64[K*9] for ids[K] (device). */
int cbtm_decode_triangles(const uint64_t *ids, int64_t K, int32_t rank,
                          const double *root_tris, double *out, uintptr_t stream);

/* ---- state.decode_live (state.py:104-113) without the host: re-indexes the pool (cache_live :=
 *      active list of the current state, ascending slot order) and decodes every live bisector
 *      into out f64[min(n, out_capacity)*9] in that order; n is read from the CBT root on the
 *      device.  draw_args (device u32[4], may be NULL) receives the indirect draw arguments
 *      {3 * triangles, 1, 0, 0} -- the step that follows the update in the paper's frame
 *      (PAPER.md:1126-1128).  Note: it overwrites cache_live[0, n) like stage 2 of the next
 *      update would. */
int cbtm_export_live_triangles(const cbtm_pool *pool, const double *root_tris, double *out,
                               int64_t out_capacity, uint32_t *draw_args, uintptr_t stream);

/* ---- pointer_violations (state.py:169-203) as a device-side check, so that a
 *      parity failure can be localised without downloading the pool.  out is
 *      device i64[CBTM_VALIDATE_WORDS] = {live slots, ids below the root range or
 *      mapping to an invalid halfedge, ids deeper than max_depth, dangling
 *      pointers (out of range or to a free slot), pointers without a reciprocal
 *      pointer (next answered by prev|twin, prev by next|twin, twin by any),
 *      neighbour depth gaps > 1, first offending slot or -1, 0}. */
#define CBTM_VALIDATE_WORDS 8
int cbtm_validate(const cbtm_pool *pool, int32_t n_halfedges, int64_t *out, uintptr_t stream);

/* ---- ParallelEngine.update (pipeline.py:204-322): one nine-stage frame.
 *      cbtm_update            = stages 1-9
 *      cbtm_update_begin      = stages 1-2 (counter reset + cache pointers); after
 *                               it the caller may read ids[cache_live[:n]] to
 *                               evaluate host verdicts (python-callable path)
 *      cbtm_update_finish     = stages 3-9
 *      Six UpdateStats counters + live counts land in pool->stats (device). */
int cbtm_update(const cbtm_pool *pool, const cbtm_verdict *verdict, uintptr_t stream);
int cbtm_update_begin(const cbtm_pool *pool, uintptr_t stream);
int cbtm_update_finish(const cbtm_pool *pool, const cbtm_verdict *verdict, uintptr_t stream);

/* ---- host side of the zero-copy stats path (the one call that blocks, and the only one that
 *      takes a HOST pointer to pool memory): spins until host_stats[CBTM_STAT_SEQ] >= frame, where
 *      host_stats is the host address of a pinned, device-mapped buffer that was passed as
 *      cbtm_pool.stats.  Replaces "copy the stats back + synchronise the stream" in
 *      ParallelEngine.update (pipeline.py:303-322 reads its counters on the host after every
 *      update).  Returns 0, or CBTM_E_TIMEOUT after timeout_ns. */
int cbtm_wait_frame(const int64_t *host_stats, int64_t frame, uint64_t timeout_ns);
/* same for host_stats[CBTM_STAT_DONE]: the frame has finished completely (reduction included) */
int cbtm_wait_frame_done(const int64_t *host_stats, int64_t frame, uint64_t timeout_ns);
/* cbtm_update + cbtm_wait_frame in one call (one FFI crossing per frame): launches the frame and
 * spins until its counters are in host_stats (= the host address of pool->stats, pinned and
 * device-mapped).  The frame number waited for is host_stats[CBTM_STAT_SEQ] + 1 as read before the
 * launch.  Returns 0, a contract / CUDA status of the launch, or CBTM_E_TIMEOUT. */
int cbtm_update_wait(const cbtm_pool *pool, const cbtm_verdict *verdict, const int64_t *host_stats,
                     uint64_t timeout_ns, uintptr_t stream);

/* ---- the frame loop of a real-time client (cmd_animate, cli.py:226-237: one update per camera,
 *      counters read back every frame) without a kernel launch per frame.  cbtm_update_linger =
 *      cbtm_update (LOD verdict source only) whose kernel, after publishing the frame, keeps
 *      polling `mailbox` (pinned host memory mapped into the device's address space, i64[64]) for
 *      up to linger_ns: if request number `request + 1` is posted in time (cbtm_post_request: the
 *      23 camera parameters, then the number), it runs that frame too, publishes, and listens
 *      again -- and so on.  A request that is not picked up in time is never served by that
 *      kernel, so the caller posts only while it knows the kernel still listens (ParallelEngine
 *      keeps a margin of half the linger time) and otherwise calls cbtm_update_linger again.
 *      `request` numbers start at 1 and grow by one per frame across launches.  cbtm_pool.stats
 *      should be host-mapped memory (cbtm_wait_frame).  Work queued on the same stream waits for
 *      the kernel to stop listening (at most linger_ns after its last frame). */
int cbtm_update_linger(const cbtm_pool *pool, const cbtm_verdict *verdict, const int64_t *mailbox,
                       int64_t request, int64_t linger_ns, uintptr_t stream);
/* host side: mailbox_host is the HOST address of the same buffer */
int cbtm_post_request(int64_t *mailbox_host, int64_t request, const double *prm);

/* ---- ParallelEngine.run_epochs / cmd_animate (pipeline.py:324-337,
 *      cli.py:226-231) for LOD sequences: n_frames updates back to back, no host
 *      synchronisation; prm_host is HOST f64[n_frames*23]; stats_out (device
 *      i64[n_frames*CBTM_STATS_WORDS], may be NULL) receives each frame's stats. */
int cbtm_run_lod_sequence(const cbtm_pool *pool, const double *root_tris,
                          const double *prm_host, int32_t n_frames, int64_t *stats_out,
                          uintptr_t stream);

/* ---- ParallelEngine.run_epochs (pipeline.py:324-337) with one verdict source for all epochs
 *      (KeepAll / SplitAll / MergeAll / UniformSplit, or one LodDecide): n_frames updates in one
 *      launch, no host synchronisation; stats_out as above. */
int cbtm_run_epochs(const cbtm_pool *pool, const cbtm_verdict *verdict, int32_t n_frames,
                    int64_t *stats_out, uintptr_t stream);

/* ---- the same for a BATCH of independent pools (cmd_animate over several planets, BASELINE
 *      config 5): the n_pools <= CBTM_MAX_BATCH pools advance in lockstep inside one cooperative
 *      launch, sharing every grid barrier -- P latency-bound planets cost little more than one.
 *      pools / root_tris / prm_host / stats_out are HOST arrays of n_pools entries: pool structs
 *      (by value), device f64[H*9] pointers, host f64[n_frames*23] pointers and device
 *      i64[n_frames*CBTM_STATS_WORDS] pointers (stats_out or any entry may be NULL).  Results are
 *      identical to n_pools separate cbtm_run_lod_sequence calls.  n_frames <= 4096 per call. */
int cbtm_run_lod_sequence_batch(const cbtm_pool *pools, int32_t n_pools, const double *const *root_tris,
                                const double *const *prm_host, int32_t n_frames,
                                int64_t *const *stats_out, uintptr_t stream);

#ifdef __cplusplus
}
#endif
#endif /* CBTM_H_ */
