// cbtm_frame.cuh -- the per-frame bisector update (stages 3-8 of
// ParallelEngine.update, pkg/src/cbtmesh/pipeline.py:204-322) as deterministic
// data-parallel kernels.
//
// The serial reference decides admission and slot placement through two
// order-dependent atomics (kernels.py:283-288, 315-319, 357-360).  Here both are
// restated as scans over the live ranks so that the result is bit-identical to
// the reference at threads=1 no matter how the GPU schedules the work:
//
//   admission  accept rank i iff running + need_i <= F, running over accepted
//              needs in rank order  ==  every rank before the first overflow
//              i0 is accepted; from i0 on a first-fit walk accepts any later
//              rank whose need still fits the remaining room (room < 187, so at
//              most 93 acceptances)
//   placement  rank i with n_alloc_i slots receives the free ranks
//              [T - incl_i, T - incl_i + n_alloc_i), incl = inclusive scan of
//              n_alloc, T = total admitted reservation
//
// A frame is latency bound: a few MB of traffic, but every pass is a chain of
// dependent steps (measured on B200, benchmarks/latency_probe.cu: L2 load
// 160 ns, returning atomic 255 ns, CTA barrier ~65 ns, a flag seen by another
// SM 430 ns, grid barrier 1.2 us).  What matters is the number of device-wide
// joins and of single-CTA passes between them:
//
//   P1 index    stages 1-3: active list by stream compaction, command reset
//   P2 classify stage 4: verdicts and reservation needs.  If even the worst
//               case n * (3 * max_depth + 4) fits the free count -- always true
//               for a pool sized like the paper's -- nothing can be rejected:
//               chunks scatter their commands right away and the total T is one
//               fire-and-forget atomic per warp.
//               Otherwise the scatter follows behind the barrier: everything, if the
//               total (known then) fits; under real reservation pressure one CTA
//               first scans the chunk needs, finds the first rejected rank and
//               runs the first-fit tail (P2b), then P2c scatters what was admitted.
//   P3 agree    stage 5a: merge agreement snapshot, allocation count per chunk;
//               meanwhile the CTA with the fewest chunks reads T (complete behind
//               the P2 barrier, nobody spins) and builds the free-rank window table
//   P4 reserve  stage 5b: every CTA sums the chunk counts before its chunk
//               (a redundant range sum instead of a single-CTA scan phase) and
//               hands out the free slots
//   P5 apply    stages 6-8 fused; touched leaf blocks marked in a byte map
//   P6 reduce   stage 9: marked leaf blocks recount their line, the levels up to
//               the tile roots are rebuilt, the few levels above receive each
//               tile's delta by atomics (no last-CTA pass, no fences)
//
// Inside a phase every load that does not depend on another is issued before the
// first result is consumed or stored (a store between two loads serialises them:
// the compiler must assume aliasing), which is where most of the last 5 us came from.
//
// They run either as ONE persistent cooperative kernel (k_frames: phases
// separated by grid barriers, any number of frames per launch) or as one kernel
// per phase (k_<phase> wrappers: the staged path, used for per-stage profiling
// and where cooperative launch is unavailable).
#pragma once

#include <cooperative_groups.h>

// -DCBTM_DEBUG_TIMING: every CTA records when its work of a phase ends (stats words 22..27 = latest end of work
// relative to the phase start, in ns), to tell work from barrier wait (benchmarks/phase_probe.py)
#ifdef CBTM_DEBUG_TIMING
#define WORK_END(ctl, k) do { if (threadIdx.x == 0) atomicMax(&(ctl)->work_end[k], global_ns()); } while (0)
// finer probes (benchmarks/probe_phases.py): latest arrival of any CTA at a point of the frame, per
// frame of a sequence run; slots 0..6 = phase starts as stamped by CTA 0
#define PROBE_FRAMES 128
#define PROBE_SLOTS 32
#define PROBE(slot)                                                                                      \
    do {                                                                                                 \
        __syncthreads();                                                                                 \
        if (threadIdx.x == 0) atomicMax(&cbtm::g_probe[cbtm::probe_frame() & (PROBE_FRAMES - 1)][slot], cbtm::probe_now()); \
    } while (0)
// per warp, no CTA barrier (usable in divergent code); `dep` makes the stamp wait for a loaded value
#define PROBE_W(slot, dep)                                                                               \
    do {                                                                                                 \
        asm volatile("" ::"r"(dep) : "memory");                                                          \
        const unsigned am_ = __activemask();                                                             \
        if ((am_ & (0u - am_)) == (1u << (threadIdx.x & 31))) /* lowest lane that got here */            \
            atomicMax(&cbtm::g_probe[cbtm::probe_frame() & (PROBE_FRAMES - 1)][slot], cbtm::probe_now()); \
    } while (0)
#define PROBE_SET_FRAME(f) do { if (threadIdx.x == 0) cbtm::probe_frame() = (f); __syncthreads(); } while (0)
#define PROBE_T0(slot, f)                                                                                \
    do {                                                                                                 \
        if (blockIdx.x == 0 && threadIdx.x == 0) cbtm::g_probe[(f) & (PROBE_FRAMES - 1)][slot] = cbtm::probe_now(); \
    } while (0)
namespace cbtm {
__device__ unsigned long long g_probe[PROBE_FRAMES][PROBE_SLOTS];
__device__ __forceinline__ int &probe_frame() { __shared__ int f; return f; }
__device__ __forceinline__ unsigned long long probe_now()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
} // namespace cbtm
#else
#define WORK_END(ctl, k) do { } while (0)
#define PROBE(slot) do { } while (0)
#define PROBE_W(slot, dep) do { } while (0)
#define PROBE_SET_FRAME(f) do { } while (0)
#define PROBE_T0(slot, f) do { } while (0)
#endif

#include "cbtm_cbt.cuh"
#include "cbtm_classify.cuh"

namespace cbtm {

constexpr int TAIL_MAX = 96;
constexpr int MAX_SEQ_FRAMES = 4096;
constexpr int WIN_MAX = 4096;       // leaf blocks covered by the free-rank window table
constexpr int WIN_SMEM = 1024;      // ... of which the reserve phase keeps up to this many in shared memory

// device-resident control block of one pool (lives in the workspace)
struct Control {
    int64_t n, F, T, A; // live, free, reserved total, allocated total
    int64_t i0;         // first rank rejected by admission (n if none)
    int32_t tail_count;
    uint32_t seq_frame; // index into prm_seq for sequence runs
    unsigned long long need_total; // sum of the frame's reservation needs (zero between frames)
    int32_t mb_go;                 // linger mode: 1 = a request arrived in time, run another frame
    int32_t mb_pad_;
    double mb_prm[CBTM_PRM_WORDS]; // linger mode: the camera parameters of that request
    int32_t tail_idx[TAIL_MAX];
    uint32_t win_lo; // first leaf block of the free-rank window table
    uint32_t win_n;  // leaf blocks in the window table (0: table not built, descend)
    unsigned long long phase_t[2][CBTM_STAT_PHASES + 1]; // %globaltimer at the start of each phase, by frame parity
    int64_t stats[CBTM_STATS_WORDS];
#ifdef CBTM_DEBUG_TIMING
    unsigned long long work_end[CBTM_STAT_PHASES + 3]; // latest end of a CTA's work in each phase (before the barrier); 3 spare probes
#endif
};


struct Workspace {
    uint8_t *need8;   // [N] by live rank: slots to reserve (0 = no command)
    uint8_t *mbits8;  // [N] by live rank: merge command bits of a merge request
    uint8_t *nalloc8; // [N] by live rank: slots actually allocated
    int32_t *j4s;     // [N] by live rank: fourth member of a valid quad merge configuration
    int32_t *merge_ref; // [N] by slot: -1, or for a member of an agreed merge 2 * owner slot + (1 if the
                        // member sits in the pair opposite to the owner's, i.e. its parent is reserved[owner][1])
    uint32_t *chunk_need;     // [N/256] reservation need of each chunk of 256 live ranks
    uint64_t *chunk_need_off; // [N/256] exclusive scan of chunk_need (pressure path only)
    uint8_t *chunk_minneed;   // [N/256] smallest non-zero need of the chunk (255: none)
    uint32_t *chunk_alloc;    // [N/256] slots allocated by each chunk
    uint32_t *win_prefix; // [WIN_MAX + 1] free ranks before each leaf block of the window
    uint8_t *dirty;       // [N/1024] leaf blocks whose bits changed since the last reduction
    Control *ctl;
    double *prm_seq;  // [MAX_SEQ_FRAMES * 23]
    unsigned *ticket; // first word of the workspace: k_sum_reduce's CTA ticket
};

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Carves the caller's scratch buffer.  Returns the bytes used.
inline size_t carve_workspace(void *base, int depth, Workspace *ws)
{
    const size_t N = (size_t)1 << depth;
    const size_t nch = (N + CHUNK - 1) / CHUNK;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        void *p = base ? (char *)base + off : nullptr;
        off = align_up(off + bytes, 256);
        return p;
    };
    Workspace w;
    w.ticket = (unsigned *)take(256); // must stay first: cbtm_sum_reduce uses word 0
    w.ctl = (Control *)take(sizeof(Control));
    w.prm_seq = (double *)take(sizeof(double) * CBTM_PRM_WORDS * MAX_SEQ_FRAMES);
    w.need8 = (uint8_t *)take(N);
    w.mbits8 = (uint8_t *)take(N);
    w.nalloc8 = (uint8_t *)take(N);
    w.j4s = (int32_t *)take(4 * N);
    w.merge_ref = (int32_t *)take(4 * N);
    w.chunk_need = (uint32_t *)take(4 * nch);
    w.chunk_need_off = (uint64_t *)take(8 * nch);
    w.chunk_minneed = (uint8_t *)take(nch);
    w.chunk_alloc = (uint32_t *)take(4 * nch);
    w.win_prefix = (uint32_t *)take(4 * (WIN_MAX + 1));
    w.dirty = (uint8_t *)take(N >> LEAF_LOG2 ? N >> LEAF_LOG2 : 1);
    if (ws) *ws = w;
    return off;
}

struct FrameArgs {
    cbtm_pool pool;
    Workspace ws;
    int32_t vmode, vvalue;
    const int8_t *vexplicit;
    const double *root_tris;
    int32_t use_prm_seq;
    int32_t pad_;
    double prm[CBTM_PRM_WORDS];
};

// No admission can fail when even the worst case fits: every live bisector asking
// for the deepest split's reservation (kernels.py:279-288).  CTA- and grid-uniform.
__device__ __forceinline__ bool fits_a_priori(const cbtm_pool &p, uint32_t n)
{
    const uint64_t F = ((uint64_t)1 << p.depth) - n;
    return (uint64_t)n * (uint64_t)(3 * p.max_depth + 4) <= F;
}

// ---------------------------------------------------------------------------
// merge configuration (kernels.py:112-191)
// ---------------------------------------------------------------------------
struct MergeCfg {
    int kind; // 0 none, 1 boundary pair, 2 quad
    int32_t sib, oth, j4;
    uint64_t id_sib, id_oth, id_j4; // ids of the members (valid per kind)
};

// kernels.py:113-134 on values gathered ahead of time (phase_classify issues these
// loads before the classifier runs so that their latency hides behind it):
// js = ids[sib], jo = ids[oth], j4 = next-or-prev[oth]; only ids[j4] is still
// to be fetched, and only for a quad.
__device__ __forceinline__ MergeCfg merge_config_gathered(const cbtm_pool &p, uint64_t j1, int32_t sib, int32_t oth,
                                                          uint64_t js, uint64_t jo, int32_t j4,
                                                          const uint64_t *id_j4 = nullptr /* ids[j4], if fetched already */)
{
    MergeCfg c = {0, -1, -1, -1, 0, 0, 0};
    if (depth_of(j1, p.rank) < 1) return c; // roots never merge
    if (sib < 0) return c;
    if ((js >> 1) != (j1 >> 1)) return c;
    c.sib = sib;
    c.id_sib = js;
    if (oth < 0) {
        c.kind = 1;
        return c;
    }
    if (bit_length64(jo) != bit_length64(j1)) return c;
    if (j4 < 0) return c;
    const uint64_t j4id = id_j4 ? *id_j4 : p.ids[j4];
    if ((j4id >> 1) != (jo >> 1)) return c;
    c.kind = 2;
    c.oth = oth;
    c.j4 = j4;
    c.id_oth = jo;
    c.id_j4 = j4id;
    return c;
}

// Same configuration for a bisector whose merge request was admitted this
// frame: k_classify validated it and left the fourth member in j4s (so no
// pointer chasing here); kind comes from the command word.
__device__ __forceinline__ MergeCfg merge_config_admitted(uint64_t j1, int32_t nx, int32_t pv, uint32_t cmd,
                                                          int32_t j4)
{
    const bool odd = j1 & 1;
    MergeCfg c = {1, odd ? pv : nx, -1, -1, 0, 0, 0};
    if (cmd & CBTM_CMD_QUAD) {
        c.kind = 2;
        c.oth = odd ? nx : pv;
        c.j4 = j4;
    }
    return c;
}

__device__ __forceinline__ bool wants_only_merge(uint32_t cmd)
{
    return !(cmd & CBTM_CMD_SPLIT_MASK) && (cmd & CBTM_CMD_MERGE);
}

// ---------------------------------------------------------------------------
// start of a frame without an index phase (cbtm_update_finish: the caller ran
// stages 1-2 and evaluated its verdicts on the host): stage 3 on its own.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void phase_reset(const FrameArgs &a, uint32_t bid, uint32_t nb)
{
    const cbtm_pool &p = a.pool;
    const uint32_t n = p.counters[1];
    for (uint64_t i = bid * (uint64_t)CHUNK + threadIdx.x; i < n; i += (uint64_t)nb * CHUNK)
        p.commands[p.cache_live[i]] = 0; // kernels.py:256-259
}

// ---------------------------------------------------------------------------
// verdict sources (pipeline.py:87-119, lod.py:177-269)
// ---------------------------------------------------------------------------
__device__ __forceinline__ int verdict_of(const FrameArgs &a, const double *prm, uint64_t id, uint32_t i)
{
    const cbtm_pool &p = a.pool;
    switch (a.vmode) {
    case CBTM_VERDICT_CONST: return a.vvalue;
    case CBTM_VERDICT_UNIFORM: return depth_of(id, p.rank) < a.vvalue ? 1 : 0;
    case CBTM_VERDICT_LOD: return lod_verdict(id, p.rank, p.max_depth, a.root_tris, prm);
    default: return a.vexplicit[i];
    }
}

__device__ __forceinline__ void load_prm(const FrameArgs &a, double *prm)
{
    if (a.vmode == CBTM_VERDICT_LOD) {
        if (threadIdx.x < CBTM_PRM_WORDS)
            prm[threadIdx.x] = a.use_prm_seq
                                   ? a.ws.prm_seq[(size_t)CBTM_PRM_WORDS * a.ws.ctl->seq_frame + threadIdx.x]
                                   : a.prm[threadIdx.x];
        __syncthreads();
    }
}

// standalone (KernelDecide.fill): no side effects on the pool
__global__ void __launch_bounds__(CHUNK)
k_classify(const __grid_constant__ FrameArgs a, int8_t *verdict_out)
{
    __shared__ double prm[CBTM_PRM_WORDS];
    const cbtm_pool &p = a.pool;
    const uint32_t n = p.counters[1];
    load_prm(a, prm);
    for (uint64_t i = blockIdx.x * (uint64_t)CHUNK + threadIdx.x; i < n; i += (uint64_t)gridDim.x * CHUNK)
        verdict_out[i] = (int8_t)verdict_of(a, prm, p.ids[p.cache_live[i]], (uint32_t)i);
}

// Leaf block holding the free (unset) rank `rank` and the number of free slots before that block.
// A whole CTA descends the counter heap eight levels per step (the 256 descendants of a
// node eight levels down are contiguous): two round trips for D = 26.
// scratch: 32 words, out: 2 words of shared memory.
// first_step: the counter this thread needs for the first step (node (1 << s0) + tid, s0 = min(lc, 8)),
// fetched by the caller ahead of time -- it does not depend on the rank (nullptr: fetched here).
__device__ __forceinline__ void cta_find_free_block(const uint32_t *counters, const Geo &g, uint32_t rank,
                                                    uint32_t *scratch, uint32_t *out, uint32_t &block,
                                                    uint32_t &free_before, const uint32_t *first_step = nullptr)
{
    const int tid = threadIdx.x;
    uint32_t idx = 0, before = 0;
    int l = 0;
    while (l < g.lc) {
        const int s = g.lc - l < 8 ? g.lc - l : 8;
        const uint32_t fan = 1u << s;
        const uint32_t child_span = (uint32_t)(g.n >> (l + s));
        const uint32_t ones = (uint32_t)tid < fan ? ((l == 0 && first_step) ? *first_step
                                                                            : counters[(1u << (l + s)) + (idx << s) + tid])
                                                  : 0u;
        const uint32_t z = (uint32_t)tid < fan ? child_span - ones : 0u;
        uint32_t total;
        const uint32_t incl = block_inclusive_scan<CHUNK>(z, scratch, &total);
        if ((uint32_t)tid == fan - 1) { // default: the last child (rank beyond the free count)
            out[0] = fan - 1;
            out[1] = incl - z;
        }
        __syncthreads();
        if ((uint32_t)tid < fan && incl > rank && incl - z <= rank) {
            out[0] = (uint32_t)tid;
            out[1] = incl - z;
        }
        __syncthreads();
        const uint32_t child = out[0], excl = out[1];
        __syncthreads();
        rank -= excl;
        before += excl;
        idx = (idx << s) + child;
        l += s;
    }
    block = idx;
    free_before = before;
}

// The table that lets the reserve phase resolve free ranks without a tree
// descent: all allocations of a frame draw from ONE interval of free ranks
// [T - A, T) which lives in a short run of leaf blocks ending at the block of
// free rank T - 1.  A is not known yet when T is, so the table is anchored at
// the top: it covers the last WIN_MAX leaf blocks up to that one;
// win_prefix[j] = free slots before leaf block win_lo + j.  (One CTA.)
__device__ __forceinline__ void build_window_table(const FrameArgs &a, long long T, const uint32_t *first_step = nullptr)
{
    __shared__ uint32_t scratch[32];
    __shared__ uint32_t s_out[2];
    Control *ctl = a.ws.ctl;
    const cbtm_pool &p = a.pool;
    const Geo g = make_geo(p.depth);
    const int tid = threadIdx.x;
    if (tid == 0) ctl->win_n = 0;
    if (T <= 0 || (p.flags & (CBTM_POOL_FULL_FREE_CACHE | CBTM_POOL_DESCEND_FREE_RANKS))) return;
    uint32_t hi, before_hi;
    cta_find_free_block(p.counters, g, (uint32_t)(T - 1), scratch, s_out, hi, before_hi, first_step);
    const uint32_t ones_hi = p.counters[g.nblocks + hi]; // (issued with the loads below, not behind their scan)
    const uint32_t lo = hi + 1 > (uint32_t)WIN_MAX ? hi + 1 - WIN_MAX : 0u;
    const uint32_t nbw = hi - lo + 1;
    constexpr int PER = WIN_MAX / CHUNK;
    const uint32_t per = (nbw + CHUNK - 1) / CHUNK; // <= PER
    const uint32_t j0 = tid * per;
    uint32_t z[PER], sum = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const uint32_t j = j0 + k;
        z[k] = ((uint32_t)k < per && j < nbw) ? g.span - p.counters[g.nblocks + lo + j] : 0u;
        sum += z[k];
    }
    uint32_t total;
    const uint32_t incl = block_inclusive_scan<CHUNK>(sum, scratch, &total);
    // free slots before block lo = (free before block hi) - (free in [lo, hi))
    const uint32_t z_hi = g.span - ones_hi;
    const uint32_t base = before_hi - (total - z_hi);
    uint32_t run = base + incl - sum;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const uint32_t j = j0 + k;
        if ((uint32_t)k < per && j < nbw) a.ws.win_prefix[j] = run;
        run += z[k];
    }
    if (tid == 0) {
        a.ws.win_prefix[nbw] = base + total;
        ctl->win_lo = lo;
        ctl->win_n = nbw;
    }
}

// ---------------------------------------------------------------------------
// What a thread learns about ITS rank of the CTA's first chunk (chunk == bid: the only chunk of a CTA
// up to 75 k live bisectors) in one phase and needs again in a later one, kept in shared memory across
// the grid barriers of the persistent kernel instead of being fetched again: the slot and the record
// (P2), the final command word, the twin, the allocation count and the agreement reference (P3), the
// reserved slots (P4).  Every value is private to the thread's rank or unchanged until the apply phase
// writes (own records of consumed bisectors are never rewritten), so the copies cannot go stale.  It
// removes the rank -> slot round trip from the head of P3 and both the rank-indexed and the own-record
// round trips from the head of P5.  Lives in the index phase's staging area (dead between P1 and P6).
// ---------------------------------------------------------------------------
struct Carry {
    int32_t s[CHUNK];
    uint32_t id_lo[CHUNK], id_hi[CHUNK];
    int32_t nx[CHUNK], pv[CHUNK], tw[CHUNK], j4[CHUNK];
    uint32_t cmd[CHUNK];
    int32_t mref[CHUNK];
    uint32_t na[CHUNK];
    int32_t res[4][CHUNK];
};

// ---------------------------------------------------------------------------
// P2 = stage 4: evaluate verdicts and compute each rank's reservation need
// (3d+4 for a split, 2 for a valid merge, 0 otherwise).  Splits walk their
// compatibility chain OR-ing edge-split bits (kernels.py:289-310); merges OR
// their configuration bits (kernels.py:320-333).  OR is commutative, so the
// final command words do not depend on scheduling.
// ---------------------------------------------------------------------------
// t0: twins[s] if the caller has it already (kNoTwinYet: fetched here)
constexpr int32_t kNoTwinYet = INT32_MIN;
__device__ __forceinline__ void walk_split_chain(const cbtm_pool &p, int32_t s, int32_t t0 = kNoTwinYet)
{
    // Pointer fields do not change during this phase, so the twin's operators
    // are fetched while the atomic on `cur` is still in flight, and the twin's
    // twin doubles as the next hop's twin: one dependent round trip per hop.
    // The old value of the atomic must be honoured BEFORE the next node is
    // touched: "T already set" means "whoever set it walks the rest of the
    // chain", which only holds if nobody marks a node and then stops (a variant
    // that looked at the old value one hop late lost parts of chains).
    int32_t cur = s;
    int32_t t = t0 != kNoTwinYet ? t0 : p.twins[cur];
    for (int hops = 0;;) {
        int32_t t_twin = -1, t_next = -1, t_prev = -1;
        if (t >= 0) {
            t_twin = p.twins[t];
            t_next = p.nexts[t];
            t_prev = p.prevs[t];
        }
        const uint32_t before = atomicOr(&p.commands[cur], CBTM_CMD_SPLIT_T);
        if (before & CBTM_CMD_SPLIT_T) break; // another walker owns the rest of the chain
        if (t < 0) break;
        if (t_twin == cur) {
            atomicOr(&p.commands[t], CBTM_CMD_SPLIT_T);
            break;
        }
        if (t_next == cur)
            atomicOr(&p.commands[t], CBTM_CMD_SPLIT_N);
        else if (t_prev == cur)
            atomicOr(&p.commands[t], CBTM_CMD_SPLIT_P);
        else
            break;
        cur = t;
        t = t_twin;
        if (++hops > 70) break;
    }
}

__device__ __forceinline__ void phase_classify(const FrameArgs &a, uint32_t n, uint32_t bid, uint32_t nb,
                                               const double *prm_row = nullptr, Carry *carry = nullptr)
{
    __shared__ double prm[CBTM_PRM_WORDS];
    __shared__ uint32_t wsum[CHUNK / 32], wmin[CHUNK / 32];
    const cbtm_pool &p = a.pool;
    Control *ctl = a.ws.ctl;
    const uint32_t nch = (n + CHUNK - 1) / CHUNK;
    const bool fast = fits_a_priori(p, n); // nothing can be rejected: scatter right away
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // frame totals (need, deepest bisector): accumulated per warp in registers over all its chunks, then
    // per CTA in shared memory -- ONE global atomic per CTA and phase (one per warp and chunk put up to
    // 60 000 atomics per frame on a single address: same-address atomics serialise in L2)
    __shared__ unsigned long long s_need;
    __shared__ int s_depth;
    unsigned long long acc_need = 0;
    int acc_depth = 0;
    if (tid == 0) {
        s_need = 0;
        s_depth = 0;
    }

    // the camera parameters of a sequence run sit behind two dependent loads (frame index, then
    // the row): issued now, parked in a register, put into shared memory only when the first
    // verdict needs them -- the record gathers below run meanwhile
    double prm_reg = 0.0;
    bool prm_pending = a.vmode == CBTM_VERDICT_LOD;
    if (prm_pending && tid < CBTM_PRM_WORDS)
        prm_reg = prm_row ? prm_row[tid]
                          : a.use_prm_seq ? a.ws.prm_seq[(size_t)CBTM_PRM_WORDS * ctl->seq_frame + tid] : a.prm[tid];

    for (uint32_t chunk = bid; chunk < nch; chunk += nb) {
        const uint32_t i = chunk * CHUNK + tid;
        uint32_t need = 0, mbits = 0;
        int32_t s = -1;
        struct {
            uint64_t id, js, jo;
            int32_t sib, oth, j4, nx, pv, tw;
        } gathered = {0, 0, 0, -1, -1, -1, -1, -1, -1};
        if (i < n) {
            s = p.cache_live[i];
            const uint64_t id = p.ids[s];
            const int32_t nx = p.nexts[s], pv = p.prevs[s];
            // the twin rides along: a split's chain walk starts from it (one round trip less per walk)
            // and the apply phase wants it (carried)
            // (only for the CTA's first chunk: with many chunks per CTA -- 10^6 live bisectors -- a fourth
            // scattered load for everybody costs more than the walks of the few that split gain)
            const int32_t tw = (carry && chunk == bid) ? p.twins[s] : kNoTwinYet;
            // what a merge request will ask about its sibling and the opposite pair: with the LOD
            // classifier gathered now, for everybody, so that the round trip hides behind the fp64 work;
            // the other verdict sources are known at once, so only merge requests gather (three scattered
            // sectors per bisector saved: at 10^6 live bisectors this phase is bound by L2 transactions)
            const bool odd = id & 1;
            const int32_t sib = odd ? pv : nx, oth = odd ? nx : pv;
            uint64_t js = 0, jo = 0;
            int32_t j4 = -1;
            const bool gather = a.vmode == CBTM_VERDICT_LOD || verdict_of(a, prm, id, i) == 2;
            if (gather && sib >= 0) js = p.ids[sib];
            if (gather && oth >= 0) {
                jo = p.ids[oth];
                j4 = odd ? p.nexts[oth] : p.prevs[oth];
            }
            gathered = {id, js, jo, sib, oth, j4, nx, pv, tw};
        }
        PROBE(8); // classify: gathers issued (loads may still be in flight)
        { // deepest live bisector of the frame
            const int d = i < n ? depth_of(gathered.id, p.rank) : 0;
            acc_depth = max(acc_depth, __reduce_max_sync(FULL_MASK, d));
        }
        if (prm_pending) { // CTA-uniform
            if (tid < CBTM_PRM_WORDS) prm[tid] = prm_reg;
            __syncthreads();
            prm_pending = false;
        }
        if (i < n) {
            const uint64_t id = gathered.id, js = gathered.js, jo = gathered.jo;
            const int32_t sib = gathered.sib, oth = gathered.oth, j4 = gathered.j4;
            // LOD: the id of a quad's fourth member -- the one gather that hangs on the gathers above -- is
            // fetched between the decode and the projection, so that it too hides behind fp64 work
            // instead of following the verdict
            int v;
            uint64_t id_j4 = 0;
            const bool j4_early = a.vmode == CBTM_VERDICT_LOD;
            if (j4_early) {
                double tri[9];
                decode_triangle(id, p.rank, a.root_tris, tri);
                if (j4 >= 0) id_j4 = p.ids[j4];
                v = lod_verdict_of_triangle(tri, id, p.rank, p.max_depth, prm);
            } else {
                v = verdict_of(a, prm, id, i);
            }
            if (v == 1) {
                const int d = depth_of(id, p.rank);
                if (d < p.max_depth) need = 3 * d + 4;
            } else if (v == 2) {
                const MergeCfg c = merge_config_gathered(p, id, sib, oth, js, jo, j4, j4_early ? &id_j4 : nullptr);
                if (c.kind) {
                    need = 2;
                    mbits = CBTM_CMD_MERGE;
                    uint64_t lowest = umin64(id, c.id_sib);
                    if (c.kind == 2) {
                        mbits |= CBTM_CMD_QUAD;
                        lowest = umin64(lowest, c.id_oth);
                        lowest = umin64(lowest, c.id_j4);
                        a.ws.j4s[i] = c.j4;
                    }
                    if (lowest == id) mbits |= CBTM_CMD_OWNER;
                }
            }
            a.ws.need8[i] = (uint8_t)need;
            a.ws.mbits8[i] = (uint8_t)mbits;
            if (carry && chunk == bid) { // (here, not at the loads: a store in between would serialise them)
                carry->s[tid] = s;
                carry->id_lo[tid] = (uint32_t)id;
                carry->id_hi[tid] = (uint32_t)(id >> 32);
                carry->nx[tid] = gathered.nx;
                carry->pv[tid] = gathered.pv;
                carry->tw[tid] = gathered.tw;
                carry->j4[tid] = (mbits & CBTM_CMD_QUAD) ? j4 : -1;
            }
        }
        PROBE(9); // classify: verdicts and needs known
#ifdef CBTM_DEBUG_TIMING
        WORK_END(ctl, 0);
#endif
        uint32_t sum = warp_sum(need);
        acc_need += sum; // the frame's total need
        if (fast) {
            if (need == 2)
                atomicOr(&p.commands[s], mbits);
            else if (need)
                walk_split_chain(p, s, gathered.tw);
            PROBE(10); // classify: commands scattered
            continue;
        }
        uint32_t mn = need ? need : 255u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(FULL_MASK, mn, o));
        if (lane == 0) {
            wsum[warp] = sum;
            wmin[warp] = mn;
        }
        __syncthreads();
        if (tid == 0) {
            uint32_t ts = 0, tm = 255u;
#pragma unroll
            for (int w = 0; w < CHUNK / 32; ++w) {
                ts += wsum[w];
                tm = min(tm, wmin[w]);
            }
            a.ws.chunk_need[chunk] = ts;
            a.ws.chunk_minneed[chunk] = (uint8_t)tm;
        }
        __syncthreads();
    }

    __syncthreads();
    if (lane == 0) {
        if (acc_need) atomicAdd(&s_need, acc_need);
        if (acc_depth) atomicMax(&s_depth, acc_depth);
    }
    __syncthreads();
    if (tid == 0) {
        if (s_need) atomicAdd(&ctl->need_total, s_need);
        if (s_depth) atomicMax((long long *)&ctl->stats[CBTM_STAT_PEAK_DEPTH], (long long)s_depth);
    }
}

// The frame's total need (complete behind the barrier that ends P2) and whether all of it fits.
// Grid-uniform; need_total is zeroed by frame_totals, behind another barrier.
__device__ __forceinline__ bool frame_fits(const FrameArgs &a, uint32_t n)
{
    const unsigned long long total = a.ws.ctl->need_total;
    return total <= (((unsigned long long)1 << a.pool.depth) - n);
}

// One CTA, once per frame, after the scatter: if the frame fits, T = total need and the other
// per-frame fields phase_admit would have set; in any case need_total returns to zero.
// Returns T (thread 0 only).
__device__ __forceinline__ long long frame_totals(const FrameArgs &a, uint32_t n, bool fits)
{
    const cbtm_pool &p = a.pool;
    Control *ctl = a.ws.ctl;
    long long T = 0;
    if (threadIdx.x == 0) {
        const unsigned long long total = ctl->need_total;
        ctl->need_total = 0;
        T = fits ? (long long)total : ctl->T; // (pressure path: phase_admit set it)
        if (fits) {
            ctl->n = n;
            ctl->F = (int64_t)(((uint64_t)1 << p.depth) - n);
            ctl->T = (int64_t)total;
            ctl->i0 = n;
            ctl->tail_count = 0;
            ctl->stats[CBTM_STAT_LIVE_BEFORE] = n;
            ctl->stats[CBTM_STAT_RESERVED] = (int64_t)total;
        }
    }
    __syncthreads(); // ctl->T is read right away by the same CTA (window table)
    return T;
}

// frame_totals + build_window_table by one CTA with the round trips that do not depend on each other
// taken together: the counters of the descent's first step are fetched while thread 0 reads the frame's
// total, and T reaches the other threads through shared memory instead of through the control block.
__device__ __forceinline__ void frame_totals_and_window(const FrameArgs &a, uint32_t n, bool fits)
{
    __shared__ long long s_T;
    const cbtm_pool &p = a.pool;
    const Geo g = make_geo(p.depth);
    const int s0 = g.lc < 8 ? g.lc : 8;
    uint32_t first_step = 0;
    if (g.lc > 0 && threadIdx.x < (1u << s0)) first_step = p.counters[(1u << s0) + threadIdx.x];
    const long long T = frame_totals(a, n, fits);
    if (threadIdx.x == 0) s_T = T;
    __syncthreads();
    build_window_table(a, s_T, g.lc > 0 ? &first_step : nullptr);
}

// ---------------------------------------------------------------------------
// P2b (one CTA; only when the pool is too full for the a-priori bound):
// admission.  Scans the per-chunk needs, locates the first overflowing rank i0,
// runs the first-fit tail walk, then builds the window table.
// ---------------------------------------------------------------------------
template <int NT>
__device__ __forceinline__ void phase_admit(const FrameArgs &a)
{
    __shared__ uint32_t scratch[32];
    __shared__ uint32_t s_warpmin[32];
    __shared__ unsigned long long s_carry;
    __shared__ uint32_t s_c0, s_found, s_next, s_room;
    __shared__ long long s_pos;
    __shared__ int s_cnt;

    const cbtm_pool &p = a.pool;
    Control *ctl = a.ws.ctl;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t n = p.counters[1];
    const uint64_t F = ((uint64_t)1 << p.depth) - n;
    const uint32_t nch = (n + CHUNK - 1) / CHUNK;

    if (tid == 0) {
        s_carry = 0;
        s_c0 = nch;
    }
    __syncthreads();

    // ---- exclusive scan of the chunk needs, first overflowing chunk ----
    for (uint32_t base = 0; base < nch; base += NT) {
        const uint32_t c = base + tid;
        const uint32_t v = c < nch ? a.ws.chunk_need[c] : 0;
        uint32_t total;
        const uint32_t incl = block_inclusive_scan<NT>(v, scratch, &total);
        const unsigned long long carry = s_carry;
        if (c < nch) {
            const unsigned long long off = carry + incl - v;
            a.ws.chunk_need_off[c] = off;
            if (off + v > F) atomicMin(&s_c0, c);
        }
        __syncthreads();
        if (tid == 0) s_carry = carry + total;
        __syncthreads();
    }
    const unsigned long long total_need = s_carry;
    const uint32_t c0 = s_c0;

    if (c0 == nch) { // everything fits
        if (tid == 0) {
            ctl->n = n;
            ctl->F = (int64_t)F;
            ctl->T = (int64_t)total_need;
            ctl->i0 = n;
            ctl->tail_count = 0;
            ctl->stats[CBTM_STAT_LIVE_BEFORE] = n;
            ctl->stats[CBTM_STAT_RESERVED] = (int64_t)total_need;
        }
        return;
    }

    // ---- first overflowing rank inside chunk c0 ----
    {
        const uint32_t i = c0 * CHUNK + tid;
        const uint32_t v = (tid < CHUNK && i < n) ? a.ws.need8[i] : 0;
        uint32_t total;
        const uint32_t incl = block_inclusive_scan<NT>(v, scratch, &total);
        const unsigned long long off = a.ws.chunk_need_off[c0];
        if (tid == 0) s_found = 0xffffffffu;
        __syncthreads();
        if (tid < CHUNK && v && off + incl > F) atomicMin(&s_found, (uint32_t)tid);
        __syncthreads();
        const uint32_t f = s_found; // exists by construction
        if ((uint32_t)tid == f) {
            s_room = (uint32_t)(F - (off + incl - v));
            s_pos = (long long)c0 * CHUNK + f;
            ctl->i0 = (long long)c0 * CHUNK + f;
            s_cnt = 0;
        }
        __syncthreads();
    }

    // ---- first-fit tail walk from i0 ----
    while (true) {
        const long long pos = s_pos;
        if (s_room < 2 || pos >= (long long)n) break;
        const uint32_t c = (uint32_t)(pos / CHUNK);
        const long long idx = (long long)c * CHUNK + tid;
        uint32_t need = (tid < CHUNK && idx >= pos && idx < (long long)n) ? a.ws.need8[idx] : 0;
        while (true) { // accept, in rank order, whatever still fits in this chunk
            const uint32_t room = s_room;
            const bool ok = need > 0 && need <= room;
            const unsigned b = __ballot_sync(FULL_MASK, ok);
            if (lane == 0) s_warpmin[warp] = b ? (uint32_t)(warp * 32 + __ffs(b) - 1) : 0xffffffffu;
            __syncthreads();
            if (tid == 0) {
                uint32_t m = 0xffffffffu;
                for (int w = 0; w < CHUNK / 32; ++w) m = min(m, s_warpmin[w]);
                s_found = m;
            }
            __syncthreads();
            const uint32_t f = s_found;
            if (f == 0xffffffffu) break;
            if ((uint32_t)tid == f) {
                ctl->tail_idx[s_cnt] = (int32_t)idx;
                s_cnt = s_cnt + 1;
                s_room = room - need;
            }
            if ((uint32_t)tid <= f) need = 0;
            __syncthreads();
        }
        // next chunk holding a need that still fits
        const uint32_t room = s_room;
        if (room < 2) break;
        if (tid == 0) s_next = nch;
        __syncthreads();
        for (uint32_t base = c + 1; base < nch; base += NT) {
            const uint32_t cc = base + tid;
            const bool ok = cc < nch && a.ws.chunk_minneed[cc] <= room;
            const unsigned b = __ballot_sync(FULL_MASK, ok);
            if (lane == 0) s_warpmin[warp] = b ? (uint32_t)(base + warp * 32 + __ffs(b) - 1) : 0xffffffffu;
            __syncthreads();
            if (tid == 0) {
                uint32_t m = 0xffffffffu;
                for (int w = 0; w < NT / 32; ++w) m = min(m, s_warpmin[w]);
                if (m != 0xffffffffu) s_next = m;
            }
            __syncthreads();
            if (s_next != nch) break;
        }
        const uint32_t nxt = s_next;
        __syncthreads();
        if (nxt >= nch) break;
        if (tid == 0) s_pos = (long long)nxt * CHUNK;
        __syncthreads();
    }
    __syncthreads();
    const long long T = (long long)F - (long long)s_room;
    if (tid == 0) {
        ctl->n = n;
        ctl->F = (int64_t)F;
        ctl->T = T;
        ctl->tail_count = s_cnt;
        ctl->stats[CBTM_STAT_LIVE_BEFORE] = n;
        ctl->stats[CBTM_STAT_RESERVED] = T;
    }
}

// P2c: scatter the admitted commands (pressure path)
// all_n != 0: every request of the frame's all_n live ranks is admitted (the scan total fits), the
// admission fields of the control block are not consulted (they are written later)
__device__ __forceinline__ void phase_scatter(const FrameArgs &a, uint32_t bid, uint32_t nb, uint32_t all_n = 0)
{
    __shared__ int32_t tail[TAIL_MAX];
    __shared__ uint32_t oom[2];
    const cbtm_pool &p = a.pool;
    const Control *ctl = a.ws.ctl;
    const int tid = threadIdx.x;
    const uint32_t n = all_n ? all_n : (uint32_t)ctl->n;
    const uint32_t nch = (n + CHUNK - 1) / CHUNK;
    const long long i0 = all_n ? (long long)n : ctl->i0;
    const int tail_count = all_n ? 0 : ctl->tail_count;
    if (tid < TAIL_MAX) tail[tid] = tid < tail_count ? ctl->tail_idx[tid] : -1;
    if (tid < 2) oom[tid] = 0;
    __syncthreads();

    uint32_t my_oom_s = 0, my_oom_m = 0;
    for (uint32_t chunk = bid; chunk < nch; chunk += nb) {
        const uint32_t i = chunk * CHUNK + tid;
        if (i >= n) continue;
        const uint32_t need = a.ws.need8[i];
        if (!need) continue;
        bool accepted = (long long)i < i0;
        if (!accepted) {
            for (int k = 0; k < tail_count; ++k)
                if (tail[k] == (int32_t)i) accepted = true;
        }
        if (!accepted) {
            if (need == 2) ++my_oom_m; else ++my_oom_s;
            continue;
        }
        const int32_t s = p.cache_live[i];
        if (need == 2)
            atomicOr(&p.commands[s], (uint32_t)a.ws.mbits8[i]);
        else
            walk_split_chain(p, s);
    }
    if (i0 < (long long)n) { // only frames under reservation pressure count rejections
        if (my_oom_s) atomicAdd(&oom[0], my_oom_s);
        if (my_oom_m) atomicAdd(&oom[1], my_oom_m);
        __syncthreads();
        if (tid < 2 && oom[tid])
            atomicAdd((unsigned long long *)&a.ws.ctl->stats[tid], (unsigned long long)oom[tid]);
    }
}

// ---------------------------------------------------------------------------
// stage 5a: with all commands final, snapshot the merge agreement of every
// live slot (merge_ref: owner and pair of every agreed-merge member) and count
// each rank's allocations (kernels.py:347-368).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void phase_agree(const FrameArgs &a, uint32_t n, uint32_t bid, uint32_t nb,
                                            Carry *carry = nullptr)
{
    __shared__ uint32_t wsum[CHUNK / 32];
    __shared__ uint32_t acc[4];
    const cbtm_pool &p = a.pool;
    const uint32_t nch = (n + CHUNK - 1) / CHUNK;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // The frame's counters (kernels.py:609-632 counts them in stage 8) are decided here: who is
    // consumed by a split, who by an agreed merge, how many slots each allocates.  Counting them
    // now lets the frame publish its UpdateStats two phases before it has been applied.
    uint32_t split_freed = 0, merge_freed = 0, split_alloc = 0, merge_alloc = 0;
    if (tid < 4) acc[tid] = 0; // (ordered before the atomics below by the barriers of the chunk loop / the one after it)
    for (uint32_t chunk = bid; chunk < nch; chunk += nb) {
        const uint32_t i = chunk * CHUNK + tid;
        uint32_t na = 0;
        if (i < n) {
            const bool carried = carry && chunk == bid; // CTA-uniform
            const int32_t s = carried ? carry->s[tid] : p.cache_live[i];
            const int32_t j4_hint = carried ? carry->j4[tid] : a.ws.j4s[i]; // meaningful only under a QUAD command of this frame
            // the record's fields together with its command word: one round trip instead of two
            // (carried: the command word alone)
            const uint32_t cmd = p.commands[s];
            const uint64_t js = carried ? ((uint64_t)carry->id_hi[tid] << 32) | carry->id_lo[tid] : p.ids[s];
            const int32_t nx = carried ? carry->nx[tid] : p.nexts[s], pv = carried ? carry->pv[tid] : p.prevs[s];
            const uint32_t sm = cmd & CBTM_CMD_SPLIT_MASK;
            int32_t ref = -1;
            if (sm) {
                na = 2 + ((sm >> 1) & 1) + ((sm >> 2) & 1);
                ++split_freed;
                split_alloc += na;
            } else if (cmd & CBTM_CMD_MERGE) {
                const MergeCfg c = merge_config_admitted(js, nx, pv, cmd, j4_hint);
                // one round trip: the members' command words and ids
                const uint32_t c_sib = p.commands[c.sib];
                const uint64_t jb = p.ids[c.sib];
                uint32_t c_oth = CBTM_CMD_MERGE, c_j4 = CBTM_CMD_MERGE;
                uint64_t jo = ~0ull, j4 = ~0ull;
                if (c.kind == 2) {
                    c_oth = p.commands[c.oth];
                    c_j4 = p.commands[c.j4];
                    jo = p.ids[c.oth];
                    j4 = p.ids[c.j4];
                }
                if (wants_only_merge(c_sib) && wants_only_merge(c_oth) && wants_only_merge(c_j4)) {
                    // owner = member with the smallest id (kernels.py:159-180)
                    int32_t owner = s;
                    uint64_t best = js;
                    if (jb < best) best = jb, owner = c.sib;
                    if (jo < best) best = jo, owner = c.oth;
                    if (j4 < best) best = j4, owner = c.j4;
                    ref = 2 * owner + ((c.kind == 2 && (js >> 1) != (best >> 1)) ? 1 : 0);
                    if (cmd & CBTM_CMD_OWNER) na = (cmd & CBTM_CMD_QUAD) ? 2 : 1;
                    ++merge_freed; // every member of an agreed merge is consumed; the owner allocates
                    merge_alloc += na;
                }
            }
            a.ws.merge_ref[s] = ref;
            a.ws.nalloc8[i] = (uint8_t)na;
            if (carried) {
                carry->cmd[tid] = cmd;
                carry->mref[tid] = ref;
                carry->na[tid] = na;
            }
        }
        const uint32_t sum = warp_sum(na);
        if (lane == 0) wsum[warp] = sum;
        __syncthreads();
        if (tid == 0) {
            uint32_t ts = 0;
#pragma unroll
            for (int w = 0; w < CHUNK / 32; ++w) ts += wsum[w];
            a.ws.chunk_alloc[chunk] = ts;
        }
        __syncthreads();
    }
    __syncthreads();
    // one atomic per counter and warp in shared memory, one per counter and CTA in global memory
    const uint32_t w_sf = warp_sum(split_freed), w_mf = warp_sum(merge_freed);
    const uint32_t w_sa = warp_sum(split_alloc), w_ma = warp_sum(merge_alloc);
    if (lane == 0) {
        if (w_sf) atomicAdd(&acc[0], w_sf);
        if (w_mf) atomicAdd(&acc[1], w_mf);
        if (w_sa) atomicAdd(&acc[2], w_sa);
        if (w_ma) atomicAdd(&acc[3], w_ma);
    }
    __syncthreads();
    if (tid < 4 && acc[tid])
        atomicAdd((unsigned long long *)&a.ws.ctl->stats[CBTM_STAT_SPLIT_FREED + tid], (unsigned long long)acc[tid]);
}

// sum of v[lo, hi) by the whole CTA (every thread gets it); scratch: CHUNK / 32 words.
// between_loads_and_barrier() runs once the loads have been issued and before the first CTA barrier (for
// shared-memory stores that wait on loads of their own and want the barrier)
template <typename F>
__device__ __forceinline__ uint64_t cta_range_sum(const uint32_t *v, uint32_t lo, uint32_t hi, unsigned long long *scratch,
                                                  F between_loads_and_barrier)
{
    unsigned long long acc = 0;
    for (uint32_t j = lo + threadIdx.x; j < hi; j += CHUNK) acc += v[j];
    between_loads_and_barrier();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL_MASK, acc, o);
    if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = acc;
    __syncthreads();
    unsigned long long total = 0;
#pragma unroll
    for (int w = 0; w < CHUNK / 32; ++w) total += scratch[w];
    __syncthreads();
    return total;
}

__device__ __forceinline__ uint64_t cta_range_sum(const uint32_t *v, uint32_t lo, uint32_t hi, unsigned long long *scratch)
{
    return cta_range_sum(v, lo, hi, scratch, [] {});
}

// ---------------------------------------------------------------------------
// P4 = stage 5b: hand out free slots.  Rank i owns free ranks [T - incl_i, ...):
// windows are popped from the top of the reserved range exactly like the serial
// atomic_sub of kernels.py:357-360.  The exclusive prefix of a chunk is a range
// sum over the chunk counts before it, computed redundantly by the CTA that
// needs it (the counts of a frame are a few KB that every CTA reads from L2 in
// one round trip) -- cheaper than a single-CTA scan phase between two barriers.
// The 256 ranks of a chunk draw ONE contiguous interval of free ranks
// [T - off - total, T - off), total <= 1024.  With the window table the CTA
// expands the free bits of the few leaf blocks that hold that interval into
// shared memory (a warp per leaf block, like the index phase) and every thread
// then just picks its slots; outside the table (fragmented pool) each thread
// descends the tree.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void phase_reserve(const FrameArgs &a, uint32_t n, uint32_t bid, uint32_t nb,
                                              Carry *carry = nullptr)
{
    __shared__ uint32_t scratch[32];
    __shared__ unsigned long long scratch64[CHUNK / 32];
    __shared__ int32_t slots[4 * CHUNK];
    __shared__ uint32_t s_j0;
    const cbtm_pool &p = a.pool;
    Control *ctl = a.ws.ctl;
    const Geo g = make_geo(p.depth);
    const uint32_t nch = (n + CHUNK - 1) / CHUNK;
    const long long T = ctl->T;
    const bool full = p.flags & CBTM_POOL_FULL_FREE_CACHE;
    const uint32_t *win = a.ws.win_prefix;
    const uint32_t *bits32 = reinterpret_cast<const uint32_t *>(p.bits);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    WORK_END(ctl, 6); // (debug) latest CTA entering the phase = barrier exit skew
    const uint32_t win_n = ctl->win_n, win_lo = ctl->win_lo; // CTA-uniform: written before the last barrier
    const uint32_t win_first = win[0]; // (garbage while win_n == 0, never used then)
    // The window table of a frame is short (one entry per leaf block the frame allocates from: a few
    // dozen): it is copied into shared memory while the first chunk's prefix loads are in flight, so that
    // finding the chunk's window block afterwards is not another round trip to L2.
    __shared__ uint32_t s_win[WIN_SMEM + 1];
    const bool win_cached = win_n != 0 && win_n <= (uint32_t)WIN_SMEM; // CTA-uniform
    uint32_t wreg[WIN_SMEM / CHUNK + 1];
    if (win_cached) {
#pragma unroll
        for (int k = 0; k <= WIN_SMEM / CHUNK; ++k) {
            const uint32_t j = (uint32_t)k * CHUNK + tid;
            wreg[k] = j <= win_n ? win[j] : 0u;
        }
    }
    bool win_pending = win_cached;
    const uint32_t *wtab = win_cached ? s_win : win;

    long long off = 0;      // slots allocated by chunks [0, summed)
    uint32_t summed = 0;
    uint32_t totals = 0; // lane k: the count of the k-th of this CTA's next 32 chunks (one round trip for 32 of them)
    for (uint32_t chunk = bid, k32 = 0; chunk < nch; chunk += nb, k32 = (k32 + 1) & 31u) {
        // one round trip: the chunk's own count, this rank's count and slot, and the counts of the
        // chunks between the previous chunk of this CTA and this one
        if (k32 == 0) {
            const uint64_t mine = chunk + (uint64_t)lane * nb;
            totals = mine < nch ? a.ws.chunk_alloc[mine] : 0u;
        }
        const uint32_t total = __shfl_sync(FULL_MASK, totals, (int)k32);
        // A CTA with many chunks (10^5 .. 10^7 live bisectors) does not sum the counts in front of a chunk
        // that allocates nothing: the sum is caught up by the next chunk that does (most chunks of a quiet
        // frame allocate nothing, and every sum is a round trip and two CTA barriers).  With one chunk per
        // CTA the sum is issued together with `total` instead of behind it.
        if (nch > nb && total == 0) continue; // CTA-uniform
        const uint32_t i = chunk * CHUNK + tid;
        const bool carried = carry && chunk == bid; // CTA-uniform
        const uint32_t na = i < n ? (carried ? carry->na[tid] : a.ws.nalloc8[i]) : 0;
        const int32_t s = i < n ? (carried ? carry->s[tid] : p.cache_live[i]) : -1;
        off += (long long)cta_range_sum(a.ws.chunk_alloc, summed, chunk, scratch64, [&] {
            if (win_pending) { // (first chunk: the table lands next to the prefix; the barriers of the sum publish it)
#pragma unroll
                for (int k = 0; k <= WIN_SMEM / CHUNK; ++k) {
                    const uint32_t j = (uint32_t)k * CHUNK + tid;
                    if (j <= win_n) s_win[j] = wreg[k];
                }
            }
        });
        win_pending = false;
        summed = chunk;
        if (total == 0) continue; // CTA-uniform
        PROBE(14); // reserve: prefix known
        uint32_t total_chk;
        const uint32_t incl = block_inclusive_scan<CHUNK>(na, scratch, &total_chk);

        const long long base = T - (off + incl); // this rank's first free rank
        const uint32_t lo_rank = (uint32_t)(T - off - total), hi_rank = (uint32_t)(T - off);
        const bool coop = !full && win_n != 0 && lo_rank >= win_first;
        if (coop) {
            // window block holding the lowest rank of the chunk; windows sit near the top of the table
            uint32_t top = win_n;
            while (true) {
                bool hit = false;
                if ((uint32_t)tid < top) {
                    const uint32_t j = top - 1 - tid;
                    if (wtab[j] <= lo_rank && lo_rank < wtab[j + 1]) {
                        s_j0 = j;
                        hit = true;
                    }
                }
                if (__syncthreads_or(hit) || top <= (uint32_t)CHUNK) break;
                top -= CHUNK;
            }
            WORK_END(ctl, 7); // window block found
            PROBE(15);
            // The interval may span many leaf blocks when the pool is dense around it (few free slots per
            // block): a warp per block, and the next block's table entry and bits are fetched while the
            // current one is expanded (one round trip per block otherwise).
            const uint32_t valid = g.span >= 1024 ? 32u
                                 : (lane * 32u >= g.span ? 0u : (g.span - lane * 32u >= 32u ? 32u : g.span - lane * 32u));
            const uint32_t vmask = valid == 32 ? 0xffffffffu : (valid ? (1u << valid) - 1u : 0u);
            auto fetch = [&](uint32_t j, uint32_t &first, uint32_t &word) {
                first = 0xffffffffu; // beyond the table: ends the loop
                word = 0;
                if (j < win_n) {
                    first = wtab[j]; // free rank of the block's first free slot
                    // (with the table in shared memory `first` is known at once: a block beyond the chunk's
                    // interval is not fetched -- its line would come from DRAM and the warp would wait for it)
                    if (!win_cached || first < hi_rank)
                        word = valid ? bits32[(size_t)(win_lo + j) * 32 + lane] : 0xffffffffu;
                }
            };
            uint32_t first, word, first_nx, word_nx;
            fetch(s_j0 + warp, first, word);
            PROBE_W(27, word ^ first); // reserve: first block's bits arrived
            for (uint32_t j = s_j0 + warp; first < hi_rank; j += CHUNK / 32) {
                fetch(j + CHUNK / 32, first_nx, word_nx);
                const uint32_t b = win_lo + j;
                uint32_t z = ~word & vmask;
                const uint32_t c = __popc(z);
                uint32_t r = first + warp_inclusive_scan(c) - c; // free rank of this lane's first free slot
                const int32_t lane_base = (int32_t)(b * g.span + lane * 32);
                if (r + c > lo_rank && r < hi_rank) { // some of this word's free slots are wanted
                    // Bit by bit, BRANCH FREE: the position in the interval is an unsigned counter that is in
                    // range iff it is below the interval's length (ranks before the interval wrap around),
                    // a step is test-bit / compare / predicated store / add.  (Written with the store and
                    // the increment inside `if (bit)` the compiler emitted a divergent branch with a
                    // reconvergence barrier per step: 32 of them, ~2 us per leaf block and the longest
                    // step of the phase.)
                    uint32_t at = r - lo_rank;
                    const uint32_t len = hi_rank - lo_rank;
#pragma unroll
                    for (int k = 0; k < 32; ++k) {
                        const uint32_t bit = (z >> k) & 1u;
                        if (bit != 0u && at < len) slots[at] = lane_base + k;
                        at += bit;
                    }
                }
                first = first_nx;
                word = word_nx;
            }
            PROBE_W(28, first); // reserve: this warp's blocks expanded
            __syncthreads();
            WORK_END(ctl, 8); // slots expanded
            PROBE(16);
        }
        if (na) {
            for (uint32_t k = 0; k < na; ++k) {
                const long long r = base + k;
                int32_t slot;
                if (full) {
                    slot = p.cache_free[r];
                } else {
                    slot = coop ? slots[(uint32_t)r - lo_rank] : cbt_find<false>(p.bits, p.counters, g, (uint32_t)r);
                    p.cache_free[r] = slot;
                }
                p.reserved[4 * (size_t)s + k] = slot;
                if (carried) carry->res[k][tid] = slot;
            }
        }
        __syncthreads(); // slots / s_j0 are reused by the next chunk
    }
    if (bid == nb - 1) { // totals of the allocation scan
        const long long A = off + (long long)cta_range_sum(a.ws.chunk_alloc, summed, nch, scratch64);
        if (tid == 0) {
            ctl->A = A;
            ctl->stats[CBTM_STAT_ALLOCATED] = A;
            p.counter[0] = T - A; // reservation slack left in the counter (kernels.py:357)
        }
    }
}

// ---------------------------------------------------------------------------
// stages 6 + 7 + 8 fused: write the fresh records, redirect surviving
// neighbours, flip the occupancy bits.
//
// Why fusing is safe: fresh records go to slots that were free at frame start
// and are read by nobody this frame; redirects touch only pointer fields of
// *surviving* records, one writer per field (kernels.py:533-594); everything a
// fill or a redirect reads is either a consumed record (never rewritten), a
// command word (final since k_scatter), a reservation (final since k_reserve)
// or the agreement snapshot merge_ref (final since k_agree).
// ---------------------------------------------------------------------------
enum { E_TWIN = 0, E_NEXT = 1, E_PREV = 2 };
enum { H_WHOLE = 0, H_V0 = 1, H_V1 = 2, H_V2 = 3 };

// PIECE_IDX of kernels.py:50-72 derived from the child layout: the v0-side half
// of a split bisector yields [2j] or [4j, 4j+1], the v1-side half follows with
// [2j+1] or [4j+2, 4j+3].
__device__ __forceinline__ int piece_index(uint32_t mask, int edge, int half)
{
    const int left_n = (mask & CBTM_CMD_SPLIT_P) ? 2 : 1;
    const int right_n = (mask & CBTM_CMD_SPLIT_N) ? 2 : 1;
    const int last = left_n + right_n - 1;
    if (edge == E_TWIN) return half == H_V0 ? 0 : (half == H_V1 ? last : -1);
    if (edge == E_NEXT) {
        if (right_n == 1) return half == H_WHOLE ? left_n : -1;
        return half == H_V1 ? last : (half == H_V2 ? left_n : -1);
    }
    if (left_n == 1) return half == H_WHOLE ? 0 : -1;
    return half == H_V0 ? 0 : (half == H_V2 ? 1 : -1);
}

// (my edge, my half) seen from the neighbour answering through t_role
// (kernels.py:75-100; vertex correspondences of state.py:271-279)
__device__ __forceinline__ void correspond(int my_side, int my_half, int t_role, int &t_edge, int &t_half)
{
    if (my_side == E_TWIN) {
        t_edge = t_role;
        if (t_role == E_TWIN) t_half = my_half == H_V1 ? H_V0 : H_V1;
        else if (t_role == E_PREV) t_half = my_half == H_V0 ? H_V2 : H_V0;
        else t_half = my_half == H_V0 ? H_V1 : H_V2;
    } else if (my_side == E_NEXT) {
        if (t_role == E_PREV) {
            t_edge = E_PREV;
            t_half = my_half == H_WHOLE ? H_WHOLE : (my_half == H_V1 ? H_V0 : H_V2);
        } else {
            t_edge = E_TWIN;
            t_half = my_half == H_V1 ? H_V0 : H_V1;
        }
    } else {
        if (t_role == E_NEXT) {
            t_edge = E_NEXT;
            t_half = my_half == H_WHOLE ? H_WHOLE : (my_half == H_V0 ? H_V1 : H_V2);
        } else {
            t_edge = E_TWIN;
            t_half = my_half == H_V0 ? H_V1 : H_V0;
        }
    }
}

// Everything stage 6/7 ever asks about one pre-update neighbour, fetched with
// six independent loads (one round trip) instead of a chain of dependent ones.
struct Neighbour {
    int32_t slot;     // -1: no neighbour
    uint32_t cmd;     // its command word (final since k_scatter)
    int32_t tw, nx, pv;
    int4 res;         // its reservation (final since k_reserve)
    int32_t mref;     // its agreed-merge reference (k_agree), -1 if none
    int32_t parent;   // slot of the parent that replaces it if it is a member of an agreed merge
                      // (resolve_parent; one more dependent load, issued for all neighbours together)
};

struct ApplyCtx {
    const cbtm_pool &p;
    const int32_t *merge_ref;
    uint8_t *dirty;
    uint32_t poison;
};

__device__ __forceinline__ Neighbour load_neighbour(const ApplyCtx &cx, int32_t slot)
{
    Neighbour nbr;
    nbr.slot = slot;
    if (slot < 0) {
        nbr.cmd = 0;
        nbr.tw = nbr.nx = nbr.pv = nbr.mref = nbr.parent = -1;
        nbr.res = make_int4(-1, -1, -1, -1);
        return nbr;
    }
    nbr.parent = -1;
    const cbtm_pool &p = cx.p;
    nbr.cmd = p.commands[slot];
    nbr.tw = p.twins[slot];
    nbr.nx = p.nexts[slot];
    nbr.pv = p.prevs[slot];
    nbr.res = *reinterpret_cast<const int4 *>(p.reserved + 4 * (size_t)slot);
    nbr.mref = cx.merge_ref[slot];
    return nbr;
}

// kernels.py:183-191 / 159-180: does the neighbour vanish into an agreed merge?
__device__ __forceinline__ bool merges_away(const Neighbour &t)
{
    return t.slot >= 0 && !(t.cmd & CBTM_CMD_SPLIT_MASK) && (t.cmd & CBTM_CMD_MERGE) && t.mref >= 0;
}

// parent slot held by the merge owner; call it for all neighbours before using any result
__device__ __forceinline__ void resolve_parent(const ApplyCtx &cx, Neighbour &t)
{
    if (merges_away(t)) t.parent = cx.p.reserved[4 * (size_t)(t.mref >> 1) + (t.mref & 1)];
}

__device__ __forceinline__ int32_t pick4(const int4 &v, int idx)
{
    return idx == 0 ? v.x : idx == 1 ? v.y : idx == 2 ? v.z : v.w;
}

// post-update slot of the record across (my_side, my_half); kernels.py:194-238
__device__ __forceinline__ int32_t piece_of(ApplyCtx &cx, const Neighbour &t, int my_side, int my_half,
                                            int32_t backref)
{
    if (t.slot < 0) return -1;
    const uint32_t sm = t.cmd & CBTM_CMD_SPLIT_MASK;
    if (sm) {
        int role = -1;
        if (my_side == E_TWIN) {
            if (t.tw == backref) role = E_TWIN;
            else if (t.nx == backref) role = E_NEXT;
            else if (t.pv == backref) role = E_PREV;
        } else if (my_side == E_NEXT) {
            if (t.pv == backref) role = E_PREV;
            else if (t.tw == backref) role = E_TWIN;
        } else {
            if (t.nx == backref) role = E_NEXT;
            else if (t.tw == backref) role = E_TWIN;
        }
        int idx = -1;
        if (role >= 0) {
            int t_edge, t_half;
            correspond(my_side, my_half, role, t_edge, t_half);
            idx = piece_index(sm, t_edge, t_half);
        }
        if (idx < 0) {
            ++cx.poison;
            return -2;
        }
        return pick4(t.res, idx);
    }
    if ((t.cmd & CBTM_CMD_MERGE) && t.mref >= 0) return t.parent; // kernels.py:159-180 (resolve_parent)
    return t.slot;
}

// kernels.py:183-191
__device__ __forceinline__ bool survives(const Neighbour &t)
{
    if (t.cmd & CBTM_CMD_SPLIT_MASK) return false;
    return !((t.cmd & CBTM_CMD_MERGE) && t.mref >= 0);
}

// kernels.py:514-530.  The bundle's pointer values are as good as fresh ones:
// a field equal to old_slot has exactly one writer (this thread).
__device__ __forceinline__ void redirect_to(const cbtm_pool &p, const Neighbour &t, int32_t old_slot,
                                            int32_t new_slot, int first)
{
    if (first == E_PREV) {
        if (t.pv == old_slot) {
            p.prevs[t.slot] = new_slot;
            return;
        }
    } else {
        if (t.nx == old_slot) {
            p.nexts[t.slot] = new_slot;
            return;
        }
    }
    if (t.tw == old_slot) p.twins[t.slot] = new_slot;
}

// Every flipped occupancy bit marks its leaf block in the dirty map, so the
// frame's reduction recounts only the touched blocks (upper_reduce_phase).
struct BitSink {
    uint32_t *bits32;
    uint8_t *dirty;
};

__device__ __forceinline__ void set_live(const BitSink &b, int32_t slot)
{
    atomicOr(&b.bits32[slot >> 5], 1u << (slot & 31));
    b.dirty[(uint32_t)slot >> LEAF_LOG2] = 1;
}

// Stage 8 for a whole warp at once.  The slots a warp flips are neighbours -- consecutive ranks free
// consecutive live slots and reserve consecutive free ranks -- so its lanes hit a handful of 32-bit words
// of the bitfield and ONE byte of the dirty map; sent one by one, a frame's ~50 k atomics and as many
// mark stores queue up on a few L2 sectors (same-address requests are served one per clock by their
// slice) and their drain is the tail of the apply phase.  Here a lane hands in one (word, mask) pair;
// runs of lanes with the same word (the active list is sorted by slot, so equal words sit in
// neighbouring lanes) are OR-ed together with five shuffle steps and the first lane of each run issues
// ONE atomic and ONE mark.  Correct for any arrangement of the words: a lane is skipped only if the lane
// before it carries the same word, and then that run's leader has collected its bits; OR / AND-NOT are
// idempotent, so bits that two leaders both collected do no harm.  word = ~0u: nothing to flip.
// All 32 lanes must call it.
__device__ __forceinline__ void warp_flip(const BitSink &b, uint32_t word, uint32_t mask, bool live, int lane)
{
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t w2 = __shfl_down_sync(FULL_MASK, word, d);
        const uint32_t m2 = __shfl_down_sync(FULL_MASK, mask, d);
        if (lane + d < 32 && w2 == word) mask |= m2;
    }
    const uint32_t before = __shfl_up_sync(FULL_MASK, word, 1);
    if (word != ~0u && (lane == 0 || before != word)) {
        if (live) atomicOr(&b.bits32[word], mask);
        else atomicAnd(&b.bits32[word], ~mask);
        b.dirty[word >> (LEAF_LOG2 - 5)] = 1;
    }
}

// the slot a bisector frees and the first `na` of the slots it reserved (all lanes of the warp call it;
// freed < 0: nothing freed)
__device__ __forceinline__ void warp_flip_bits(const BitSink &b, int32_t freed, uint32_t na, int4 res, int lane)
{
    warp_flip(b, freed >= 0 ? (uint32_t)freed >> 5 : ~0u, freed >= 0 ? 1u << (freed & 31) : 0u, false, lane);
    // the 2..4 reserved slots are consecutive free ranks: almost always one word, sometimes two; whatever
    // does not share the first slot's word goes out on its own
    int32_t slot[4] = {na > 0 ? res.x : -1, na > 1 ? res.y : -1, na > 2 ? res.z : -1, na > 3 ? res.w : -1};
    uint32_t word = ~0u, mask = 0;
    if (slot[0] >= 0) {
        word = (uint32_t)slot[0] >> 5;
        mask = 1u << (slot[0] & 31);
#pragma unroll
        for (int k = 1; k < 4; ++k)
            if (slot[k] >= 0 && ((uint32_t)slot[k] >> 5) == word) {
                mask |= 1u << (slot[k] & 31);
                slot[k] = -1;
            }
    }
    warp_flip(b, word, mask, true, lane);
#pragma unroll
    for (int k = 1; k < 4; ++k)
        if (slot[k] >= 0) set_live(b, slot[k]);
}

// a consumed bisector's own record, fetched together with its command word (or carried)
struct OwnRecord {
    uint64_t id;
    int32_t nx, pv, tw;
    int4 res;
};

__device__ __forceinline__ OwnRecord load_own(const cbtm_pool &p, int32_t s)
{
    OwnRecord r;
    r.id = p.ids[s];
    r.nx = p.nexts[s];
    r.pv = p.prevs[s];
    r.tw = p.twins[s];
    r.res = *reinterpret_cast<const int4 *>(p.reserved + 4 * (size_t)s);
    return r;
}

// tn / tp / tt: the resolved bundles of the neighbours across the next, prev and twin edge (phase_apply
// fetches them: bundles, then the parents of those that merge away; only then is anything consumed or
// stored -- a store in between would serialise the loads)
__device__ __forceinline__ void apply_split(ApplyCtx &cx, int32_t s, uint32_t sm, const OwnRecord &own,
                                            const Neighbour &tn, const Neighbour &tp, const Neighbour &tt)
{
    const cbtm_pool &p = cx.p;
    const uint64_t j = own.id;
    const int32_t nb_n = own.nx, nb_p = own.pv;
    const int4 r4 = own.res;
    const bool split_p = sm & CBTM_CMD_SPLIT_P, split_n = sm & CBTM_CMD_SPLIT_N;
    const int left_n = split_p ? 2 : 1;
    const int32_t left_last = split_p ? r4.y : r4.x;
    const int32_t right_first = split_p ? r4.z : r4.y;
    const int32_t right_second = split_p ? r4.w : r4.z;
    const int32_t t_v0 = piece_of(cx, tt, E_TWIN, H_V0, s), t_v1 = piece_of(cx, tt, E_TWIN, H_V1, s);
    const int32_t p_a = piece_of(cx, tp, E_PREV, split_p ? H_V0 : H_WHOLE, s);
    const int32_t p_b = split_p ? piece_of(cx, tp, E_PREV, H_V2, s) : -1;
    const int32_t n_a = piece_of(cx, tn, E_NEXT, split_n ? H_V2 : H_WHOLE, s);
    const int32_t n_b = split_n ? piece_of(cx, tn, E_NEXT, H_V1, s) : -1;

    // stage 6: fresh records (kernels.py:373-461 restated over the two halves of the bisector)
    if (!split_p) {
        const int32_t a = r4.x;
        p.ids[a] = j << 1;
        p.nexts[a] = right_first;
        p.prevs[a] = t_v0;
        p.twins[a] = p_a;
    } else {
        const int32_t a = r4.x, b = r4.y;
        p.ids[a] = j << 2;
        p.twins[a] = t_v0;
        p.nexts[a] = b;
        p.prevs[a] = p_a;
        p.ids[b] = (j << 2) + 1;
        p.twins[b] = right_first;
        p.prevs[b] = a;
        p.nexts[b] = p_b;
    }
    if (!split_n) {
        const int32_t c = right_first;
        p.ids[c] = (j << 1) + 1;
        p.prevs[c] = left_last;
        p.nexts[c] = t_v1;
        p.twins[c] = n_a;
    } else {
        const int32_t c = right_first, d = right_second;
        p.ids[c] = (j << 2) + 2;
        p.twins[c] = left_last;
        p.nexts[c] = d;
        p.prevs[c] = n_a;
        p.ids[d] = (j << 2) + 3;
        p.prevs[d] = c;
        p.twins[d] = t_v1;
        p.nexts[d] = n_b;
    }

    // stage 7: surviving neighbours across unsplit edges (kernels.py:547-561)
    if (!split_n && nb_n >= 0 && survives(tn)) redirect_to(p, tn, s, right_first, E_PREV);
    if (!split_p && nb_p >= 0 && survives(tp)) redirect_to(p, tp, s, r4.x, E_NEXT);

    // (stage 8: phase_apply flipped the bits of this bisector's slot and of its reservation up front)
    (void)left_n;
    PROBE_W(25, 0); // apply: split stores issued
}

// one sibling pair (even id e, odd id o) collapses into parent slot par; n_ext / q_ext are the
// (resolved) bundles of the neighbours across the odd member's twin edge and the even member's
// twin edge (kernels.py:464-491, 562-594)
__device__ __forceinline__ void apply_merged_pair(ApplyCtx &cx, int32_t e, int32_t o, uint64_t id_e, int32_t par,
                                                  int32_t twin_slot, const Neighbour &n_ext, const Neighbour &q_ext)
{
    const cbtm_pool &p = cx.p;
    const int32_t nx = piece_of(cx, n_ext, E_NEXT, H_WHOLE, o), pv = piece_of(cx, q_ext, E_PREV, H_WHOLE, e);
    p.ids[par] = id_e >> 1;
    p.nexts[par] = nx;
    p.prevs[par] = pv;
    p.twins[par] = twin_slot;
    if (n_ext.slot >= 0 && survives(n_ext)) redirect_to(p, n_ext, o, par, E_PREV);
    if (q_ext.slot >= 0 && survives(q_ext)) redirect_to(p, q_ext, e, par, E_NEXT);
}

// (Dealing the 32-rank groups of the active list round-robin to the warps of the grid was measured too: the
// bisectors a frame consumes are not spread evenly over the ranks -- 38 .. 93 per chunk on average, 256 in
// the fullest chunks of the Earth sweep, benchmarks/apply_imbalance.py -- but a balanced deal gives up the
// carried values, and the two round trips that costs outweigh the balance: 5.4 vs 4.9 us.)
// skip_quiet_warps: for kernels whose CTAs work through many chunks (wide grid, batches) -- most warps of a
// quiet frame flip nothing and skip the shuffles of stage 8 with one vote; in the latency-bound frame of a
// single planet the vote and its branch cost more (apply 4.9 -> 5.2 us) than they can save
__device__ __forceinline__ void phase_apply(const FrameArgs &a, uint32_t n, uint32_t bid, uint32_t nb,
                                            Carry *carry = nullptr, bool skip_quiet_warps = true)
{
    __shared__ uint32_t poisoned;
    const cbtm_pool &p = a.pool;
    const uint32_t nch = (n + CHUNK - 1) / CHUNK;
    const int tid = threadIdx.x;
    if (tid == 0) poisoned = 0;
    __syncthreads();
    ApplyCtx cx{p, a.ws.merge_ref, a.ws.dirty, 0};
    const BitSink bits32{reinterpret_cast<uint32_t *>(p.bits), cx.dirty};

    for (uint32_t chunk = bid; chunk < nch; chunk += nb) {
        const uint32_t i = chunk * CHUNK + tid;
        const bool valid = i < n;
        // round trip 1: by rank; round trip 2: everything about the own record at once
        // (carried: neither -- the thread has all of it from the earlier phases of this frame)
        const bool carried = carry && chunk == bid; // CTA-uniform
        uint32_t na = 0, cmd = 0;
        int32_t s = -1, j4_hint = -1, mref = -1;
        OwnRecord own = {};
        if (valid) {
            na = carried ? carry->na[tid] : a.ws.nalloc8[i];
            s = carried ? carry->s[tid] : p.cache_live[i];
            j4_hint = carried ? carry->j4[tid] : a.ws.j4s[i];
            cmd = carried ? carry->cmd[tid] : p.commands[s];
            mref = carried ? carry->mref[tid] : a.ws.merge_ref[s];
            if (na && carried) {
                own.id = ((uint64_t)carry->id_hi[tid] << 32) | carry->id_lo[tid];
                own.nx = carry->nx[tid];
                own.pv = carry->pv[tid];
                own.tw = carry->tw[tid];
                own.res = make_int4(carry->res[0][tid], carry->res[1][tid], carry->res[2][tid], carry->res[3][tid]);
            } else if (na) {
                own = load_own(p, s);
            }
        }
        const uint32_t sm = cmd & CBTM_CMD_SPLIT_MASK;
        // stage 8 first, by the whole warp (kernels.py:598-632): a bisector that splits or belongs to an
        // agreed merge frees its slot, the first na reserved slots come alive
        const bool consumed = valid && (sm || mref >= 0);
        if (!skip_quiet_warps || __any_sync(FULL_MASK, consumed || na != 0)) // (warp-uniform)
            warp_flip_bits(bits32, consumed ? s : -1, na, own.res, tid & 31);
        if (na == 0) continue; // not allocating: untouched, or a non-owner member of an agreed merge
        // A warp holds splitting bisectors and owners of agreed merges side by side, and the two kinds
        // need different things: the split's three neighbour bundles and their parents; the merge's other
        // members first (kernels.py:464-491, 562-594, 624-628), then the bundles of the pairs' outer
        // neighbours and their parents.  Written as two branches the warp would run one chain of round
        // trips after the other; here the loads of both kinds are issued level by level -- the split's
        // bundles go out while the merge's members are on their way, the bundles of both kinds land in
        // the same four variables, and the parents are resolved by common code -- so the phase is three
        // round trips long, not five.
        const bool is_split = sm != 0;
        MergeCfg c = {0, -1, -1, -1, 0, 0, 0};
        uint64_t id_sib = 0, jo = 0, id_j4 = 0;
        int32_t tw_sib = -1, tw_oth = -1, tw_j4 = -1;
        if (!is_split) { // level 1 of a merge: ids and twin pointers of the other members (parities are not
                         // known yet, so everything that may be needed is fetched)
            c = merge_config_admitted(own.id, own.nx, own.pv, cmd, j4_hint);
            id_sib = p.ids[c.sib];
            tw_sib = p.twins[c.sib];
            if (c.kind == 2) {
                jo = p.ids[c.oth];
                id_j4 = p.ids[c.j4];
                tw_oth = p.twins[c.oth];
                tw_j4 = p.twins[c.j4];
            }
        }
        Neighbour b0, b1, b2, b3; // split: across next, prev, twin, (none); merge: n1, q1, n2, q2
        const bool quad = c.kind == 2;
        const uint64_t js = own.id;
        const bool s_even = !(js & 1);
        if (is_split) { // level 1 of a split
            b0 = load_neighbour(cx, own.nx);
            b1 = load_neighbour(cx, own.pv);
            b2 = load_neighbour(cx, own.tw);
            b3 = load_neighbour(cx, -1);
        }
        bool oth_even = false;
        if (!is_split) { // level 2 of a merge (the members have arrived)
            PROBE_W(21, (uint32_t)id_sib ^ (uint32_t)tw_sib ^ (uint32_t)jo ^ (uint32_t)id_j4 ^ (uint32_t)tw_oth ^ (uint32_t)tw_j4); // apply: merge members arrived
            oth_even = !(jo & 1);
            b0 = load_neighbour(cx, s_even ? tw_sib : own.tw); // across twins[o1]
            b1 = load_neighbour(cx, s_even ? own.tw : tw_sib); // across twins[e1]
            b2 = load_neighbour(cx, quad ? (oth_even ? tw_j4 : tw_oth) : -1);
            b3 = load_neighbour(cx, quad ? (oth_even ? tw_oth : tw_j4) : -1);
        }
        PROBE_W(18, b0.cmd ^ b1.cmd ^ b2.cmd ^ b3.cmd ^ (uint32_t)(b0.res.x ^ b1.res.x ^ b2.res.x ^ b3.res.x ^ b0.mref ^ b1.mref ^ b2.mref ^ b3.mref)); // apply: neighbour bundles arrived
        resolve_parent(cx, b0);
        resolve_parent(cx, b1);
        resolve_parent(cx, b2);
        resolve_parent(cx, b3);
        PROBE_W(19, b0.parent ^ b1.parent ^ b2.parent ^ b3.parent); // apply: parents arrived (first store follows)
        if (is_split) {
            apply_split(cx, s, sm, own, b0, b1, b2);
        } else {
            const int32_t e1 = s_even ? s : c.sib, o1 = s_even ? c.sib : s;
            const int32_t e2 = oth_even ? c.oth : c.j4, o2 = oth_even ? c.j4 : c.oth;
            const int32_t p1 = own.res.x;
            const uint64_t id_e1 = s_even ? js : id_sib;
            if (quad) {
                const int32_t p2 = own.res.y;
                const uint64_t id_e2 = oth_even ? jo : id_j4;
                apply_merged_pair(cx, e1, o1, id_e1, p1, p2, b0, b1);
                apply_merged_pair(cx, e2, o2, id_e2, p2, p1, b2, b3);
            } else {
                apply_merged_pair(cx, e1, o1, id_e1, p1, -1, b0, b1);
            }
            PROBE_W(26, 0); // apply: merge stores issued
        }
    }
    // (the frame's counters were taken in phase_agree; what is left to report is the poison count)
    if (cx.poison) atomicAdd(&poisoned, cx.poison);
    __syncthreads();
    if (tid == 0 && poisoned)
        atomicAdd((unsigned long long *)&a.ws.ctl->stats[CBTM_STAT_POISON], (unsigned long long)poisoned);
}

// ---------------------------------------------------------------------------
// one kernel per phase (staged path)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(CHUNK) k_reset(const __grid_constant__ FrameArgs a)
{
    phase_reset(a, blockIdx.x, gridDim.x);
}

__global__ void __launch_bounds__(CHUNK) k_classify_frame(const __grid_constant__ FrameArgs a)
{
    phase_classify(a, a.pool.counters[1], blockIdx.x, gridDim.x);
}

__global__ void __launch_bounds__(CHUNK) k_admit(const __grid_constant__ FrameArgs a)
{
    const uint32_t n = a.pool.counters[1];
    if (!fits_a_priori(a.pool, n) && !frame_fits(a, n)) phase_admit<CHUNK>(a);
}

__global__ void __launch_bounds__(CHUNK) k_scatter(const __grid_constant__ FrameArgs a)
{
    const uint32_t n = a.pool.counters[1];
    if (!fits_a_priori(a.pool, n)) phase_scatter(a, blockIdx.x, gridDim.x, frame_fits(a, n) ? n : 0);
}

__global__ void __launch_bounds__(CHUNK) k_agree(const __grid_constant__ FrameArgs a)
{
    // n from the CBT root: ctl->n is only written below (fast path) / by k_admit (slow path)
    const uint32_t n = a.pool.counters[1];
    if (blockIdx.x == gridDim.x - 1) {
        frame_totals_and_window(a, n, fits_a_priori(a.pool, n) || frame_fits(a, n));
    }
    phase_agree(a, n, blockIdx.x, gridDim.x);
}

__global__ void __launch_bounds__(CHUNK) k_reserve(const __grid_constant__ FrameArgs a)
{
    phase_reserve(a, (uint32_t)a.ws.ctl->n, blockIdx.x, gridDim.x);
}

__global__ void __launch_bounds__(CHUNK) k_apply(const __grid_constant__ FrameArgs a)
{
    phase_apply(a, (uint32_t)a.ws.ctl->n, blockIdx.x, gridDim.x);
}

__global__ void __launch_bounds__(CHUNK) k_publish(const __grid_constant__ FrameArgs a, int64_t *stats_seq)
{
    const ReducePublish pub = {a.ws.ctl->stats, a.pool.stats, stats_seq, &a.ws.ctl->seq_frame, nullptr};
    publish_frame(pub, a.pool.counters[1], threadIdx.x);
}

// ---------------------------------------------------------------------------
// the persistent frame kernel: n_frames full updates in one cooperative launch
// ---------------------------------------------------------------------------
constexpr int FRAMES_DYN_SMEM = IDX_WARPS * IDX_STAGE_WORDS * 4; // 36 KB: index staging (P1), Carry (P2-P5), tile values (P6)
static_assert(sizeof(Carry) <= FRAMES_DYN_SMEM, "the carry lives in the index staging area");

// CTAS = co-resident CTAs per SM the register budget is cut for: 2 (latency-bound frames of a few hundred
// chunks: fewer CTAs, cheaper barriers, no spills) or 4 (CBTM_POOL_WIDE_GRID, pools with 10^5 .. 10^7 live
// bisectors: a CTA works through its chunks one after the other, each a chain of round trips, so twice the
// CTAs in flight is close to twice the throughput)
template <int CTAS>
__global__ void __launch_bounds__(CHUNK, CTAS)
k_frames(const __grid_constant__ FrameArgs a, int n_frames, int64_t *stats_seq, int do_index,
         const volatile int64_t *mailbox, long long linger_ns, long long next_request)
{
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(128) uint8_t dyn_smem[];
    __shared__ uint32_t wroot[2][RED_THREADS / 32];

    const cbtm_pool &p = a.pool;
    Control *ctl = a.ws.ctl;
    const uint32_t bid = blockIdx.x, nb = gridDim.x;
    const Geo g = make_geo(p.depth);
    const bool stamper = bid == 0 && threadIdx.x == 0;
    int32_t *free_list = (p.flags & CBTM_POOL_FULL_FREE_CACHE) ? p.cache_free : nullptr;

    // linger mode (mailbox != NULL, n_frames == 1): after a frame the kernel polls a host-mapped
    // mailbox for the next request for up to linger_ns and, if one arrives, runs it without a new
    // launch (cbtm_update_linger / cbtm_post_request)
    for (int f = 0; f < n_frames || mailbox; ++f) {
        unsigned long long *stamp = stamper ? ctl->phase_t[f & 1] : nullptr;
        if (stamp) stamp[0] = global_ns();
        PROBE_SET_FRAME(f);
        PROBE_T0(0, f);
        if (do_index)
            index_phase<true>(reinterpret_cast<const uint32_t *>(p.bits), p.counters, p.depth, p.cache_live,
                        free_list, p.dispatch, p.commands,
                        reinterpret_cast<int32_t(*)[IDX_STAGE_WORDS]>(dyn_smem), bid, nb);
        else
            phase_reset(a, bid, nb);
        PROBE(7); // index work done
        grid.sync();
        PROBE_T0(1, f);
        if (stamp) stamp[1] = global_ns();
        const uint32_t n = p.counters[1];      // the frame's live count: one read per CTA, kept in a register
        const bool fast = fits_a_priori(p, n); // grid-uniform
        // (the staging area of the index phase is free until P6; the wide-grid variant goes without: its CTAs
        // work through many chunks, only the first could be carried, and at 64 registers the extra live
        // values spill -- measured at 2 M live bisectors: 87 us per frame without, 93 us with)
        Carry *carry = CTAS == 2 ? reinterpret_cast<Carry *>(dyn_smem) : nullptr;
        phase_classify(a, n, bid, nb, (mailbox && f > 0) ? ctl->mb_prm : nullptr, carry);
        WORK_END(ctl, 1);
        grid.sync();
        const bool fits = fast || frame_fits(a, n); // grid-uniform
        if (!fast) {
            if (fits) { // the total turned out to fit: everything is admitted, scatter now
                phase_scatter(a, bid, nb, n);
            } else { // reservation pressure: one CTA admits (first rejected rank, first-fit tail), then everybody scatters
                if (bid == 0) phase_admit<CHUNK>(a);
                grid.sync();
                phase_scatter(a, bid, nb);
            }
            grid.sync();
        }
        if (stamp) stamp[2] = global_ns();
        PROBE_T0(2, f);
        // T is final: the free-rank window table is built by the CTA with the fewest chunks while the
        // others take the agreement snapshot (it was the straggler of P2 when built there)
        if (bid == nb - 1) {
            frame_totals_and_window(a, n, fits);
            PROBE(12); // window table built
        }
        phase_agree(a, n, bid, nb, carry);
        PROBE(13); // agreement done
        WORK_END(ctl, 2);
        grid.sync();
        if (stamp) stamp[3] = global_ns();
        PROBE_T0(3, f);
        // The launch's last frame: every counter of the frame is decided (admission, agreement,
        // allocation counts), so they go to the host NOW, three phases before the frame is done --
        // ParallelEngine.update returns on them and the host's work between two frames (stats
        // object, next camera, next launch call) overlaps with reserve / apply / reduce instead of
        // following them; the next launch is queued while this one still runs.  The CTA with the
        // fewest chunks does it (none at all for up to 75 k live bisectors).
        if (bid == nb - 1 && !mailbox && f == n_frames - 1 && p.stats)
            publish_early(ctl->stats, p.stats, ctl->phase_t[f & 1], threadIdx.x);
        phase_reserve(a, n, bid, nb, carry);
        PROBE(17); // reserve done
        WORK_END(ctl, 3);
        grid.sync();
        if (stamp) stamp[4] = global_ns();
        PROBE_T0(4, f);
        phase_apply(a, n, bid, nb, carry, CTAS != 2);
        PROBE(20); // apply done
        WORK_END(ctl, 4);
        grid.sync();
        PROBE_T0(5, f);
        if (stamp) {
            stamp[5] = global_ns();
            __threadfence(); // read by the publishing CTA after the next barrier
        }
        // cbtm_update (one frame, counters already on the host since P3): the frame is retired here and
        // the kernel ends with its reduction work, without a barrier and a host write on its tail
        const bool early_only = n_frames == 1 && !mailbox && !stats_seq && p.stats && !(p.flags & CBTM_POOL_FINAL_ROW);
        if (early_only && bid == nb - 1 && threadIdx.x < 32) retire_frame(ctl->stats, &ctl->seq_frame, threadIdx.x);
        upper_reduce_phase(p.bits, a.ws.dirty, p.counters, g.lc, reinterpret_cast<uint32_t *>(dyn_smem), wroot, bid, nb);
        PROBE(22); // reduce done
        WORK_END(ctl, 5);
        if (early_only) break; // grid-uniform
        grid.sync();
        PROBE_T0(6, f);
        // the frame's counters go out while the next frame's index phase is already running
        // (pool->stats may be host-mapped memory: only the launch's last frame pays for that write)
        if (bid == nb - 1) {
            const ReducePublish pub = {ctl->stats, (mailbox || f == n_frames - 1) ? p.stats : nullptr, stats_seq,
                                       &ctl->seq_frame, ctl->phase_t[f & 1]};
            publish_frame(pub, p.counters[1], threadIdx.x);
#ifdef CBTM_DEBUG_TIMING
            if (threadIdx.x < CBTM_STAT_PHASES + 3) {
                // spare probes 6..8 are reported relative to the start of the reserve phase
                const unsigned long long t0 = ctl->phase_t[f & 1][threadIdx.x < CBTM_STAT_PHASES ? threadIdx.x : 3],
                                         t1 = ctl->work_end[threadIdx.x];
                if (stats_seq) stats_seq[(size_t)CBTM_STATS_WORDS * f + 22 + threadIdx.x] = t1 > t0 ? (int64_t)(t1 - t0) : 0;
                ctl->work_end[threadIdx.x] = 0;
            }
#endif
        }
        if (mailbox) {
            // One thread watches the mailbox (a load from host memory every ~1.5 us) until request
            // number next_request + f shows up or the linger time is over; everybody else waits in
            // the barrier.  The host posts a request only while it knows the kernel is still
            // listening (ParallelEngine keeps a safety margin) and otherwise launches afresh, so a
            // request is served exactly once.
            if (bid == 0 && threadIdx.x < 32) { // one warp: lane 0 watches, then 23 lanes fetch the parameters
                int go = 0;
                if (threadIdx.x == 0 && ctl->seq_frame + 1 < (uint32_t)MAX_SEQ_FRAMES) {
                    const unsigned long long t0 = global_ns();
                    const long long want = next_request + f;
                    do {
                        if (mailbox[0] >= want) {
                            go = 1;
                            break;
                        }
                    } while (global_ns() - t0 < (unsigned long long)linger_ns);
                }
                go = __shfl_sync(FULL_MASK, go, 0);
                if (go) {
                    __threadfence_system();
                    // (one load from host memory per lane, all in flight together: a loop in one
                    // thread pays a PCIe round trip per word)
                    if (threadIdx.x < CBTM_PRM_WORDS)
                        ctl->mb_prm[threadIdx.x] = __longlong_as_double(mailbox[8 + threadIdx.x]);
                }
                __syncwarp();
                if (threadIdx.x == 0) {
                    ctl->mb_go = go;
                    __threadfence();
                }
            }
            grid.sync();
            if (!ctl->mb_go) break; // grid-uniform: rewritten only behind the barriers of another frame
        }
    }
}

// ---------------------------------------------------------------------------
// Batches of independent pools (BASELINE config 5: several planets per GPU).
// A frame of one planet leaves the GPU mostly idle (latency bound, a few hundred
// CTAs' worth of work), so the planets of a batch advance in lockstep inside ONE
// cooperative launch: every phase runs over all pools before the grid barrier
// that ends it -- P planets pay for the barriers and the dependent round trips
// of one.  Pool q sees the CTAs rotated by q * nb / P, which spreads the chunks
// (and the admin / single-CTA duties) of the pools over different SMs.
// ---------------------------------------------------------------------------
#ifndef CBTM_BATCH_CTAS_PER_SM
#define CBTM_BATCH_CTAS_PER_SM 4
#endif
constexpr int BATCH_CTAS_PER_SM = CBTM_BATCH_CTAS_PER_SM; // more chunks in flight per SM: a batch has work for them

struct BatchArgs {
    FrameArgs a[CBTM_MAX_BATCH];
    int64_t *stats_seq[CBTM_MAX_BATCH];
};

__global__ void __launch_bounds__(CHUNK, BATCH_CTAS_PER_SM)
k_frames_batch(const __grid_constant__ BatchArgs b, int n_pools, int n_frames)
{
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(128) uint8_t dyn_smem[];
    __shared__ uint32_t wroot[2][RED_THREADS / 32];

    const uint32_t bid = blockIdx.x, nb = gridDim.x;
    const uint32_t shift = nb / (uint32_t)n_pools;
    auto vbid = [&](int q) { return (bid + (uint32_t)q * shift) % nb; };
    auto stamp = [&](int f, int k) { // every pool records the batch's phase boundaries
        if (bid == 0 && threadIdx.x == 0) {
            const unsigned long long t = global_ns();
            for (int q = 0; q < n_pools; ++q) b.a[q].ws.ctl->phase_t[f & 1][k] = t;
        }
    };

    for (int f = 0; f < n_frames; ++f) {
        stamp(f, 0);
        for (int q = 0; q < n_pools; ++q) {
            const FrameArgs &a = b.a[q];
            const cbtm_pool &p = a.pool;
            index_phase<true>(reinterpret_cast<const uint32_t *>(p.bits), p.counters, p.depth, p.cache_live,
                              (p.flags & CBTM_POOL_FULL_FREE_CACHE) ? p.cache_free : nullptr, p.dispatch, p.commands,
                              reinterpret_cast<int32_t(*)[IDX_STAGE_WORDS]>(dyn_smem), vbid(q), nb);
            __syncthreads(); // the staging area is reused by the next pool
        }
        grid.sync();
        stamp(f, 1);
        bool any_late = false; // grid-uniform
        for (int q = 0; q < n_pools; ++q) {
            any_late |= !fits_a_priori(b.a[q].pool, b.a[q].pool.counters[1]);
            phase_classify(b.a[q], b.a[q].pool.counters[1], vbid(q), nb);
            __syncthreads();
        }
        grid.sync();
        // per pool (bit q): 1 = the commands were scattered in P2 or the scan total fits, 0 = pressure
        unsigned fits_mask = 0;
        for (int q = 0; q < n_pools; ++q) {
            const uint32_t nq = b.a[q].pool.counters[1];
            if (fits_a_priori(b.a[q].pool, nq) || frame_fits(b.a[q], nq)) fits_mask |= 1u << q;
        }
        if (any_late) { // pools that could not scatter in P2
            const bool any_pressure = fits_mask != (1u << n_pools) - 1u;
            if (any_pressure) { // one CTA each admits (first rejected rank, first-fit tail)
                for (int q = 0; q < n_pools; ++q)
                    if (vbid(q) == 0 && !((fits_mask >> q) & 1u)) phase_admit<CHUNK>(b.a[q]);
                grid.sync();
            }
            for (int q = 0; q < n_pools; ++q) {
                const uint32_t nq = b.a[q].pool.counters[1];
                if (!fits_a_priori(b.a[q].pool, nq)) {
                    phase_scatter(b.a[q], vbid(q), nb, ((fits_mask >> q) & 1u) ? nq : 0u);
                    __syncthreads();
                }
            }
            grid.sync();
        }
        stamp(f, 2);
        for (int q = 0; q < n_pools; ++q) {
            const uint32_t nq = b.a[q].pool.counters[1];
            if (vbid(q) == nb - 1) {
                frame_totals_and_window(b.a[q], nq, (fits_mask >> q) & 1u);
            }
            phase_agree(b.a[q], nq, vbid(q), nb);
            __syncthreads();
        }
        grid.sync();
        stamp(f, 3);
        for (int q = 0; q < n_pools; ++q) {
            phase_reserve(b.a[q], (uint32_t)b.a[q].ws.ctl->n, vbid(q), nb);
            __syncthreads();
        }
        grid.sync();
        stamp(f, 4);
        for (int q = 0; q < n_pools; ++q) {
            phase_apply(b.a[q], (uint32_t)b.a[q].ws.ctl->n, vbid(q), nb);
            __syncthreads();
        }
        grid.sync();
        stamp(f, 5);
        if (bid == 0 && threadIdx.x == 0) __threadfence();
        for (int q = 0; q < n_pools; ++q) {
            const cbtm_pool &p = b.a[q].pool;
            upper_reduce_phase(p.bits, b.a[q].ws.dirty, p.counters, make_geo(p.depth).lc,
                               reinterpret_cast<uint32_t *>(dyn_smem), wroot, vbid(q), nb);
            __syncthreads();
        }
        grid.sync();
        for (int q = 0; q < n_pools; ++q)
            if (vbid(q) == nb - 1) {
                const FrameArgs &a = b.a[q];
                Control *ctl = a.ws.ctl;
                const ReducePublish pub = {ctl->stats, f == n_frames - 1 ? a.pool.stats : nullptr, b.stats_seq[q],
                                           &ctl->seq_frame, ctl->phase_t[f & 1]};
                publish_frame(pub, a.pool.counters[1], threadIdx.x);
                __syncthreads();
            }
    }
}

// ---------------------------------------------------------------------------
// structural validator (state.py:169-203): one thread per slot, live slots only
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
k_validate(const cbtm_pool p, int n_halfedges, unsigned long long *out)
{
    __shared__ unsigned long long acc[6];
    if (threadIdx.x < 6) acc[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t N = (uint64_t)1 << p.depth;
    const uint32_t *bits32 = reinterpret_cast<const uint32_t *>(p.bits);
    auto live = [&](int64_t q) { return (bits32[q >> 5] >> (q & 31)) & 1u; };
    unsigned cnt[6] = {0, 0, 0, 0, 0, 0};
    long long first_bad = -1;
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < N;
         s += (uint64_t)gridDim.x * blockDim.x) {
        if (!live((int64_t)s)) continue;
        ++cnt[0];
        const uint64_t id = p.ids[s];
        bool bad = false;
        if (id < ((uint64_t)1 << p.rank)) {
            ++cnt[1];
            if (first_bad < 0) first_bad = (long long)s;
            continue;
        }
        const int d = depth_of(id, p.rank);
        const uint64_t he = (id >> d) - ((uint64_t)1 << p.rank);
        if (he >= (uint64_t)n_halfedges) ++cnt[1], bad = true;
        if (d > p.max_depth) ++cnt[2], bad = true;
        const int32_t ptr[3] = {p.nexts[s], p.prevs[s], p.twins[s]};
#pragma unroll
        for (int role = 0; role < 3; ++role) { // 0 next, 1 prev, 2 twin
            const int64_t q = ptr[role];
            if (q == -1) continue;
            if (q < 0 || (uint64_t)q >= N || !live(q)) {
                ++cnt[3], bad = true;
                continue;
            }
            const bool via_next = p.nexts[q] == (int32_t)s, via_prev = p.prevs[q] == (int32_t)s,
                       via_twin = p.twins[q] == (int32_t)s;
            const bool answered = role == 0 ? (via_prev || via_twin)
                                : role == 1 ? (via_next || via_twin)
                                            : (via_next || via_prev || via_twin);
            if (!answered) ++cnt[4], bad = true;
            const int nd = depth_of(p.ids[q], p.rank);
            if (nd - d > 1 || d - nd > 1) ++cnt[5], bad = true;
        }
        if (bad && first_bad < 0) first_bad = (long long)s;
    }
    for (int k = 0; k < 6; ++k)
        if (cnt[k]) atomicAdd(&acc[k], (unsigned long long)cnt[k]);
    if (first_bad >= 0) atomicMin(reinterpret_cast<unsigned long long *>(out) + 6, (unsigned long long)first_bad);
    __syncthreads();
    if (threadIdx.x < 6 && acc[threadIdx.x]) atomicAdd(&out[threadIdx.x], acc[threadIdx.x]);
}

// ---------------------------------------------------------------------------
// initialize (state.py:139-156)
// ---------------------------------------------------------------------------
__global__ void k_initialize(const cbtm_pool p, const int32_t *__restrict__ he_next,
                             const int32_t *__restrict__ he_prev,
                             const int32_t *__restrict__ he_twin, int n_halfedges, const Workspace ws)
{
    Control *ctl = ws.ctl;
    unsigned *ticket = ws.ticket;
    const uint64_t N = (uint64_t)1 << p.depth;
    const uint64_t base = (uint64_t)1 << p.rank;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t gid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    for (uint64_t s = gid; s < N; s += stride) {
        const bool root = s < (uint64_t)n_halfedges;
        p.ids[s] = root ? base + s : 0;
        p.nexts[s] = root ? he_next[s] : -1;
        p.prevs[s] = root ? he_prev[s] : -1;
        p.twins[s] = root ? he_twin[s] : -1;
        p.commands[s] = 0;
        reinterpret_cast<int4 *>(p.reserved)[s] = make_int4(-1, -1, -1, -1);
        p.cache_live[s] = -1;
        p.cache_free[s] = -1;
    }
    if (ws.dirty) {
        const uint64_t nblk = N >> LEAF_LOG2 ? N >> LEAF_LOG2 : 1;
        for (uint64_t b = gid; b < nblk; b += stride) ws.dirty[b] = 0;
    }
    const uint64_t words = bitfield_words(p.depth);
    for (uint64_t w = gid; w < words; w += stride) {
        const uint64_t first = w * 64;
        uint64_t x = 0;
        if (first + 64 <= (uint64_t)n_halfedges) x = ~(uint64_t)0;
        else if (first < (uint64_t)n_halfedges) x = (((uint64_t)1) << (n_halfedges - first)) - 1;
        p.bits[w] = x;
    }
    if (gid == 0) {
        p.counter[0] = 0;
        p.counters[0] = 0; // no stamp: the reduction that follows rebuilds every level
        if (p.stats)
            for (int k = 0; k < CBTM_STATS_WORDS; ++k) p.stats[k] = 0;
        if (ctl) {
            ctl->n = ctl->F = ctl->T = ctl->A = 0;
            ctl->i0 = 0;
            ctl->tail_count = 0;
            ctl->seq_frame = 0;
            ctl->need_total = 0;
            ticket[0] = 0;
            ticket[1] = 0; // (spare)
            for (int k = 0; k < CBTM_STATS_WORDS; ++k) ctl->stats[k] = 0;
        }
    }
}

} // namespace cbtm
