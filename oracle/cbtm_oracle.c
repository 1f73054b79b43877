/*
 * oracle/cbtm_oracle.c -- CPU restatement of the reference per-frame bisector
 * update (arXiv 2407.02215, reference package `cbtmesh`).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl reference
 * legs may load it.  The product path (paper_2407_02215_b200/csrc) never links
 * or calls anything in this directory.
 *
 * Parity status: PINNED.  oracle/pin_against_reference.py runs this library and
 * the reference's own ParallelEngine(threads=1) (importable in the build
 * container from /root/reference/pkg/src) side by side and requires every
 * array (cbt.nodes, ids, nexts, prevs, twins, commands, reserved, counter,
 * cache_live, cache_free) to be identical after every frame; its digests are
 * committed under tests/golden/ and re-checked by tests/test_oracle_golden.py.
 *
 * Layout is the REFERENCE layout (so dumps compare 1:1 with the reference):
 *   nodes    u32[2N]  binary heap, index 0 padding, leaves at [N, 2N) hold 0/1
 *                     (pkg/src/cbtmesh/cbt.py:21-57)
 *   ids      u64[N], nexts/prevs/twins i32[N] (-1 = null), commands u32[N],
 *   reserved i32[N*4], counter i64[1], cache_live/cache_free i32[N]
 *                     (pkg/src/cbtmesh/state.py:32-55)
 *
 * Build: gcc -O2 -fPIC -shared -ffp-contract=off -fopenmp (see oracle/Makefile).
 * -ffp-contract=off matters: the reference's numba code issues separate
 * multiplies and adds (no FMA), and the classifier must round identically.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* command-word bits, pkg/src/cbtmesh/state.py:17-25 */
enum {
    CMD_SPLIT_T = 1, CMD_SPLIT_N = 2, CMD_SPLIT_P = 4, CMD_SPLIT_MASK = 7,
    CMD_MERGE = 8, CMD_QUAD = 16, CMD_OWNER = 32
};
/* edge roles and sub-segment selectors, pkg/src/cbtmesh/kernels.py:40-48 */
enum { E_TWIN = 0, E_NEXT = 1, E_PREV = 2 };
enum { H_WHOLE = 0, H_V0 = 1, H_V1 = 2, H_V2 = 3 };

typedef struct orc_pool {
    uint64_t *ids;
    int32_t *nexts, *prevs, *twins;
    uint32_t *commands;
    int32_t *reserved; /* [N][4] */
    uint32_t *nodes;   /* [2N] */
    int64_t *counter;  /* [1] */
    int32_t *cache_live, *cache_free;
    int64_t capacity;
    int32_t depth, rank, max_depth, pad_;
} orc_pool;

/* ------------------------------------------------------------------ */
/* CBT: sum reduction and ranked queries                              */
/* ------------------------------------------------------------------ */

/* cbt.py:61-68 / :165-170 -- every internal node = sum of its children,
 * bottom level first. */
void orc_sum_reduce(uint32_t *nodes, int depth, int threads)
{
    for (int level = depth - 1; level >= 0; --level) {
        const int64_t lo = (int64_t)1 << level;
#ifdef _OPENMP
#pragma omp parallel for num_threads(threads) schedule(static) if (threads > 1 && lo >= 4096)
#endif
        for (int64_t k = lo; k < 2 * lo; ++k)
            nodes[k] = nodes[2 * k] + nodes[2 * k + 1];
    }
    (void)threads;
}

/* cbt.py:127-136 -- slot of the (rank+1)-th set bit: descend from the root,
 * going right whenever the rank is not covered by the left child's count. */
int64_t orc_one_to_bit_id(const uint32_t *nodes, int64_t capacity, int64_t rank)
{
    int64_t node = 1;
    while (node < capacity) {
        node *= 2;
        const int64_t left = nodes[node];
        if (rank >= left) {
            rank -= left;
            node += 1;
        }
    }
    return node - capacity;
}

/* cbt.py:139-150 -- same descent over unset bits; the zero count of a left
 * child is its span (halved per level) minus its one-count. */
int64_t orc_zero_to_bit_id(const uint32_t *nodes, int64_t capacity, int64_t rank)
{
    int64_t node = 1;
    int64_t span = capacity / 2;
    while (node < capacity) {
        node *= 2;
        const int64_t left_zeros = span - (int64_t)nodes[node];
        if (rank >= left_zeros) {
            rank -= left_zeros;
            node += 1;
        }
        span /= 2;
    }
    return node - capacity;
}

/* cbt.py:153-162 batch forms */
void orc_one_to_bit_ids(const uint32_t *nodes, int64_t capacity,
                        const int64_t *ranks, int64_t *out, int64_t n)
{
    for (int64_t i = 0; i < n; ++i)
        out[i] = orc_one_to_bit_id(nodes, capacity, ranks[i]);
}

void orc_zero_to_bit_ids(const uint32_t *nodes, int64_t capacity,
                         const int64_t *ranks, int64_t *out, int64_t n)
{
    for (int64_t i = 0; i < n; ++i)
        out[i] = orc_zero_to_bit_id(nodes, capacity, ranks[i]);
}

/* ------------------------------------------------------------------ */
/* id helpers                                                         */
/* ------------------------------------------------------------------ */

static inline int bit_length_u64(uint64_t x)
{
    return x ? 64 - __builtin_clzll(x) : 0;
}

/* bisector.py:91-97 */
static inline int depth_of(uint64_t id, int rank)
{
    return bit_length_u64(id) - 1 - rank;
}

/* ------------------------------------------------------------------ */
/* fp64 triangle decode and verdict sources                            */
/* ------------------------------------------------------------------ */

/* bisector.py:100-183.  Operation order is part of the contract: each matrix
 * row (a, b, c) becomes (c/2, b + c/2, a) for an odd path bit and
 * (a + c/2, c/2, b) for an even one, walking the id from its lowest bit up;
 * the apex is the face mean accumulated along `next`; each coordinate is
 * (m0*r0 + m1*r1) + m2*r2. */
void orc_decode_tri(uint64_t id, int rank, const int32_t *he_next,
                    const int32_t *he_vert, const double *pos, double *out9)
{
    const int d = depth_of(id, rank);
    const uint64_t root = id >> d;
    double m[3][3] = {{1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}};
    for (uint64_t h = id; h != root; h >>= 1) {
        for (int r = 0; r < 3; ++r) {
            const double a = m[r][0], b = m[r][1], c = m[r][2];
            const double hc = 0.5 * c;
            if (h & 1) {
                m[r][0] = hc;
                m[r][1] = b + hc;
                m[r][2] = a;
            } else {
                m[r][0] = a + hc;
                m[r][1] = hc;
                m[r][2] = b;
            }
        }
    }
    const int64_t he = (int64_t)(root - ((uint64_t)1 << rank));
    const int32_t nx = he_next[he];
    const double *p0 = pos + 3 * (int64_t)he_vert[he];
    const double *p1 = pos + 3 * (int64_t)he_vert[nx];
    double s[3] = {p0[0], p0[1], p0[2]};
    int n = 1;
    for (int32_t w = nx; w != he; w = he_next[w]) {
        const double *pw = pos + 3 * (int64_t)he_vert[w];
        s[0] += pw[0];
        s[1] += pw[1];
        s[2] += pw[2];
        ++n;
    }
    const double p2[3] = {s[0] / n, s[1] / n, s[2] / n};
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k)
            out9[3 * r + k] = m[r][0] * p0[k] + m[r][1] * p1[k] + m[r][2] * p2[k];
}

void orc_decode_tris(const uint64_t *ids, int64_t n, int rank,
                     const int32_t *he_next, const int32_t *he_vert,
                     const double *pos, double *out)
{
    for (int64_t i = 0; i < n; ++i)
        orc_decode_tri(ids[i], rank, he_next, he_vert, pos, out + 9 * i);
}

/* lod.py:177-269.  prm layout: lod.py:286-304. */
static int8_t lod_verdict(uint64_t id, int rank, int64_t depth_limit,
                          const int32_t *he_next, const int32_t *he_vert,
                          const double *pos, const double *prm)
{
    double t[9];
    orc_decode_tri(id, rank, he_next, he_vert, pos, t);
    if (prm[18] > 0.0) { /* planet mode: radial projection, lod.py:185-191 */
        for (int r = 0; r < 3; ++r) {
            double *v = t + 3 * r;
            const double len = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
            const double scale = prm[18] / len;
            v[0] *= scale;
            v[1] *= scale;
            v[2] *= scale;
        }
    }
    if (prm[20] > 0.0) { /* sine displacement demo, lod.py:192-208 */
        const double amp = prm[21], freq = prm[22];
        for (int r = 0; r < 3; ++r) {
            double *v = t + 3 * r;
            const double d = amp * sin(freq * v[0]) * sin(freq * v[1] + 0.5)
                             * sin(freq * v[2] + 1.0);
            const double len = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
            if (len > 0) {
                v[0] += v[0] / len * d;
                v[1] += v[1] / len * d;
                v[2] += v[2] / len * d;
            } else {
                v[2] += d;
            }
        }
    }
    double cx[3], cy[3], cz[3];
    for (int r = 0; r < 3; ++r) { /* camera space, lod.py:210-227 */
        const double x = t[3 * r] - prm[0];
        const double y = t[3 * r + 1] - prm[1];
        const double z = t[3 * r + 2] - prm[2];
        cx[r] = x * prm[3] + y * prm[4] + z * prm[5];
        cy[r] = x * prm[6] + y * prm[7] + z * prm[8];
        cz[r] = x * prm[9] + y * prm[10] + z * prm[11];
    }
    const double f = prm[12], near = prm[13], tx = prm[14], ty = prm[15];
    if (prm[19] > 0.0) { /* conservative frustum cull, lod.py:233-247 */
        int out = 0;
        if (cz[0] < near && cz[1] < near && cz[2] < near)
            out = 1;
        else if (cx[0] + tx * cz[0] < 0 && cx[1] + tx * cz[1] < 0 && cx[2] + tx * cz[2] < 0)
            out = 1;
        else if (tx * cz[0] - cx[0] < 0 && tx * cz[1] - cx[1] < 0 && tx * cz[2] - cx[2] < 0)
            out = 1;
        else if (cy[0] + ty * cz[0] < 0 && cy[1] + ty * cz[1] < 0 && cy[2] + ty * cz[2] < 0)
            out = 1;
        else if (ty * cz[0] - cy[0] < 0 && ty * cz[1] - cy[1] < 0 && ty * cz[2] - cy[2] < 0)
            out = 1;
        if (out)
            return 2;
    }
    double sx[3], sy[3];
    for (int r = 0; r < 3; ++r) { /* near clamp + pinhole, lod.py:249-257 */
        const double zc = cz[r] > near ? cz[r] : near;
        sx[r] = f * cx[r] / zc;
        sy[r] = f * cy[r] / zc;
    }
    const double cross = (sx[1] - sx[0]) * (sy[2] - sy[0]) - (sx[2] - sx[0]) * (sy[1] - sy[0]);
    const double area = 0.5 * fabs(cross);
    if (area > prm[16])
        return depth_of(id, rank) < depth_limit ? 1 : 0;
    if (area < prm[17])
        return 2;
    return 0;
}

void orc_verdict_lod(int8_t *verdicts, const int32_t *cache_live,
                     const uint64_t *ids, int rank, int64_t depth_limit,
                     const int32_t *he_next, const int32_t *he_vert,
                     const double *pos, const double *prm, int64_t start,
                     int64_t end, int threads)
{
#ifdef _OPENMP
#pragma omp parallel for num_threads(threads) schedule(static) if (threads > 1)
#endif
    for (int64_t i = start; i < end; ++i)
        verdicts[i] = lod_verdict(ids[cache_live[i]], rank, depth_limit,
                                  he_next, he_vert, pos, prm);
    (void)threads;
}

/* kernels.py:635-647 */
void orc_verdict_const(int8_t *verdicts, int value, int64_t start, int64_t end)
{
    for (int64_t i = start; i < end; ++i)
        verdicts[i] = (int8_t)value;
}

void orc_verdict_uniform(int8_t *verdicts, const int32_t *cache_live,
                         const uint64_t *ids, int rank, int target_depth,
                         int64_t start, int64_t end)
{
    for (int64_t i = start; i < end; ++i)
        verdicts[i] = depth_of(ids[cache_live[i]], rank) < target_depth ? 1 : 0;
}

/* ------------------------------------------------------------------ */
/* merge configuration helpers                                        */
/* ------------------------------------------------------------------ */

typedef struct {
    int kind; /* 0 none, 1 boundary pair, 2 quad */
    int64_t sib, oth, j4;
} merge_cfg;

/* kernels.py:112-134 */
static merge_cfg merge_config(const orc_pool *p, int64_t s)
{
    merge_cfg c = {0, -1, -1, -1};
    const uint64_t j1 = p->ids[s];
    if (depth_of(j1, p->rank) < 1)
        return c; /* roots never merge */
    const int odd = (int)(j1 & 1);
    const int64_t sib = odd ? p->prevs[s] : p->nexts[s];
    const int64_t oth = odd ? p->nexts[s] : p->prevs[s];
    if (sib == -1 || (p->ids[sib] >> 1) != (j1 >> 1))
        return c;
    if (oth == -1) {
        c.kind = 1;
        c.sib = sib;
        return c;
    }
    if (bit_length_u64(p->ids[oth]) != bit_length_u64(j1))
        return c;
    const int64_t j4 = odd ? p->nexts[oth] : p->prevs[oth];
    if (j4 == -1 || (p->ids[j4] >> 1) != (p->ids[oth] >> 1))
        return c;
    c.kind = 2;
    c.sib = sib;
    c.oth = oth;
    c.j4 = j4;
    return c;
}

static inline int wants_only_merge(uint32_t cmd)
{
    return !(cmd & CMD_SPLIT_MASK) && (cmd & CMD_MERGE);
}

/* kernels.py:137-156 */
static int merge_agreed(const orc_pool *p, int64_t s)
{
    const merge_cfg c = merge_config(p, s);
    if (c.kind == 0)
        return 0;
    if (!wants_only_merge(p->commands[s]) || !wants_only_merge(p->commands[c.sib]))
        return 0;
    if (c.kind == 2 && (!wants_only_merge(p->commands[c.oth])
                        || !wants_only_merge(p->commands[c.j4])))
        return 0;
    return 1;
}

/* kernels.py:159-180 -- the member with the smallest id owns the merge; its
 * reserved[.,0] is the parent of the owner's own pair, reserved[.,1] the
 * parent of the opposite pair of a quad. */
static int32_t merge_parent_slot(const orc_pool *p, int64_t m)
{
    const merge_cfg c = merge_config(p, m);
    int64_t owner = m;
    uint64_t best = p->ids[m];
    if (p->ids[c.sib] < best) {
        best = p->ids[c.sib];
        owner = c.sib;
    }
    if (c.kind == 2) {
        if (p->ids[c.oth] < best) {
            best = p->ids[c.oth];
            owner = c.oth;
        }
        if (p->ids[c.j4] < best) {
            best = p->ids[c.j4];
            owner = c.j4;
        }
    }
    if (c.kind == 1)
        return p->reserved[4 * owner];
    if ((p->ids[m] >> 1) == (p->ids[owner] >> 1))
        return p->reserved[4 * owner];
    return p->reserved[4 * owner + 1];
}

/* kernels.py:183-191 */
static int survives(const orc_pool *p, int64_t x)
{
    const uint32_t cmd = p->commands[x];
    if (cmd & CMD_SPLIT_MASK)
        return 0;
    if ((cmd & CMD_MERGE) && merge_agreed(p, x))
        return 0;
    return 1;
}

/* ------------------------------------------------------------------ */
/* split composition                                                  */
/* ------------------------------------------------------------------ */

/* Reserved-slot index of the child of a bisector split with `mask` that owns
 * (sub)segment `half` of its edge `edge`; -1 when that combination cannot
 * occur.  Equals PIECE_IDX of kernels.py:50-72, derived from the child layout
 * (kernels.py:12-17): the v0-side half of the bisector yields 1 record (2j) or,
 * with the prev edge split, 2 records (4j, 4j+1); the v1-side half follows
 * with 1 (2j+1) or 2 (4j+2, 4j+3) records. */
static int piece_index(unsigned mask, int edge, int half)
{
    if (!(mask & CMD_SPLIT_T))
        return -1;
    const int left_n = (mask & CMD_SPLIT_P) ? 2 : 1;
    const int right_n = (mask & CMD_SPLIT_N) ? 2 : 1;
    const int last = left_n + right_n - 1;
    switch (edge) {
    case E_TWIN:
        if (half == H_V0)
            return 0;
        if (half == H_V1)
            return last;
        return -1;
    case E_NEXT:
        if (right_n == 1)
            return half == H_WHOLE ? left_n : -1;
        if (half == H_V1)
            return last;
        if (half == H_V2)
            return left_n;
        return -1;
    default: /* E_PREV */
        if (left_n == 1)
            return half == H_WHOLE ? 0 : -1;
        if (half == H_V0)
            return 0;
        if (half == H_V2)
            return 1;
        return -1;
    }
}

/* kernels.py:75-100 -- translate (my edge, my half) into the frame of the
 * neighbour that answers through operator t_role. */
static void correspond(int my_side, int my_half, int t_role, int *t_edge, int *t_half)
{
    if (my_side == E_TWIN) {
        if (t_role == E_TWIN) {
            *t_edge = E_TWIN;
            *t_half = my_half == H_V1 ? H_V0 : H_V1;
        } else if (t_role == E_PREV) {
            *t_edge = E_PREV;
            *t_half = my_half == H_V0 ? H_V2 : H_V0;
        } else {
            *t_edge = E_NEXT;
            *t_half = my_half == H_V0 ? H_V1 : H_V2;
        }
    } else if (my_side == E_NEXT) {
        if (t_role == E_PREV) {
            *t_edge = E_PREV;
            *t_half = my_half == H_WHOLE ? H_WHOLE : (my_half == H_V1 ? H_V0 : H_V2);
        } else {
            *t_edge = E_TWIN;
            *t_half = my_half == H_V1 ? H_V0 : H_V1;
        }
    } else {
        if (t_role == E_NEXT) {
            *t_edge = E_NEXT;
            *t_half = my_half == H_WHOLE ? H_WHOLE : (my_half == H_V0 ? H_V1 : H_V2);
        } else {
            *t_edge = E_TWIN;
            *t_half = my_half == H_V0 ? H_V1 : H_V0;
        }
    }
}

/* kernels.py:194-238 -- post-update slot of the record adjacent across
 * (my_side, my_half); `backref` is my own (consumed) slot. */
static int32_t piece_of(const orc_pool *p, int64_t target, int my_side,
                        int my_half, int64_t backref)
{
    if (target == -1)
        return -1;
    const uint32_t cmd = p->commands[target];
    const unsigned smask = cmd & CMD_SPLIT_MASK;
    if (smask) {
        int role = -1;
        if (my_side == E_TWIN) {
            if (p->twins[target] == backref)
                role = E_TWIN;
            else if (p->nexts[target] == backref)
                role = E_NEXT;
            else if (p->prevs[target] == backref)
                role = E_PREV;
        } else if (my_side == E_NEXT) {
            if (p->prevs[target] == backref)
                role = E_PREV;
            else if (p->twins[target] == backref)
                role = E_TWIN;
        } else {
            if (p->nexts[target] == backref)
                role = E_NEXT;
            else if (p->twins[target] == backref)
                role = E_TWIN;
        }
        if (role < 0)
            return -2;
        int t_edge, t_half;
        correspond(my_side, my_half, role, &t_edge, &t_half);
        const int idx = piece_index(smask, t_edge, t_half);
        if (idx < 0)
            return -2;
        return p->reserved[4 * target + idx];
    }
    if ((cmd & CMD_MERGE) && merge_agreed(p, target))
        return merge_parent_slot(p, target);
    return (int32_t)target;
}

/* ------------------------------------------------------------------ */
/* stage kernels                                                      */
/* ------------------------------------------------------------------ */

/* stage 2, kernels.py:244-252 */
void orc_cache_pointers(orc_pool *p, int64_t count, int64_t free_ct,
                        int64_t start, int64_t end, int threads)
{
#ifdef _OPENMP
#pragma omp parallel for num_threads(threads) schedule(static) if (threads > 1)
#endif
    for (int64_t i = start; i < end; ++i) {
        if (i < count)
            p->cache_live[i] = (int32_t)orc_one_to_bit_id(p->nodes, p->capacity, i);
        if (i < free_ct)
            p->cache_free[i] = (int32_t)orc_zero_to_bit_id(p->nodes, p->capacity, i);
    }
    (void)threads;
}

/* Same output as orc_cache_pointers (ascending positions of set / unset bits,
 * kernels.py:244-252) by one linear pass over the leaves.  NOT the reference's
 * algorithm: used only to fast-forward untimed setup frames of the CPU
 * baseline; every timed or parity-checked frame uses the descents above. */
void orc_cache_pointers_scan(orc_pool *p)
{
    const uint32_t *leaves = p->nodes + p->capacity;
    int64_t n1 = 0, n0 = 0;
    for (int64_t s = 0; s < p->capacity; ++s) {
        if (leaves[s])
            p->cache_live[n1++] = (int32_t)s;
        else
            p->cache_free[n0++] = (int32_t)s;
    }
}

/* stage 3, kernels.py:255-259 */
void orc_reset_commands(orc_pool *p, int64_t start, int64_t end)
{
    for (int64_t i = start; i < end; ++i)
        p->commands[p->cache_live[i]] = 0;
}

/* stage 4, kernels.py:262-335.  Serial: admission is order dependent. */
void orc_generate_commands(orc_pool *p, const int8_t *verdicts, int64_t free_ct,
                           int64_t depth_limit, int64_t *stats6, int64_t start,
                           int64_t end)
{
    int64_t oom_splits = 0, oom_merges = 0;
    for (int64_t i = start; i < end; ++i) {
        const int64_t s = p->cache_live[i];
        const int v = verdicts[i];
        if (v == 1) {
            const int d = depth_of(p->ids[s], p->rank);
            if (d >= depth_limit)
                continue;
            const int64_t need = 3 * (int64_t)d + 4;
            if (p->counter[0] + need > free_ct) {
                ++oom_splits; /* add + roll back == untouched counter */
                continue;
            }
            p->counter[0] += need;
            int64_t cur = s;
            for (int hops = 0;;) {
                const uint32_t before = p->commands[cur];
                p->commands[cur] = before | CMD_SPLIT_T;
                if (before & CMD_SPLIT_T)
                    break;
                const int64_t t = p->twins[cur];
                if (t == -1)
                    break;
                if (p->twins[t] == cur) {
                    p->commands[t] |= CMD_SPLIT_T;
                    break;
                }
                if (p->nexts[t] == cur)
                    p->commands[t] |= CMD_SPLIT_N;
                else if (p->prevs[t] == cur)
                    p->commands[t] |= CMD_SPLIT_P;
                else
                    break;
                cur = t;
                if (++hops > 70)
                    break;
            }
        } else if (v == 2) {
            const merge_cfg c = merge_config(p, s);
            if (c.kind == 0)
                continue;
            if (p->counter[0] + 2 > free_ct) {
                ++oom_merges;
                continue;
            }
            p->counter[0] += 2;
            uint32_t bits = CMD_MERGE;
            uint64_t lowest = p->ids[s];
            if (p->ids[c.sib] < lowest)
                lowest = p->ids[c.sib];
            if (c.kind == 2) {
                bits |= CMD_QUAD;
                if (p->ids[c.oth] < lowest)
                    lowest = p->ids[c.oth];
                if (p->ids[c.j4] < lowest)
                    lowest = p->ids[c.j4];
            }
            if (lowest == p->ids[s])
                bits |= CMD_OWNER;
            p->commands[s] |= bits;
        }
    }
    stats6[0] += oom_splits;
    stats6[1] += oom_merges;
}

static inline int split_alloc_count(unsigned smask)
{
    return 2 + ((smask & CMD_SPLIT_N) ? 1 : 0) + ((smask & CMD_SPLIT_P) ? 1 : 0);
}

/* stage 5, kernels.py:338-370 -- windows are popped from the top of the
 * reserved range of the free cache. */
void orc_reserve_blocks(orc_pool *p, int64_t start, int64_t end)
{
    for (int64_t i = start; i < end; ++i) {
        const int64_t s = p->cache_live[i];
        const uint32_t cmd = p->commands[s];
        const unsigned smask = cmd & CMD_SPLIT_MASK;
        int n_alloc;
        if (smask) {
            n_alloc = split_alloc_count(smask);
        } else if ((cmd & CMD_MERGE) && (cmd & CMD_OWNER) && merge_agreed(p, s)) {
            n_alloc = (cmd & CMD_QUAD) ? 2 : 1;
        } else {
            continue;
        }
        p->counter[0] -= n_alloc;
        const int64_t base = p->counter[0];
        for (int k = 0; k < n_alloc; ++k)
            p->reserved[4 * s + k] = p->cache_free[base + k];
    }
}

/* kernels.py:373-461, restated compositionally: the v0-side half produces
 * one record (2j) or two (4j, 4j+1); the v1-side half one (2j+1) or two
 * (4j+2, 4j+3); the seam between the halves is (next/prev) for unsplit halves
 * and twin for a split half's inner record. */
static void fill_split(orc_pool *p, int64_t s)
{
    const uint64_t j = p->ids[s];
    const unsigned smask = p->commands[s] & CMD_SPLIT_MASK;
    const int64_t nb_n = p->nexts[s], nb_p = p->prevs[s], nb_t = p->twins[s];
    const int32_t *r = p->reserved + 4 * s;
    const int left_n = (smask & CMD_SPLIT_P) ? 2 : 1;
    const int right_n = (smask & CMD_SPLIT_N) ? 2 : 1;
    const int32_t left_last = r[left_n - 1];
    const int32_t right_first = r[left_n];

    if (left_n == 1) {
        const int32_t a = r[0];
        p->ids[a] = j << 1;
        p->nexts[a] = right_first;
        p->prevs[a] = piece_of(p, nb_t, E_TWIN, H_V0, s);
        p->twins[a] = piece_of(p, nb_p, E_PREV, H_WHOLE, s);
    } else {
        const int32_t a = r[0], b = r[1];
        p->ids[a] = j << 2;
        p->twins[a] = piece_of(p, nb_t, E_TWIN, H_V0, s);
        p->nexts[a] = b;
        p->prevs[a] = piece_of(p, nb_p, E_PREV, H_V0, s);
        p->ids[b] = (j << 2) + 1;
        p->twins[b] = right_first;
        p->prevs[b] = a;
        p->nexts[b] = piece_of(p, nb_p, E_PREV, H_V2, s);
    }
    if (right_n == 1) {
        const int32_t c = r[left_n];
        p->ids[c] = (j << 1) + 1;
        p->prevs[c] = left_last;
        p->nexts[c] = piece_of(p, nb_t, E_TWIN, H_V1, s);
        p->twins[c] = piece_of(p, nb_n, E_NEXT, H_WHOLE, s);
    } else {
        const int32_t c = r[left_n], d = r[left_n + 1];
        p->ids[c] = (j << 2) + 2;
        p->twins[c] = left_last;
        p->nexts[c] = d;
        p->prevs[c] = piece_of(p, nb_n, E_NEXT, H_V2, s);
        p->ids[d] = (j << 2) + 3;
        p->prevs[d] = c;
        p->twins[d] = piece_of(p, nb_t, E_TWIN, H_V1, s);
        p->nexts[d] = piece_of(p, nb_n, E_NEXT, H_V1, s);
    }
}

/* one sibling pair (even id e, odd id o) collapses into parent slot `par` */
static void fill_merged_parent(orc_pool *p, int64_t e, int64_t o, int32_t par,
                               int32_t twin_slot)
{
    p->ids[par] = p->ids[e] >> 1;
    p->nexts[par] = piece_of(p, p->twins[o], E_NEXT, H_WHOLE, o);
    p->prevs[par] = piece_of(p, p->twins[e], E_PREV, H_WHOLE, e);
    p->twins[par] = twin_slot;
}

/* kernels.py:464-491 (owner only) */
static void fill_merge(orc_pool *p, int64_t s)
{
    const merge_cfg c = merge_config(p, s);
    const int s_even = (p->ids[s] & 1) == 0;
    const int64_t e1 = s_even ? s : c.sib, o1 = s_even ? c.sib : s;
    const int32_t p1 = p->reserved[4 * s];
    if (c.kind == 2) {
        const int32_t p2 = p->reserved[4 * s + 1];
        const int oth_even = (p->ids[c.oth] & 1) == 0;
        const int64_t e2 = oth_even ? c.oth : c.j4, o2 = oth_even ? c.j4 : c.oth;
        /* write order of the reference: p1 (id, next, prev, twin), then p2 */
        fill_merged_parent(p, e1, o1, p1, p2);
        fill_merged_parent(p, e2, o2, p2, p1);
    } else {
        fill_merged_parent(p, e1, o1, p1, -1);
    }
}

/* stage 6, kernels.py:494-511 */
void orc_fill_new_blocks(orc_pool *p, int64_t start, int64_t end)
{
    for (int64_t i = start; i < end; ++i) {
        const int64_t s = p->cache_live[i];
        const uint32_t cmd = p->commands[s];
        if (cmd & CMD_SPLIT_MASK)
            fill_split(p, s);
        else if ((cmd & CMD_MERGE) && (cmd & CMD_OWNER) && merge_agreed(p, s))
            fill_merge(p, s);
    }
}

/* kernels.py:514-530 */
static void redirect_to(orc_pool *p, int64_t target, int64_t old_slot,
                        int32_t new_slot, int first)
{
    int32_t *primary = first == E_PREV ? p->prevs : p->nexts;
    if (primary[target] == old_slot) {
        primary[target] = new_slot;
        return;
    }
    if (p->twins[target] == old_slot)
        p->twins[target] = new_slot;
}

static void redirect_merged_pair(orc_pool *p, int64_t e, int64_t o, int32_t par)
{
    const int64_t n_ext = p->twins[o];
    if (n_ext != -1 && survives(p, n_ext))
        redirect_to(p, n_ext, o, par, E_PREV);
    const int64_t q_ext = p->twins[e];
    if (q_ext != -1 && survives(p, q_ext))
        redirect_to(p, q_ext, e, par, E_NEXT);
}

/* stage 7, kernels.py:533-594 */
void orc_update_neighbors(orc_pool *p, int64_t start, int64_t end)
{
    for (int64_t i = start; i < end; ++i) {
        const int64_t s = p->cache_live[i];
        const uint32_t cmd = p->commands[s];
        const unsigned smask = cmd & CMD_SPLIT_MASK;
        if (smask) {
            const int32_t *r = p->reserved + 4 * s;
            if (!(smask & CMD_SPLIT_N)) {
                const int64_t tgt = p->nexts[s];
                if (tgt != -1 && survives(p, tgt))
                    redirect_to(p, tgt, s, smask == 1 ? r[1] : r[2], E_PREV);
            }
            if (!(smask & CMD_SPLIT_P)) {
                const int64_t tgt = p->prevs[s];
                if (tgt != -1 && survives(p, tgt))
                    redirect_to(p, tgt, s, r[0], E_NEXT);
            }
        } else if ((cmd & CMD_MERGE) && (cmd & CMD_OWNER)) {
            if (!merge_agreed(p, s))
                continue;
            const merge_cfg c = merge_config(p, s);
            const int s_even = (p->ids[s] & 1) == 0;
            redirect_merged_pair(p, s_even ? s : c.sib, s_even ? c.sib : s,
                                 p->reserved[4 * s]);
            if (c.kind == 2) {
                const int oth_even = (p->ids[c.oth] & 1) == 0;
                redirect_merged_pair(p, oth_even ? c.oth : c.j4,
                                     oth_even ? c.j4 : c.oth,
                                     p->reserved[4 * s + 1]);
            }
        }
    }
}

/* stage 8, kernels.py:597-632 */
void orc_update_bitfield(orc_pool *p, int64_t *stats6, int64_t start, int64_t end)
{
    int64_t split_freed = 0, merge_freed = 0, split_alloc = 0, merge_alloc = 0;
    uint32_t *leaves = p->nodes + p->capacity;
    for (int64_t i = start; i < end; ++i) {
        const int64_t s = p->cache_live[i];
        const uint32_t cmd = p->commands[s];
        const unsigned smask = cmd & CMD_SPLIT_MASK;
        if (smask) {
            leaves[s] = 0;
            ++split_freed;
            const int n_alloc = split_alloc_count(smask);
            for (int k = 0; k < n_alloc; ++k)
                leaves[p->reserved[4 * s + k]] = 1;
            split_alloc += n_alloc;
        } else if ((cmd & CMD_MERGE) && merge_agreed(p, s)) {
            leaves[s] = 0;
            ++merge_freed;
            if (cmd & CMD_OWNER) {
                const int n_alloc = (cmd & CMD_QUAD) ? 2 : 1;
                for (int k = 0; k < n_alloc; ++k)
                    leaves[p->reserved[4 * s + k]] = 1;
                merge_alloc += n_alloc;
            }
        }
    }
    stats6[2] += split_freed;
    stats6[3] += merge_freed;
    stats6[4] += split_alloc;
    stats6[5] += merge_alloc;
}

/* ------------------------------------------------------------------ */
/* whole-frame driver                                                 */
/* ------------------------------------------------------------------ */

typedef struct orc_verdict {
    int32_t mode;  /* 0 const, 1 uniform depth, 2 LOD, 3 explicit array */
    int32_t value; /* const verdict / uniform target depth */
    const int8_t *explicit_verdicts; /* mode 3, cache_live order */
    const int32_t *he_next, *he_vert;
    const double *positions;
    double prm[23];
} orc_verdict;

static int64_t now_ns(void)
{
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (int64_t)ts.tv_sec * 1000000000 + ts.tv_nsec;
}

/* pipeline.py:204-322.  stats8 = {oom_splits, oom_merges, split_freed,
 * merge_freed, split_alloc, merge_alloc, live_before, live_after};
 * stage_ns[9] receives per-stage wall time (may be NULL).
 * threads > 1 parallelises only the stages whose result is independent of
 * execution order (2 cache pointers, the verdict source of 4, 9 reduction);
 * the order-dependent stages stay serial so every array stays bit-identical
 * to the reference at threads=1.  verdict_scratch: int8[max(count,1)]. */
int orc_update(orc_pool *p, const orc_verdict *v, int8_t *verdict_scratch,
               int64_t *stats8, int64_t *stage_ns, int threads)
{
    const int fast_setup = threads < 0; /* untimed setup frames, see orc_cache_pointers_scan */
    if (fast_setup)
        threads = -threads;
    const int64_t count = p->nodes[1];
    const int64_t free_ct = p->capacity - count;
    int64_t stats6[6] = {0, 0, 0, 0, 0, 0};
    int64_t t[10];
    if (threads < 1)
        threads = 1;

    t[0] = now_ns();
    p->counter[0] = 0; /* (1) */
    t[1] = now_ns();
    if (fast_setup)
        orc_cache_pointers_scan(p);
    else
        orc_cache_pointers(p, count, free_ct, 0, count > free_ct ? count : free_ct, threads); /* (2) */
    t[2] = now_ns();
    orc_reset_commands(p, 0, count); /* (3) */
    t[3] = now_ns();
    const int8_t *verdicts = verdict_scratch; /* (4) */
    switch (v->mode) {
    case 0:
        orc_verdict_const(verdict_scratch, v->value, 0, count);
        break;
    case 1:
        orc_verdict_uniform(verdict_scratch, p->cache_live, p->ids, p->rank, v->value, 0, count);
        break;
    case 2:
        orc_verdict_lod(verdict_scratch, p->cache_live, p->ids, p->rank, p->max_depth,
                        v->he_next, v->he_vert, v->positions, v->prm, 0, count, threads);
        break;
    case 3:
        verdicts = v->explicit_verdicts;
        break;
    default:
        return 1;
    }
    orc_generate_commands(p, verdicts, free_ct, p->max_depth, stats6, 0, count);
    t[4] = now_ns();
    orc_reserve_blocks(p, 0, count); /* (5) */
    t[5] = now_ns();
    orc_fill_new_blocks(p, 0, count); /* (6) */
    t[6] = now_ns();
    orc_update_neighbors(p, 0, count); /* (7) */
    t[7] = now_ns();
    orc_update_bitfield(p, stats6, 0, count); /* (8) */
    t[8] = now_ns();
    orc_sum_reduce(p->nodes, p->depth, threads); /* (9) */
    t[9] = now_ns();

    for (int k = 0; k < 6; ++k)
        stats8[k] = stats6[k];
    stats8[6] = count;
    stats8[7] = p->nodes[1];
    if (stage_ns)
        for (int k = 0; k < 9; ++k)
            stage_ns[k] = t[k + 1] - t[k];
    /* pipeline.py:319-321 accounting identity */
    if (stats8[7] != count - stats6[2] + stats6[4] - stats6[3] + stats6[5])
        return 2;
    return 0;
}

/* state.py:139-156 -- one root bisector per halfedge at slots [0, H). */
void orc_initialize(orc_pool *p, const int32_t *he_next, const int32_t *he_prev,
                    const int32_t *he_twin, int64_t n_halfedges)
{
    const int64_t N = p->capacity;
    memset(p->ids, 0, sizeof(uint64_t) * N);
    memset(p->commands, 0, sizeof(uint32_t) * N);
    memset(p->nodes, 0, sizeof(uint32_t) * 2 * N);
    for (int64_t i = 0; i < N; ++i) {
        p->nexts[i] = p->prevs[i] = p->twins[i] = -1;
        p->cache_live[i] = p->cache_free[i] = -1;
    }
    for (int64_t i = 0; i < 4 * N; ++i)
        p->reserved[i] = -1;
    p->counter[0] = 0;
    const uint64_t base = (uint64_t)1 << p->rank;
    for (int64_t h = 0; h < n_halfedges; ++h) {
        p->ids[h] = base + (uint64_t)h;
        p->nexts[h] = he_next[h];
        p->prevs[h] = he_prev[h];
        p->twins[h] = he_twin[h];
        p->nodes[N + h] = 1;
    }
    orc_sum_reduce(p->nodes, p->depth, 1);
}

int orc_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
