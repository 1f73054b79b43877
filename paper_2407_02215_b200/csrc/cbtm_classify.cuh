// cbtm_classify.cuh -- fp64 bisector decode and the screen-space LOD verdict.
//
// Reference semantics: nb_decode_tri (pkg/src/cbtmesh/bisector.py:100-183) and
// _k_verdict_lod (pkg/src/cbtmesh/lod.py:177-269).  The reference's compiled
// code uses separate IEEE multiplies and adds (no FMA); every product and sum
// here goes through __dmul_rn / __dadd_rn / __dsub_rn / __ddiv_rn / __dsqrt_rn,
// which the compiler never contracts, in the reference's operation order, so
// verdicts are bit-identical.
#pragma once

#include "cbtm_common.cuh"

namespace cbtm {

// Vertices (row-major v0, v1, v2) of bisector `id`.  `root_tris` holds the
// root bisector of every halfedge (cbtm_root_triangles).  The subdivision
// matrix row (a, b, c) becomes (c/2, b + c/2, a) for an odd path bit and
// (a + c/2, c/2, b) for an even one, lowest id bit first.
__device__ __forceinline__ void decode_triangle(uint64_t id, int rank,
                                                const double *__restrict__ root_tris,
                                                double tri[9])
{
    const int d = depth_of(id, rank);
    const uint64_t root = id >> d;
    double m[3][3] = {{1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}};
    uint64_t h = id;
    for (int step = 0; step < d; ++step) {
        const bool odd = h & 1;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const double a = m[r][0], b = m[r][1], c = m[r][2];
            const double hc = __dmul_rn(0.5, c);
            // one add per row, on the entry the path bit selects (the fp64 pipe is what bounds the
            // classify phase: 2 instead of 3 DP operations per row and level)
            const double y = __dadd_rn(odd ? b : a, hc);
            m[r][0] = odd ? hc : y;
            m[r][1] = odd ? y : hc;
            m[r][2] = odd ? a : b;
        }
        h >>= 1;
    }
    const double *p = root_tris + 9 * (size_t)(root - ((uint64_t)1 << rank));
    double q[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) q[k] = __ldg(&p[k]);
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            tri[3 * r + k] = __dadd_rn(__dadd_rn(__dmul_rn(m[r][0], q[k]), __dmul_rn(m[r][1], q[3 + k])),
                                       __dmul_rn(m[r][2], q[6 + k]));
}

__device__ __forceinline__ double dot3_rn(double x, double y, double z, double a, double b, double c)
{
    return __dadd_rn(__dadd_rn(__dmul_rn(x, a), __dmul_rn(y, b)), __dmul_rn(z, c));
}

// 0 keep / 1 split / 2 merge from the decoded triangle t (modified in place).  prm layout: include/cbtm.h
// (LodDecide._prm).
__device__ __forceinline__ int lod_verdict_of_triangle(double *t, uint64_t id, int rank, int depth_limit,
                                                       const double *__restrict__ prm)
{
    const double radius = prm[18];
    if (radius > 0.0) { // radial projection onto the planet, lod.py:185-191
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            double *v = t + 3 * r;
            const double len = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(v[0], v[0]), __dmul_rn(v[1], v[1])),
                                                    __dmul_rn(v[2], v[2])));
            const double scale = __ddiv_rn(radius, len);
            v[0] = __dmul_rn(v[0], scale);
            v[1] = __dmul_rn(v[1], scale);
            v[2] = __dmul_rn(v[2], scale);
        }
    }
    if (prm[20] > 0.0) {
        // sine displacement demo (lod.py:192-208).  NOT bit-exact with the
        // reference: CUDA's sin() and the host libm differ in the last ulp.
        const double amp = prm[21], freq = prm[22];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            double *v = t + 3 * r;
            const double d = __dmul_rn(__dmul_rn(__dmul_rn(amp, sin(__dmul_rn(freq, v[0]))),
                                                 sin(__dadd_rn(__dmul_rn(freq, v[1]), 0.5))),
                                       sin(__dadd_rn(__dmul_rn(freq, v[2]), 1.0)));
            const double len = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(v[0], v[0]), __dmul_rn(v[1], v[1])),
                                                    __dmul_rn(v[2], v[2])));
            if (len > 0.0) {
                v[0] = __dadd_rn(v[0], __dmul_rn(__ddiv_rn(v[0], len), d));
                v[1] = __dadd_rn(v[1], __dmul_rn(__ddiv_rn(v[1], len), d));
                v[2] = __dadd_rn(v[2], __dmul_rn(__ddiv_rn(v[2], len), d));
            } else {
                v[2] = __dadd_rn(v[2], d);
            }
        }
    }
    double cx[3], cy[3], cz[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) { // camera space, lod.py:210-227
        const double x = __dsub_rn(t[3 * r], prm[0]);
        const double y = __dsub_rn(t[3 * r + 1], prm[1]);
        const double z = __dsub_rn(t[3 * r + 2], prm[2]);
        cx[r] = dot3_rn(x, y, z, prm[3], prm[4], prm[5]);
        cy[r] = dot3_rn(x, y, z, prm[6], prm[7], prm[8]);
        cz[r] = dot3_rn(x, y, z, prm[9], prm[10], prm[11]);
    }
    const double f = prm[12], near = prm[13], tx = prm[14], ty = prm[15];
    if (prm[19] > 0.0) { // conservative frustum cull, lod.py:233-247
        bool behind = true, left = true, right = true, below = true, above = true;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const double txz = __dmul_rn(tx, cz[r]), tyz = __dmul_rn(ty, cz[r]);
            behind = behind && (cz[r] < near);
            left = left && (__dadd_rn(cx[r], txz) < 0.0);
            right = right && (__dsub_rn(txz, cx[r]) < 0.0);
            below = below && (__dadd_rn(cy[r], tyz) < 0.0);
            above = above && (__dsub_rn(tyz, cy[r]) < 0.0);
        }
        if (behind || left || right || below || above) return 2;
    }
    double sx[3], sy[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) { // near clamp + pinhole projection, lod.py:249-257
        const double zc = cz[r] > near ? cz[r] : near;
        sx[r] = __ddiv_rn(__dmul_rn(f, cx[r]), zc);
        sy[r] = __ddiv_rn(__dmul_rn(f, cy[r]), zc);
    }
    const double cross = __dsub_rn(__dmul_rn(__dsub_rn(sx[1], sx[0]), __dsub_rn(sy[2], sy[0])),
                                   __dmul_rn(__dsub_rn(sx[2], sx[0]), __dsub_rn(sy[1], sy[0])));
    const double area = __dmul_rn(0.5, fabs(cross));
    if (area > prm[16]) return depth_of(id, rank) < depth_limit ? 1 : 0;
    if (area < prm[17]) return 2;
    return 0;
}

__device__ __forceinline__ int lod_verdict(uint64_t id, int rank, int depth_limit,
                                           const double *__restrict__ root_tris,
                                           const double *__restrict__ prm)
{
    double t[9];
    decode_triangle(id, rank, root_tris, t);
    return lod_verdict_of_triangle(t, id, rank, depth_limit, prm);
}

// bisector.py:154-173 -- root bisector of each halfedge: v0, v1 and the mean
// of the face's vertices accumulated in `next` order starting at the halfedge.
__global__ void k_root_triangles(const int32_t *__restrict__ he_next,
                                 const int32_t *__restrict__ he_vert,
                                 const double *__restrict__ pos, int n_halfedges,
                                 double *__restrict__ out)
{
    const int he = blockIdx.x * blockDim.x + threadIdx.x;
    if (he >= n_halfedges) return;
    const int nx = he_next[he];
    const double *p0 = pos + 3 * (size_t)he_vert[he];
    const double *p1 = pos + 3 * (size_t)he_vert[nx];
    double s0 = p0[0], s1 = p0[1], s2 = p0[2];
    int n = 1;
    for (int w = nx; w != he && n <= n_halfedges; w = he_next[w]) {
        const double *pw = pos + 3 * (size_t)he_vert[w];
        s0 = __dadd_rn(s0, pw[0]);
        s1 = __dadd_rn(s1, pw[1]);
        s2 = __dadd_rn(s2, pw[2]);
        ++n;
    }
    double *o = out + 9 * (size_t)he;
    o[0] = p0[0]; o[1] = p0[1]; o[2] = p0[2];
    o[3] = p1[0]; o[4] = p1[1]; o[5] = p1[2];
    o[6] = __ddiv_rn(s0, (double)n);
    o[7] = __ddiv_rn(s1, (double)n);
    o[8] = __ddiv_rn(s2, (double)n);
}

__global__ void __launch_bounds__(256)
k_decode_triangles(const uint64_t *__restrict__ ids, int64_t K, int rank,
                   const double *__restrict__ root_tris, double *__restrict__ out)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < K;
         i += (int64_t)gridDim.x * blockDim.x) {
        double t[9];
        decode_triangle(ids[i], rank, root_tris, t);
#pragma unroll
        for (int k = 0; k < 9; ++k) out[9 * i + k] = t[k];
    }
}

// The step right after the update in the paper's frame: all live
// bisectors decoded into a vertex buffer, in active-list order, with the indirect draw
// arguments written on the device -- n is read from the CBT root, nothing goes through
// the host.  cache_live must be current (cbtm_index, or any update followed by an index).
__global__ void __launch_bounds__(256)
k_export_live_triangles(const uint64_t *__restrict__ ids, const int32_t *__restrict__ cache_live,
                        const uint32_t *__restrict__ counters, int rank, const double *__restrict__ root_tris,
                        double *__restrict__ out, uint64_t out_capacity, uint32_t *__restrict__ draw_args)
{
    // (launched with programmatic stream serialization behind the index pass: set up while that one drains)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint32_t n = counters[1];
    const uint64_t m = n < out_capacity ? n : out_capacity;
    if (blockIdx.x == 0 && threadIdx.x == 0 && draw_args) {
        draw_args[0] = 3u * (uint32_t)m; // vertex count
        draw_args[1] = 1;               // instance count
        draw_args[2] = 0;               // first vertex
        draw_args[3] = 0;               // first instance
    }
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        double t[9];
        decode_triangle(ids[cache_live[i]], rank, root_tris, t);
#pragma unroll
        for (int k = 0; k < 9; ++k) out[9 * i + k] = t[k];
    }
}

} // namespace cbtm
