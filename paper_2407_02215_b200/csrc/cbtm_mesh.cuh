// cbtm_mesh.cuh -- halfedge mesh construction from polygon loops on the device
// (reference: halfedge.from_polygons, pkg/src/cbtmesh/halfedge.py:158-212).
//
// The reference builds python dictionaries keyed by directed and undirected
// vertex pairs: fine for the 4..240 halfedges of the built-in meshes, seconds for
// the paper's 21 399-halfedge asset and beyond.  Here the same result comes from
// one sort: every halfedge gets the key (min(u,v) << 32 | max(u,v)), the pairs
// (key, halfedge) are radix-sorted (stable, so equal keys stay in halfedge order),
// and a run of equal keys is one undirected edge --
//   run of 1: boundary edge, twin = -1;  run of 2 with opposite directions: twins;
//   run of 2 with the same direction: inconsistent winding;  longer: non-manifold.
// The reference numbers edges by the rank of their key in sorted order
// (halfedge.py:203-209): an exclusive scan over the run starts.
#pragma once

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "cbtm_common.cuh"

namespace cbtm {

// status words written by the ingest (int64)
enum {
    MESH_DEGENERATE_FACES = 0, // faces with fewer than 3 distinct vertices
    MESH_BAD_VERTICES = 1,     // corners referencing a vertex outside [0, V)
    MESH_ZERO_EDGES = 2,       // corners whose next corner is the same vertex
    MESH_NONMANIFOLD = 3,      // undirected edges with more than two halfedges
    MESH_WINDING = 4,          // undirected edges whose two halfedges share a direction
    MESH_FIRST_FACE = 5,       // lowest offending face of the first three classes (or -1)
    MESH_FIRST_EDGE = 6,       // lowest offending edge key (min << 32 | max) of the last two (or -1)
    MESH_EDGES = 7             // number of undirected edges
};

struct MeshScratch {
    uint64_t *keys_a, *keys_b;
    int32_t *vals_a, *vals_b;
    int32_t *starts, *ranks;
    void *cub_tmp;
    size_t cub_bytes;
};

inline size_t mesh_cub_bytes(int64_t H)
{
    size_t sort_bytes = 0, scan_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, (int)H);
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const int32_t *)nullptr, (int32_t *)nullptr, (int)H);
    return sort_bytes > scan_bytes ? sort_bytes : scan_bytes;
}

inline size_t carve_mesh_scratch(void *base, int64_t H, MeshScratch *out)
{
    size_t off = 0;
    auto take = [&](size_t bytes) {
        void *p = base ? (char *)base + off : nullptr;
        off = (off + bytes + 255) / 256 * 256;
        return p;
    };
    MeshScratch m;
    m.keys_a = (uint64_t *)take(8 * (size_t)H);
    m.keys_b = (uint64_t *)take(8 * (size_t)H);
    m.vals_a = (int32_t *)take(4 * (size_t)H);
    m.vals_b = (int32_t *)take(4 * (size_t)H);
    m.starts = (int32_t *)take(4 * (size_t)H);
    m.ranks = (int32_t *)take(4 * (size_t)H);
    m.cub_bytes = mesh_cub_bytes(H);
    m.cub_tmp = take(m.cub_bytes);
    if (out) *out = m;
    return off;
}

// one thread per face: next / prev / vert / face of its corners, the sort keys,
// and the per-face checks of halfedge.py:171-181
__global__ void __launch_bounds__(256)
k_mesh_faces(const int32_t *__restrict__ face_offsets, const int32_t *__restrict__ face_verts, int32_t n_faces,
             int32_t n_vertices, int32_t *__restrict__ he_next, int32_t *__restrict__ he_prev,
             int32_t *__restrict__ he_vert, int32_t *__restrict__ he_face, uint64_t *__restrict__ keys,
             int32_t *__restrict__ vals, unsigned long long *status)
{
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n_faces; f += (int64_t)gridDim.x * blockDim.x) {
        const int32_t first = face_offsets[f], n = face_offsets[f + 1] - first;
        bool bad_vertex = false, zero_edge = false;
        int distinct = 0;
        for (int i = 0; i < n; ++i) {
            const int32_t u = face_verts[first + i], v = face_verts[first + (i + 1 == n ? 0 : i + 1)];
            const int32_t h = first + i;
            he_vert[h] = u;
            he_next[h] = first + (i + 1 == n ? 0 : i + 1);
            he_prev[h] = first + (i == 0 ? n - 1 : i - 1);
            he_face[h] = (int32_t)f;
            bad_vertex |= u < 0 || u >= n_vertices;
            zero_edge |= u == v;
            const uint32_t lo = (uint32_t)(u < v ? u : v), hi = (uint32_t)(u < v ? v : u);
            keys[h] = ((uint64_t)lo << 32) | hi;
            vals[h] = h;
            bool seen = false; // distinct vertices of the loop (loops are short)
            for (int j = 0; j < i; ++j) seen |= face_verts[first + j] == u;
            distinct += !seen;
        }
        const bool degenerate = distinct < 3;
        if (degenerate) atomicAdd(&status[MESH_DEGENERATE_FACES], 1ull);
        if (bad_vertex) atomicAdd(&status[MESH_BAD_VERTICES], 1ull);
        if (zero_edge) atomicAdd(&status[MESH_ZERO_EDGES], 1ull);
        if (degenerate || bad_vertex || zero_edge) atomicMin(&status[MESH_FIRST_FACE], (unsigned long long)f);
    }
}

// sorted position i starts a run of equal keys?
__global__ void __launch_bounds__(256)
k_mesh_run_starts(const uint64_t *__restrict__ keys, int64_t H, int32_t *__restrict__ starts)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < H; i += (int64_t)gridDim.x * blockDim.x)
        starts[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// ranks = exclusive scan of starts, so the run containing position i is edge ranks[i] + starts[i] - 1
__global__ void __launch_bounds__(256)
k_mesh_twins(const uint64_t *__restrict__ keys, const int32_t *__restrict__ vals, const int32_t *__restrict__ starts,
             const int32_t *__restrict__ ranks, int64_t H, const int32_t *__restrict__ he_vert,
             int32_t *__restrict__ he_twin, int32_t *__restrict__ he_edge, unsigned long long *status)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < H; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t key = keys[i];
        const int32_t h = vals[i];
        he_edge[h] = ranks[i] + starts[i] - 1;
        if (i == H - 1) status[MESH_EDGES] = (unsigned long long)(ranks[i] + starts[i]);
        const bool same_prev = i > 0 && keys[i - 1] == key;
        const bool same_next = i + 1 < H && keys[i + 1] == key;
        int32_t twin = -1;
        if (same_prev != same_next) { // an end of a run of at least two
            const int64_t j = same_prev ? i - 1 : i + 1;
            const bool longer = same_prev ? (i >= 2 && keys[i - 2] == key) : (i + 2 < H && keys[i + 2] == key);
            if (!longer) { // run of exactly two
                twin = vals[j];
                if (he_vert[twin] == he_vert[h] && !same_prev) { // same direction (count the edge once)
                    atomicAdd(&status[MESH_WINDING], 1ull);
                    atomicMin(&status[MESH_FIRST_EDGE], (unsigned long long)key);
                }
            }
        }
        if (same_prev && same_next && !(i >= 2 && keys[i - 2] == key)) { // second position of a run of >= 3
            atomicAdd(&status[MESH_NONMANIFOLD], 1ull);
            atomicMin(&status[MESH_FIRST_EDGE], (unsigned long long)key);
        }
        he_twin[h] = twin;
    }
}

} // namespace cbtm
