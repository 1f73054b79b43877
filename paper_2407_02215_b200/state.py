"""The bisector memory pool, resident in HBM.

Drop-in for the reference's ``cbtmesh.state`` (pkg/src/cbtmesh/state.py):
``TriangulationState`` owns the same arrays with the same shapes and initial
values (:32-55), ``initialize`` seeds one root bisector per halfedge at slots
``[0, H)`` (:139-156).  All arrays are torch CUDA tensors (``d_<name>``); the
reference's attribute names (``ids``, ``nexts``, ``commands`` ...) are
read-only HOST snapshots downloaded on demand for inspection and parity dumps.

Memory per slot: 56 B of state as in the reference minus the 8 B/slot heap
(replaced by 1 bit + 1/256 counter) plus 4 B of per-frame scratch.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib, bisector
from .cbt import Cbt, HARD_MAX_DEPTH

# command word layout (state.py:17-25)
SPLIT_T = 1
SPLIT_N = 2
SPLIT_P = 4
SPLIT_MASK = 7
MERGE_REQ = 8
MERGE_QUAD = 16
MERGE_OWNER = 32

WIDE_GRID_LIVE = 150_000  # live bisectors from which the 4-CTAs-per-SM frame kernel is used

_SNAPSHOT_DTYPES = {
    "ids": np.uint64, "nexts": np.int32, "prevs": np.int32, "twins": np.int32,
    "commands": np.uint32, "reserved": np.int32, "counter": np.int64,
    "cache_live": np.int32, "cache_free": np.int32,
}


class CapacityError(RuntimeError):
    """Pool cannot hold the requested configuration."""


class TriangulationState:
    """Pool of bisector records + CBT + pointer caches on one GPU.

    ``exact_free_cache=True`` materialises ``cache_free[0:F)`` every frame like
    the reference does (whole-array parity); the default writes only the
    window of free ranks that the frame consumes.
    ``staged_launches=True`` runs one kernel per pipeline stage instead of the
    persistent cooperative frame kernel (per-stage profiling).
    """

    def __init__(self, mesh, depth: int, device=None,
                 exact_free_cache: bool = False, staged_launches: bool = False,
                 descend_free_ranks: bool = False):
        H = mesh.n_halfedges
        rank = bisector.root_rank(H)
        if depth < rank:
            raise CapacityError(
                f"cbt depth {depth} too small for H={H}: need D >= {rank}")
        if depth > HARD_MAX_DEPTH:
            raise ValueError(f"depth must be <= {HARD_MAX_DEPTH}, got {depth}")
        self.mesh = mesh
        self.depth = depth
        self.rank = rank
        self.max_depth = bisector.max_depth(H)
        self.capacity = cap = 1 << depth
        self.exact_free_cache = bool(exact_free_cache)
        self.staged_launches = bool(staged_launches)
        # testing hook: free ranks by tree descent instead of the window table (the fallback for
        # frames whose allocations span more than 4096 leaf blocks)
        self.descend_free_ranks = bool(descend_free_ranks)
        # cbtm_update also writes the frame's complete stats row at the end of the frame
        # (CBTM_POOL_FINAL_ROW; set by ParallelEngine(profile=True))
        self.complete_rows = False
        self.device = _lib.require_cuda(device)
        L = _lib.load()
        t = _lib.torch()
        dev = self.device
        self.d_ids = t.empty(cap, dtype=t.int64, device=dev)
        self.d_nexts = t.empty(cap, dtype=t.int32, device=dev)
        self.d_prevs = t.empty(cap, dtype=t.int32, device=dev)
        self.d_twins = t.empty(cap, dtype=t.int32, device=dev)
        self.d_commands = t.empty(cap, dtype=t.int32, device=dev)
        self.d_reserved = t.empty((cap, 4), dtype=t.int32, device=dev)
        self.d_cache_live = t.empty(cap, dtype=t.int32, device=dev)
        self.d_cache_free = t.empty(cap, dtype=t.int32, device=dev)
        self.d_counter = t.zeros(1, dtype=t.int64, device=dev)
        self.d_bits = t.zeros(L.cbtm_bitfield_words(depth), dtype=t.int64, device=dev)
        self.d_counters = t.zeros(L.cbtm_counter_words(depth), dtype=t.int32, device=dev)
        # frame counters: pinned host memory mapped into the device's address space -- the frame
        # kernel writes them straight to the host (sequence word last), ParallelEngine.update polls
        # that word instead of copying the stats back and synchronising the stream
        self.d_stats = t.zeros(_lib.STATS_WORDS, dtype=t.int64).pin_memory()
        self._stats_np = self.d_stats.numpy()
        self._stats_host_ptr = int(self.d_stats.data_ptr())
        # mailbox of the lingering frame kernel (ParallelEngine(linger_us=...)): request number in
        # word 0, camera parameters in words 8..30; pinned and device-mapped like the stats
        self._mb = t.zeros(64, dtype=t.int64).pin_memory()
        self._mb_ptr = int(self._mb.data_ptr())
        self._mb_request = 0
        self._mb_listen_until = 0.0
        self._mb_pool = None
        self.d_dispatch = t.zeros(4, dtype=t.int32, device=dev)
        self.d_workspace = t.zeros(L.cbtm_workspace_bytes(depth), dtype=t.uint8, device=dev)
        # mesh operators used by the classifier (uploaded once)
        self.d_he_next = _lib.to_device(np.asarray(mesh.next, np.int32), dev)
        self.d_he_prev = _lib.to_device(np.asarray(mesh.prev, np.int32), dev)
        self.d_he_twin = _lib.to_device(np.asarray(mesh.twin, np.int32), dev)
        self.d_he_vert = _lib.to_device(np.asarray(mesh.vert, np.int32), dev)
        self.d_positions = _lib.to_device(np.asarray(mesh.positions, np.float64), dev)
        self.d_root_tris = t.empty(H * 9, dtype=t.float64, device=dev)
        rc = L.cbtm_root_triangles(_lib.ptr(self.d_he_next), _lib.ptr(self.d_he_vert),
                                   _lib.ptr(self.d_positions), H,
                                   _lib.ptr(self.d_root_tris), self.stream())
        _lib.check(rc, "cbtm_root_triangles")
        self.cbt = Cbt(depth, max_depth=HARD_MAX_DEPTH, device=dev,
                       _bits=self.d_bits, _counters=self.d_counters,
                       _scratch=self.d_workspace)
        self._version = 0
        self._snap: dict[str, tuple[int, np.ndarray]] = {}

    # -- C-ABI view -----------------------------------------------------------
    def stream(self) -> int:
        return _lib.stream_handle(self.device)

    def c_pool(self) -> _lib.CPool:
        """The cbtm_pool view of this state (cached; max_depth and the mode flags
        are plain attributes a caller may change between updates)."""
        # wide grid (4 CTAs per SM) once the pool holds more live bisectors than the narrow grid has
        # threads for two chunks each; decided from the last published live count (host-mapped stats)
        wide = int(self._stats_np[7]) > WIDE_GRID_LIVE
        key = (int(self.max_depth), self.exact_free_cache, self.staged_launches, self.descend_free_ranks, wide,
               self.complete_rows)
        cached = getattr(self, "_c_pool", None)
        if cached is not None and cached[0] == key:
            return cached[1]
        pool = self._build_c_pool(wide)
        self._c_pool = (key, pool)
        return pool

    def c_pool_ref(self):
        """ctypes reference to :meth:`c_pool` (cached with it): the per-frame path passes the
        same object every frame."""
        pool = self.c_pool()
        ref = getattr(self, "_c_pool_ref", None)
        if ref is None or ref[0] is not pool:
            self._c_pool_ref = ref = (pool, C.byref(pool))
        return ref[1]

    def _build_c_pool(self, wide: bool = False) -> _lib.CPool:
        p = _lib.ptr
        return _lib.CPool(
            p(self.d_ids), p(self.d_nexts), p(self.d_prevs), p(self.d_twins),
            p(self.d_commands), p(self.d_reserved), p(self.d_cache_live),
            p(self.d_cache_free), p(self.d_counter), p(self.d_bits),
            p(self.d_counters), p(self.d_stats), p(self.d_dispatch),
            p(self.d_workspace), self.d_workspace.numel(), self.depth,
            self.rank, int(self.max_depth),
            (_lib.POOL_FULL_FREE_CACHE if self.exact_free_cache else 0)
            | (_lib.POOL_STAGED_LAUNCHES if self.staged_launches else 0)
            | (_lib.POOL_DESCEND_FREE_RANKS if self.descend_free_ranks else 0)
            | (_lib.POOL_WIDE_GRID if wide else 0)
            | (_lib.POOL_FINAL_ROW if self.complete_rows else 0))

    def _touched(self) -> None:
        """The device arrays changed: drop host snapshots."""
        self._version += 1
        self.cbt._device_changed(dirty=False)

    def synchronize(self) -> None:
        _lib.torch().cuda.current_stream(self.device).synchronize()

    # -- host snapshots of the device arrays ------------------------------------
    def _snapshot(self, name: str) -> np.ndarray:
        hit = self._snap.get(name)
        if hit is None or hit[0] != self._version:
            arr = _lib.to_host(getattr(self, "d_" + name), _SNAPSHOT_DTYPES[name])
            arr.setflags(write=False)
            self._snap[name] = hit = (self._version, arr)
        return hit[1]

    ids = property(lambda self: self._snapshot("ids"))
    nexts = property(lambda self: self._snapshot("nexts"))
    prevs = property(lambda self: self._snapshot("prevs"))
    twins = property(lambda self: self._snapshot("twins"))
    commands = property(lambda self: self._snapshot("commands"))
    reserved = property(lambda self: self._snapshot("reserved"))
    counter = property(lambda self: self._snapshot("counter"))
    cache_live = property(lambda self: self._snapshot("cache_live"))
    cache_free = property(lambda self: self._snapshot("cache_free"))

    def to_host(self) -> dict:
        """All state arrays in the reference layout (incl. the u32 heap)."""
        out = {k: self._snapshot(k).copy() for k in _SNAPSHOT_DTYPES}
        out["nodes"] = self.cbt._pull().copy()
        return out

    # -- queries (state.py:59-136) ------------------------------------------------
    def count(self) -> int:
        return self.cbt.count()

    def live_slots(self) -> np.ndarray:
        words = _lib.to_host(self.d_bits, np.uint64)
        bits = np.unpackbits(words.view(np.uint8), bitorder="little")
        return np.flatnonzero(bits[:self.capacity]).astype(np.int32)

    def live_ids(self) -> set[int]:
        ids = self.ids
        return {int(ids[s]) for s in self.live_slots()}

    def slot_of(self, bid: int) -> int:
        ids = self.ids
        for s in self.live_slots():
            if int(ids[s]) == bid:
                return int(s)
        raise KeyError(f"bisector id {bid} is not live")

    def depth_of_slot(self, slot: int) -> int:
        return bisector.depth_of(int(self.ids[slot]), self.rank)

    def neighbor_id_map(self) -> dict[int, tuple[int, int, int]]:
        """id -> (next id, prev id, twin id) over the live pool."""
        ids, nx, pv, tw = self.ids, self.nexts, self.prevs, self.twins
        name = lambda q: int(ids[q]) if q >= 0 else -1  # noqa: E731
        return {int(ids[s]): (name(int(nx[s])), name(int(pv[s])), name(int(tw[s])))
                for s in self.live_slots()}

    def decode_slot(self, slot: int) -> np.ndarray:
        return bisector.bisector_vertices(self.mesh, int(self.ids[slot]))

    def triangles(self) -> list[tuple[int, np.ndarray]]:
        ids, tris = self.decode_live()
        return [(int(i), t) for i, t in zip(ids, tris)]

    def decode_live(self) -> tuple[np.ndarray, np.ndarray]:
        """(ids, (n, 3, 3) fp64 vertices) of all live bisectors in ascending
        slot order, decoded on the GPU (reference: state.py:104-113)."""
        d_tris, _ = self.export_live_triangles()
        n = d_tris.shape[0]
        t = _lib.torch()
        d_ids = self.d_ids[self.d_cache_live[:n].to(t.int64)]
        return _lib.to_host(d_ids, np.uint64), _lib.to_host(d_tris)

    def export_live_triangles(self, out=None):
        """Device-resident triangle export (cbtm_export_live_triangles): returns
        (float64[n, 3, 3] CUDA tensor of the live bisectors' vertices in active-list
        order, int32[4] CUDA tensor with the indirect draw arguments).  Nothing but
        the live count crosses to the host (to size the returned view); pass a
        preallocated ``out`` (float64[capacity, 3, 3]) to avoid even the allocation."""
        t = _lib.torch()
        n = self.count()
        if out is None:
            out = t.empty((max(n, 1), 3, 3), dtype=t.float64, device=self.device)
        draw = t.zeros(4, dtype=t.int32, device=self.device)
        pool = self.c_pool()
        rc = _lib.load().cbtm_export_live_triangles(C.byref(pool), _lib.ptr(self.d_root_tris), _lib.ptr(out),
                                                    out.shape[0], _lib.ptr(draw), self.stream())
        _lib.check(rc, "cbtm_export_live_triangles")
        self._version += 1  # cache_live now lists the current state
        return out[:min(n, out.shape[0])], draw

    def validate_device(self) -> dict:
        """Counts of structural violations over the live pool, computed on the
        GPU (cbtm_validate; same checks as :func:`pointer_violations`)."""
        t = _lib.torch()
        out = t.empty(8, dtype=t.int64, device=self.device)
        pool = self.c_pool()
        rc = _lib.load().cbtm_validate(C.byref(pool), self.mesh.n_halfedges,
                                       _lib.ptr(out), self.stream())
        _lib.check(rc, "cbtm_validate")
        w = [int(x) for x in _lib.to_host(out)]
        return {"live": w[0], "bad_ids": w[1], "too_deep": w[2], "dangling": w[3],
                "no_reciprocal": w[4], "depth_gaps": w[5], "first_bad_slot": w[6]}

    def memory_bytes(self) -> int:
        names = ("ids", "nexts", "prevs", "twins", "commands", "reserved",
                 "cache_live", "cache_free", "counter", "bits", "counters",
                 "workspace")
        return sum(getattr(self, "d_" + k).numel() * getattr(self, "d_" + k).element_size()
                   for k in names)

    def clone(self) -> "TriangulationState":
        other = TriangulationState(self.mesh, self.depth, device=self.device,
                                   exact_free_cache=self.exact_free_cache,
                                   staged_launches=self.staged_launches,
                                   descend_free_ranks=self.descend_free_ranks)
        for k in ("ids", "nexts", "prevs", "twins", "commands", "reserved",
                  "cache_live", "cache_free", "counter", "bits", "counters"):
            getattr(other, "d_" + k).copy_(getattr(self, "d_" + k))
        other.max_depth = self.max_depth
        other._touched()
        return other


def initialize(mesh, depth: int, device=None, exact_free_cache: bool = False,
               staged_launches: bool = False, descend_free_ranks: bool = False) -> TriangulationState:
    """One root bisector per halfedge at slots [0, H) (state.py:139-156)."""
    st = TriangulationState(mesh, depth, device=device,
                            exact_free_cache=exact_free_cache,
                            staged_launches=staged_launches,
                            descend_free_ranks=descend_free_ranks)
    pool = st.c_pool()
    rc = _lib.load().cbtm_initialize(
        C.byref(pool), _lib.ptr(st.d_he_next), _lib.ptr(st.d_he_prev),
        _lib.ptr(st.d_he_twin), mesh.n_halfedges, st.stream())
    _lib.check(rc, "cbtm_initialize")
    st._touched()
    return st


# -- structural validators (host-side checkers on downloaded state) --------------
# Same checks as state.py:159-313 of the reference; they run on host snapshots
# and are test/debug tools, not part of the update path.

_BACK_ROLES = {"next": ("prev", "twin"), "prev": ("next", "twin"),
               "twin": ("next", "prev", "twin")}


def pointer_violations(state: TriangulationState) -> list[str]:
    """Reciprocity, dangling-pointer, id-range and depth-gap violations."""
    out = []
    live = set(int(s) for s in state.live_slots())
    ids = state.ids
    arrays = {"next": state.nexts, "prev": state.prevs, "twin": state.twins}
    for s in sorted(live):
        bid = int(ids[s])
        if bid < (1 << state.rank):
            out.append(f"slot {s}: id {bid} below root range")
            continue
        d = bisector.depth_of(bid, state.rank)
        h = bisector.root_halfedge(bid, state.rank)
        if not 0 <= h < state.mesh.n_halfedges:
            out.append(f"slot {s}: id {bid} maps to invalid halfedge {h}")
        if d > state.max_depth:
            out.append(f"slot {s}: id {bid} exceeds depth limit {state.max_depth}")
        for role, arr in arrays.items():
            q = int(arr[s])
            if q == -1:
                continue
            if not 0 <= q < state.capacity or q not in live:
                out.append(f"slot {s} ({role}): dangling pointer to slot {q}")
                continue
            if not any(int(arrays[r][q]) == s for r in _BACK_ROLES[role]):
                out.append(f"slot {s} ({role}) -> {q}: no reciprocal pointer "
                           f"(neighbor id {int(ids[q])})")
            nd = bisector.depth_of(int(ids[q]), state.rank)
            if abs(nd - d) > 1:
                out.append(f"slot {s} ({role}) -> {q}: depth gap {d} vs {nd}")
    return out


_QSCALE = 1e9


def _qpoint(p) -> tuple[int, int, int]:
    return (round(p[0] * _QSCALE), round(p[1] * _QSCALE), round(p[2] * _QSCALE))


def _on_segment(p, a, b) -> bool:
    u, w = b - a, p - a
    lu = float(np.linalg.norm(u))
    cr = float(np.linalg.norm(np.cross(u, w)))
    if cr > 1e-9 * lu * max(lu, float(np.linalg.norm(w))) + 1e-12:
        return False
    s = float(u @ w) / (lu * lu)
    return -1e-9 <= s <= 1 + 1e-9


def conformity_violations(state: TriangulationState) -> list[str]:
    """T-junction check: every decoded edge is shared by exactly two live
    triangles, or lies on a boundary segment of the input mesh."""
    ids, tris = state.decode_live()
    owners: dict[tuple, list[int]] = {}
    for k in range(len(ids)):
        tri = tris[k]
        for i, j in ((0, 1), (1, 2), (2, 0)):
            key = tuple(sorted((_qpoint(tri[i]), _qpoint(tri[j]))))
            owners.setdefault(key, []).append(int(ids[k]))
    mesh = state.mesh
    border = [(mesh.positions[mesh.vert[h]], mesh.positions[mesh.vert[mesh.next[h]]])
              for h in np.flatnonzero(mesh.twin == -1)]
    out = []
    for key, who in owners.items():
        if len(who) == 2:
            continue
        if len(who) > 2:
            out.append(f"edge {key} shared by {len(who)} triangles {who}")
            continue
        a = np.array(key[0], dtype=np.float64) / _QSCALE
        b = np.array(key[1], dtype=np.float64) / _QSCALE
        if not any(_on_segment(a, s0, s1) and _on_segment(b, s0, s1)
                   for s0, s1 in border):
            out.append(f"interior edge {key} owned by single triangle "
                       f"{who[0]} (T-junction)")
    return out


# my vertex -> neighbour's vertex across a pointer, keyed by (my role, the role under which the
# neighbour points back): which corners of the two decoded triangles must coincide.  Twins of equal
# depth share the bisection edge reversed; the mixed pairs are a triangle meeting a neighbour one
# level up or down (reference: _ADJ_CORRESPONDENCE, state.py:271-279; paper Table 1).
_SHARED_CORNERS = {
    ("twin", "twin"): {0: 1, 1: 0},
    ("next", "prev"): {1: 0, 2: 2},
    ("prev", "next"): {2: 2, 0: 1},
    ("next", "twin"): {1: 0, 2: 1},
    ("prev", "twin"): {2: 0, 0: 1},
    ("twin", "next"): {0: 1, 1: 2},
    ("twin", "prev"): {0: 2, 1: 0},
}


def adjacency_geometry_violations(state: TriangulationState) -> list[str]:
    """Every pointer must join geometrically coincident edges with the corner
    correspondence its role pair implies (state.py:282-313 of the reference).
    Host-side checker on the GPU-decoded live triangles."""
    ids, tris = state.decode_live()
    live = state.live_slots()
    where = {int(s): k for k, s in enumerate(live)}
    arrays = {"next": state.nexts, "prev": state.prevs, "twin": state.twins}
    out = []
    for s, k in where.items():
        for role, arr in arrays.items():
            q = int(arr[s])
            if q == -1:
                continue
            back = [r for r in _BACK_ROLES[role] if int(arrays[r][q]) == s]
            if len(back) != 1 or q not in where:
                out.append(f"slot {s} ({role}) -> {q}: back roles {back}")
                continue
            corners = _SHARED_CORNERS.get((role, back[0]))
            if corners is None:
                out.append(f"slot {s} ({role}) -> {q}: illegal role pair {(role, back[0])}")
                continue
            for mine, theirs in corners.items():
                if _qpoint(tris[k][mine]) != _qpoint(tris[where[q]][theirs]):
                    out.append(f"slot {s} ({role}) -> {q}: vertex {mine} != neighbor vertex "
                               f"{theirs} under role pair {(role, back[0])}")
    return out
