"""ctypes/numpy front end of oracle/cbtm_oracle.c (reference-layout arrays).

TEST INFRASTRUCTURE ONLY -- see the header of cbtm_oracle.c.  ``OraclePool``
holds the same arrays as the reference's ``TriangulationState``
(pkg/src/cbtmesh/state.py:32-55) and ``OraclePool.update`` is the restatement
of ``ParallelEngine(threads=1).update`` (pkg/src/cbtmesh/pipeline.py:204-322).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (idempotent)."""
    src = os.path.join(_HERE, "cbtm_oracle.c")
    if force or not os.path.exists(_SO) or (
            os.path.getmtime(_SO) < os.path.getmtime(src)):
        base = ["make", "-s", "-C", _HERE, "-B", "liboracle.so"]
        if subprocess.call(base, stderr=subprocess.DEVNULL) != 0:
            # no usable libgomp: build the serial oracle (threads arg ignored)
            subprocess.check_call(base + ["OMP="])
    return _SO


class _CPool(C.Structure):
    _fields_ = [
        ("ids", C.c_void_p), ("nexts", C.c_void_p), ("prevs", C.c_void_p),
        ("twins", C.c_void_p), ("commands", C.c_void_p),
        ("reserved", C.c_void_p), ("nodes", C.c_void_p),
        ("counter", C.c_void_p), ("cache_live", C.c_void_p),
        ("cache_free", C.c_void_p), ("capacity", C.c_int64),
        ("depth", C.c_int32), ("rank", C.c_int32), ("max_depth", C.c_int32),
        ("pad_", C.c_int32),
    ]


class _CVerdict(C.Structure):
    _fields_ = [
        ("mode", C.c_int32), ("value", C.c_int32),
        ("explicit_verdicts", C.c_void_p), ("he_next", C.c_void_p),
        ("he_vert", C.c_void_p), ("positions", C.c_void_p),
        ("prm", C.c_double * 23),
    ]


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        L.orc_sum_reduce.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.orc_one_to_bit_ids.argtypes = [C.c_void_p, C.c_int64, C.c_void_p,
                                         C.c_void_p, C.c_int64]
        L.orc_zero_to_bit_ids.argtypes = L.orc_one_to_bit_ids.argtypes
        L.orc_decode_tris.argtypes = [C.c_void_p, C.c_int64, C.c_int,
                                      C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p]
        L.orc_update.argtypes = [C.POINTER(_CPool), C.POINTER(_CVerdict),
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        L.orc_update.restype = C.c_int
        L.orc_initialize.argtypes = [C.POINTER(_CPool), C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_int64]
        L.orc_cache_pointers.argtypes = [C.POINTER(_CPool), C.c_int64,
                                         C.c_int64, C.c_int64, C.c_int64,
                                         C.c_int]
        L.orc_verdict_lod.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_int, C.c_int64, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_int64, C.c_int64, C.c_int]
        L.orc_max_threads.restype = C.c_int
        _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().orc_max_threads())


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def sum_reduce_nodes(nodes: np.ndarray, depth: int, threads: int = 1) -> None:
    assert nodes.dtype == np.uint32 and nodes.size == 2 << depth
    lib().orc_sum_reduce(_ptr(nodes), depth, threads)


def decode_ones(nodes: np.ndarray, capacity: int, ranks) -> np.ndarray:
    ranks = np.ascontiguousarray(ranks, dtype=np.int64)
    out = np.empty_like(ranks)
    lib().orc_one_to_bit_ids(_ptr(nodes), capacity, _ptr(ranks), _ptr(out),
                             ranks.size)
    return out


def decode_zeros(nodes: np.ndarray, capacity: int, ranks) -> np.ndarray:
    ranks = np.ascontiguousarray(ranks, dtype=np.int64)
    out = np.empty_like(ranks)
    lib().orc_zero_to_bit_ids(_ptr(nodes), capacity, _ptr(ranks), _ptr(out),
                              ranks.size)
    return out


def decode_tris(ids, rank: int, he_next, he_vert, positions) -> np.ndarray:
    ids = np.ascontiguousarray(ids, dtype=np.uint64)
    out = np.empty((ids.size, 3, 3), dtype=np.float64)
    lib().orc_decode_tris(_ptr(ids), ids.size, rank,
                          _ptr(np.ascontiguousarray(he_next, dtype=np.int32)),
                          _ptr(np.ascontiguousarray(he_vert, dtype=np.int32)),
                          _ptr(np.ascontiguousarray(positions, dtype=np.float64)),
                          _ptr(out))
    return out


class OracleVerdict:
    """Verdict source description: const / uniform / lod / explicit."""

    def __init__(self, mode: int, value: int = 0, explicit=None, mesh=None,
                 prm=None):
        self.mode = mode
        self.value = value
        self.explicit = (None if explicit is None else
                         np.ascontiguousarray(explicit, dtype=np.int8))
        self.mesh = mesh
        self.prm = None if prm is None else np.asarray(prm, dtype=np.float64)

    @classmethod
    def const(cls, v):
        return cls(0, int(v))

    @classmethod
    def uniform(cls, target_depth):
        return cls(1, int(target_depth))

    @classmethod
    def lod(cls, mesh, prm):
        return cls(2, mesh=mesh, prm=prm)

    @classmethod
    def explicit_array(cls, verdicts):
        return cls(3, explicit=verdicts)


ARRAYS = ("ids", "nexts", "prevs", "twins", "commands", "reserved", "nodes",
          "counter", "cache_live", "cache_free")


class OraclePool:
    """Reference-layout bisector pool driven by the C oracle."""

    def __init__(self, mesh, depth: int):
        H = mesh.n_halfedges
        self.rank = max(1, (H - 1).bit_length())
        if depth < self.rank:
            raise RuntimeError(f"cbt depth {depth} too small for H={H}")
        self.mesh = mesh
        self.depth = depth
        self.capacity = N = 1 << depth
        self.max_depth = 63 - self.rank
        self.ids = np.zeros(N, np.uint64)
        self.nexts = np.full(N, -1, np.int32)
        self.prevs = np.full(N, -1, np.int32)
        self.twins = np.full(N, -1, np.int32)
        self.commands = np.zeros(N, np.uint32)
        self.reserved = np.full((N, 4), -1, np.int32)
        self.nodes = np.zeros(2 * N, np.uint32)
        self.counter = np.zeros(1, np.int64)
        self.cache_live = np.full(N, -1, np.int32)
        self.cache_free = np.full(N, -1, np.int32)
        self._scratch = np.zeros(N, np.int8)
        self._he_next = np.ascontiguousarray(mesh.next, np.int32)
        self._he_prev = np.ascontiguousarray(mesh.prev, np.int32)
        self._he_twin = np.ascontiguousarray(mesh.twin, np.int32)
        self._he_vert = np.ascontiguousarray(mesh.vert, np.int32)
        self._pos = np.ascontiguousarray(mesh.positions, np.float64)
        lib().orc_initialize(C.byref(self._cpool()), _ptr(self._he_next),
                             _ptr(self._he_prev), _ptr(self._he_twin), H)

    def _cpool(self) -> _CPool:
        return _CPool(_ptr(self.ids), _ptr(self.nexts), _ptr(self.prevs),
                      _ptr(self.twins), _ptr(self.commands),
                      _ptr(self.reserved), _ptr(self.nodes),
                      _ptr(self.counter), _ptr(self.cache_live),
                      _ptr(self.cache_free), self.capacity, self.depth,
                      self.rank, self.max_depth, 0)

    def count(self) -> int:
        return int(self.nodes[1])

    @property
    def leaves(self) -> np.ndarray:
        return self.nodes[self.capacity:]

    def live_slots(self) -> np.ndarray:
        return np.flatnonzero(self.leaves).astype(np.int32)

    def update(self, verdict: OracleVerdict, threads: int = 1,
               fast_setup: bool = False):
        """One frame.  Returns (stats8, stage_ns9) as int64 arrays.
        fast_setup=True replaces the stage-2 descents by a linear scan with the
        same output (untimed fast-forwarding only, never for parity/timing)."""
        if fast_setup:
            threads = -max(1, threads)
        cv = _CVerdict()
        cv.mode, cv.value = verdict.mode, verdict.value
        keep = []
        if verdict.mode == 3:
            assert verdict.explicit.size >= self.count()
            cv.explicit_verdicts = _ptr(verdict.explicit)
        if verdict.mode == 2:
            cv.he_next = _ptr(self._he_next)
            cv.he_vert = _ptr(self._he_vert)
            cv.positions = _ptr(self._pos)
            for k in range(23):
                cv.prm[k] = float(verdict.prm[k])
        stats = np.zeros(8, np.int64)
        stage = np.zeros(9, np.int64)
        rc = lib().orc_update(C.byref(self._cpool()), C.byref(cv),
                              _ptr(self._scratch), _ptr(stats), _ptr(stage),
                              threads)
        del keep
        if rc != 0:
            raise AssertionError(f"oracle update failed with status {rc}")
        return stats, stage

    def live_ids_in_cache_order(self) -> np.ndarray:
        """ids[cache_live[:n]] after a cache-pointer pass on the current CBT."""
        n = self.count()
        lib().orc_cache_pointers(C.byref(self._cpool()), n,
                                 self.capacity - n, 0,
                                 max(n, self.capacity - n), 1)
        return self.ids[self.cache_live[:n]]

    def snapshot(self) -> dict:
        return {k: getattr(self, k).copy() for k in ARRAYS}
