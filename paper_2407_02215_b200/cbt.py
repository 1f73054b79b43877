"""Concurrent binary tree over a packed occupancy bitfield, resident in HBM.

Drop-in for the reference's ``cbtmesh.cbt`` (pkg/src/cbtmesh/cbt.py): same
class, methods, attributes and error behaviour (``ValueError`` for a bad depth
or bit value, ``IndexError`` for out-of-range slots/ranks, ``AssertionError``
for ranked queries on a dirty tree).  Storage and all computation live on the
GPU (include/cbtm.h): a 1-bit-per-slot field plus 32-bit counters for nodes
spanning >= 1024 slots; ``sum_reduce``, ``one_to_bit_id`` and
``zero_to_bit_id`` are CUDA kernels.

``nodes`` / ``leaves`` expose the reference's ``uint32[2**(D+1)]`` heap as a
HOST mirror for inspection and for callers that assign leaves in bulk
(``cbt.leaves[:] = ...``): the mirror is refreshed from the device on access
and pushed back before the next device operation.  It is a compatibility
surface, not the hot path -- the update engine never touches it.
"""

from __future__ import annotations

import numpy as np

from . import _lib

MIN_DEPTH = 1
# The reference caps D at 25 (cbt.py:16-18) and its tests require Cbt(26) to
# raise.  The device layout is good to D = 30; pass ``max_depth=30`` (or raise
# this module constant) for the Earth-scale pools.
MAX_DEPTH = 25
HARD_MAX_DEPTH = _lib.MAX_DEPTH_ABI


class Cbt:
    """Sum-reduction tree whose leaves are the pool occupancy bits."""

    def __init__(self, depth: int, max_depth: int | None = None, device=None,
                 _bits=None, _counters=None, _scratch=None):
        limit = MAX_DEPTH if max_depth is None else min(int(max_depth),
                                                        HARD_MAX_DEPTH)
        if not MIN_DEPTH <= depth <= limit:
            raise ValueError(
                f"depth must be in [{MIN_DEPTH}, {limit}], got {depth}")
        self.depth = depth
        self.capacity = 1 << depth
        self.device = _lib.require_cuda(device)
        L = _lib.load()
        t = _lib.torch()
        if _bits is None:
            _bits = t.zeros(L.cbtm_bitfield_words(depth), dtype=t.int64,
                            device=self.device)
            _counters = t.zeros(L.cbtm_counter_words(depth), dtype=t.int32,
                                device=self.device)
            _scratch = t.zeros(max(256, L.cbtm_cbt_workspace_bytes(depth)),
                               dtype=t.uint8, device=self.device)
        self._bits, self._counters, self._scratch = _bits, _counters, _scratch
        self._mirror: np.ndarray | None = None  # host heap, reference layout
        self._shadow: np.ndarray | None = None  # leaves as last synchronised with the device
        self._mirror_stale = True    # device holds newer data than the mirror
        self._mirror_handed_out = False  # a caller holds a writable view of the mirror
        self._dirty = False

    # -- coherence between the host mirror and the device ------------------
    # The reference's ``nodes`` / ``leaves`` are live views of the one heap array: a caller may
    # keep the returned array and write it at any time (``lv = cbt.leaves; lv[a] = 1;
    # cbt.sum_reduce(); lv[b] = 1; cbt.sum_reduce()``).  Once a view has been handed out the
    # mirror therefore stays authoritative for the leaves the caller wrote: ``_shadow`` remembers
    # the leaves as they were when mirror and device last agreed, every device operation first
    # pushes whatever differs from it, and a refresh from the device keeps such writes.
    def _stream(self) -> int:
        return _lib.stream_handle(self.device)

    def _export(self) -> np.ndarray:
        t = _lib.torch()
        dev = t.empty(2 * self.capacity, dtype=t.int32, device=self.device)
        rc = _lib.load().cbtm_export_nodes(
            _lib.ptr(self._bits), _lib.ptr(self._counters), self.depth,
            _lib.ptr(dev), self._stream())
        _lib.check(rc, "cbtm_export_nodes")
        return _lib.to_host(dev, np.uint32)

    def _caller_writes(self) -> np.ndarray | None:
        """Leaf positions the holder of a view changed since the last synchronisation."""
        if self._mirror is None or not self._mirror_handed_out:
            return None
        diff = np.flatnonzero(self._mirror[self.capacity:] != self._shadow)
        return diff if diff.size else None

    def _pull(self) -> np.ndarray:
        """Host mirror of the heap, refreshed from the device if needed."""
        if self._mirror is None or self._mirror_stale:
            fresh = self._export()
            if self._mirror is None:
                self._mirror = fresh.copy()
            else:
                written = self._caller_writes()
                kept = None if written is None else self._mirror[self.capacity + written].copy()
                self._mirror[...] = fresh
                if written is not None:      # writes made through a held view survive the refresh
                    self._shadow = fresh[self.capacity:].copy()
                    self._mirror[self.capacity + written] = kept
                    self._mirror_stale = False
                    self._dirty = True
                    return self._mirror
            self._shadow = self._mirror[self.capacity:].copy()
            self._mirror_stale = False
        return self._mirror

    def _push(self) -> None:
        """Push leaves the caller may have written into the mirror."""
        if self._caller_writes() is None:    # host-only comparison: no device traffic when nothing was written
            return
        if self._mirror_stale:
            self._pull()                     # merges held-view writes into the device's newer leaves
        leaves = np.ascontiguousarray(self._mirror[self.capacity:])
        dev = _lib.to_device(leaves, self.device)
        rc = _lib.load().cbtm_import_leaves(_lib.ptr(self._bits), self.depth,
                                            _lib.ptr(dev), self._stream())
        _lib.check(rc, "cbtm_import_leaves")
        _lib.torch().cuda.current_stream(self.device).synchronize()
        self._shadow = leaves.copy()
        self._mirror_stale = True            # internal nodes of the mirror are out of date until the next pull

    def _device_changed(self, dirty: bool) -> None:
        """Called by the update engine after it rewrote bits/counters."""
        self._mirror_stale = True
        self._dirty = dirty

    # -- leaf access -------------------------------------------------------
    def _check_slot(self, slot: int) -> None:
        if not 0 <= slot < self.capacity:
            raise IndexError(f"slot {slot} out of range [0, {self.capacity})")

    def set_bit(self, slot: int, value: int) -> None:
        self._check_slot(slot)
        if value not in (0, 1):
            raise ValueError(f"bit value must be 0 or 1, got {value}")
        self._pull()[self.capacity + slot] = value
        self._mirror_handed_out = True
        self._dirty = True

    def get_bit(self, slot: int) -> int:
        self._check_slot(slot)
        return int(self._pull()[self.capacity + slot])

    @property
    def nodes(self) -> np.ndarray:
        self._mirror_handed_out = True
        return self._pull()

    @property
    def leaves(self) -> np.ndarray:
        self._mirror_handed_out = True
        return self._pull()[self.capacity:2 * self.capacity]

    # -- reduction and ranked queries ---------------------------------------
    def sum_reduce(self) -> None:
        """Rebuild all internal nodes from the leaves (GPU kernel)."""
        self._push()
        rc = _lib.load().cbtm_sum_reduce(
            _lib.ptr(self._bits), _lib.ptr(self._counters), self.depth,
            _lib.ptr(self._scratch), self._scratch.numel(), self._stream())
        _lib.check(rc, "cbtm_sum_reduce")
        self._mirror_stale = True
        self._dirty = False
        if self._mirror_handed_out:
            self._pull()    # a held ``nodes`` view shows the new sums in place, as the reference's array does

    def count(self) -> int:
        assert not self._dirty, "sum_reduce required before count()"
        return int(self._counters[1].item())

    def _decode(self, ranks, ones: bool) -> np.ndarray:
        self._push()
        ranks = np.ascontiguousarray(ranks, dtype=np.int64).ravel()
        t = _lib.torch()
        d_ranks = _lib.to_device(ranks, self.device)
        d_out = t.empty(ranks.size, dtype=t.int32, device=self.device)
        fn = (_lib.load().cbtm_decode_ones if ones
              else _lib.load().cbtm_decode_zeros)
        rc = fn(_lib.ptr(self._bits), _lib.ptr(self._counters), self.depth,
                _lib.ptr(d_ranks), ranks.size, _lib.ptr(d_out), self._stream())
        _lib.check(rc, "cbtm_decode")
        return _lib.to_host(d_out)

    def one_to_bit_id(self, rank: int) -> int:
        """Slot of the (rank+1)-th set bit in ascending slot order."""
        assert not self._dirty, "sum_reduce required before ranked queries"
        ones = self.count()
        if not 0 <= rank < ones:
            raise IndexError(f"rank {rank} out of range [0, {ones})")
        return int(self._decode([rank], True)[0])

    def zero_to_bit_id(self, rank: int) -> int:
        """Slot of the (rank+1)-th unset bit in ascending slot order."""
        assert not self._dirty, "sum_reduce required before ranked queries"
        zeros = self.capacity - self.count()
        if not 0 <= rank < zeros:
            raise IndexError(f"rank {rank} out of range [0, {zeros})")
        return int(self._decode([rank], False)[0])

    def one_to_bit_ids(self, ranks) -> np.ndarray:
        assert not self._dirty, "sum_reduce required before ranked queries"
        return self._decode(ranks, True)

    def zero_to_bit_ids(self, ranks) -> np.ndarray:
        assert not self._dirty, "sum_reduce required before ranked queries"
        return self._decode(ranks, False)

    def index(self, want_free: bool = True):
        """(live slots, free slots) in ascending order: the cache-pointer pass
        (pipeline stage 2) as one compaction kernel."""
        assert not self._dirty, "sum_reduce required before ranked queries"
        self._push()
        t = _lib.torch()
        n = self.count()
        live = t.empty(max(n, 1), dtype=t.int32, device=self.device)
        free = (t.empty(max(self.capacity - n, 1), dtype=t.int32,
                        device=self.device) if want_free else None)
        rc = _lib.load().cbtm_index(_lib.ptr(self._bits),
                                    _lib.ptr(self._counters), self.depth,
                                    _lib.ptr(live), _lib.ptr(free), 0,
                                    self._stream())
        _lib.check(rc, "cbtm_index")
        live_h = _lib.to_host(live)[:n]
        free_h = _lib.to_host(free)[:self.capacity - n] if want_free else None
        return live_h, free_h

    # -- diagnostics ---------------------------------------------------------
    def dump(self) -> str:
        nodes = self._pull()
        rows = []
        for level in range(self.depth + 1):
            lo = 1 << level
            rows.append(f"level {level:2d}: "
                        + " ".join(str(int(v)) for v in nodes[lo:2 * lo]))
        return "\n".join(rows)


# -- raw heap-array entry points (cbt.py:153-170) -------------------------------
# The reference exposes these on numpy heaps; here they round-trip through the
# device: leaves are uploaded, the kernels run, results are written back.

def _cbt_from_heap(nodes: np.ndarray, depth: int) -> Cbt:
    cap = 1 << depth
    c = Cbt(depth, max_depth=HARD_MAX_DEPTH)
    c._mirror = np.zeros(2 * cap, np.uint32)
    c._mirror[cap:] = nodes[cap:2 * cap]
    c._shadow = np.zeros(cap, np.uint32)   # the fresh device field is empty
    c._mirror_stale = False
    c._mirror_handed_out = True
    c.sum_reduce()
    return c


def sum_reduce_array(nodes: np.ndarray, depth: int) -> None:
    """In-place sum reduction of a reference-layout heap array."""
    nodes[...] = _cbt_from_heap(nodes, depth)._pull()


def nb_one_to_bit_ids(nodes, capacity, ranks, out, start, end) -> None:
    c = _cbt_from_heap(nodes, int(capacity).bit_length() - 1)
    out[start:end] = c.one_to_bit_ids(np.asarray(ranks)[start:end])


def nb_zero_to_bit_ids(nodes, capacity, ranks, out, start, end) -> None:
    c = _cbt_from_heap(nodes, int(capacity).bit_length() - 1)
    out[start:end] = c.zero_to_bit_ids(np.asarray(ranks)[start:end])


def nb_one_to_bit_id(nodes, capacity, rank) -> int:
    out = np.zeros(1, np.int64)
    nb_one_to_bit_ids(nodes, capacity, np.array([rank]), out, 0, 1)
    return int(out[0])


def nb_zero_to_bit_id(nodes, capacity, rank) -> int:
    out = np.zeros(1, np.int64)
    nb_zero_to_bit_ids(nodes, capacity, np.array([rank]), out, 0, 1)
    return int(out[0])
