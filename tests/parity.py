"""Helpers shared by the GPU parity tests: step the CUDA engine and the C
oracle side by side and compare every state array."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
STATE_ARRAYS = ("ids", "nexts", "prevs", "twins", "commands", "reserved",
                "counter", "cache_live", "cache_free")
STAT_NAMES = ("oom_splits", "oom_merges", "split_freed", "merge_freed",
              "split_alloc", "merge_alloc", "live_before", "live_after")


def digest(a: np.ndarray) -> str:
    return hashlib.blake2b(np.ascontiguousarray(a).tobytes(), digest_size=8).hexdigest()


def load_golden(name: str) -> dict:
    with open(os.path.join(GOLDEN, name + ".json")) as fh:
        return json.load(fh)


def stats_words(stats) -> tuple:
    """UpdateStats -> the oracle's stats8 order."""
    return (stats.splits_rejected_oom, stats.merges_rejected_oom,
            stats.splits_applied, stats.merges_applied, stats.split_allocs,
            stats.merge_allocs, stats.live_before, stats.live_after)


def first_diff(a: np.ndarray, b: np.ndarray) -> str:
    a2 = a.reshape(a.shape[0], -1)
    b2 = b.reshape(b.shape[0], -1)
    rows = np.flatnonzero((a2 != b2).any(axis=1))
    r = int(rows[0])
    return f"{rows.size} rows differ, first row {r}: gpu {a2[r].tolist()} oracle {b2[r].tolist()}"


def assert_state_equal(state, op, tag: str, exact_free_cache: bool, stats=None):
    """Every array of the GPU pool equals the oracle's (reference layout)."""
    host = state.to_host()
    for k in STATE_ARRAYS:
        g, o = host[k], getattr(op, k)
        if k == "cache_free" and not exact_free_cache:
            # only the consumed window [T - A, T) is materialised by default
            if stats is None:
                continue
            T = stats.reserved_slots
            A = stats.split_allocs + stats.merge_allocs
            g, o = g[T - A:T], o[T - A:T]
        if not np.array_equal(g, o):
            raise AssertionError(f"{tag}: {k}: {first_diff(g, o)}")
    if not np.array_equal(host["nodes"], op.nodes):
        raise AssertionError(f"{tag}: cbt.nodes: {first_diff(host['nodes'], op.nodes)}")
    return host


def golden_frame_check(host: dict, rec: dict, tag: str, exact_free_cache: bool):
    """Digests committed by oracle/pin_against_reference.py (i.e. the real
    reference's arrays) must match the GPU arrays."""
    for k in STATE_ARRAYS + ("nodes",):
        if k == "cache_free" and not exact_free_cache:
            continue
        assert digest(host[k]) == rec[k], f"{tag}: golden digest mismatch for {k}"
