"""GPU parity of the CBT kernels (sum reduction, ranked decode, indexation,
heap import/export) against the C oracle and the reference's golden vectors,
plus the drop-in behaviour of the ``Cbt`` class (reference tests/test_cbt.py)."""

import json
import os

import numpy as np
import pytest

from paper_2407_02215_b200 import cbt as cbt_mod
from paper_2407_02215_b200.cbt import Cbt
from tests.parity import GOLDEN, digest

pytestmark = pytest.mark.gpu


def make(depth, leaves):
    c = Cbt(depth, max_depth=30)
    c.leaves[:] = leaves
    c._dirty = True
    c.sum_reduce()
    return c


def oracle_nodes(depth, leaves):
    import oracle
    n = 1 << depth
    nodes = np.zeros(2 * n, np.uint32)
    nodes[n:] = leaves
    oracle.sum_reduce_nodes(nodes, depth, threads=8)
    return nodes


@pytest.mark.parametrize("depth", list(range(1, 15)) + [17, 18, 20, 21])
def test_reduce_decode_index_match_oracle(depth):
    import oracle
    n = 1 << depth
    rng = np.random.default_rng(77 + depth)
    for occ in (0.0, 0.02, 0.5, 0.98, 1.0):
        leaves = (rng.random(n) < occ).astype(np.uint32)
        c = make(depth, leaves)
        ref = oracle_nodes(depth, leaves)
        assert np.array_equal(c.nodes, ref), (depth, occ)
        ones = int(ref[1])
        assert c.count() == ones
        # ranked decode on random ranks (and out-of-range -> -1)
        for is_one, total in ((True, ones), (False, n - ones)):
            k = min(total, 2048)
            ranks = np.sort(rng.choice(total, k, replace=False)) if total else np.zeros(0, np.int64)
            want = (oracle.decode_ones if is_one else oracle.decode_zeros)(ref, n, ranks)
            got = (c.one_to_bit_ids if is_one else c.zero_to_bit_ids)(ranks)
            assert np.array_equal(got, want), (depth, occ, is_one)
            assert (c.one_to_bit_ids if is_one else c.zero_to_bit_ids)([total, -1]).tolist() == [-1, -1]
        # indexation == ascending positions of set / unset bits == all ranks decoded
        live, free = c.index()
        assert np.array_equal(live, np.flatnonzero(leaves))
        assert np.array_equal(free, np.flatnonzero(leaves == 0))
        live_only, none = c.index(want_free=False)
        assert none is None and np.array_equal(live_only, live)


def test_golden_cbt_vectors():
    with open(os.path.join(GOLDEN, "cbt_vectors.json")) as fh:
        vectors = json.load(fh)
    for v in vectors:
        depth = v["depth"]
        n = 1 << depth
        packed = np.frombuffer(bytes.fromhex(v["leaves"]), dtype=np.uint8)
        leaves = np.unpackbits(packed, bitorder="little")[:n].astype(np.uint32)
        c = make(depth, leaves)
        assert digest(c.nodes) == v["nodes_digest"]
        assert c.one_to_bit_ids(v["ranks1"]).tolist() == v["slots1"]
        assert c.zero_to_bit_ids(v["ranks0"]).tolist() == v["slots0"]


def test_pool_like_and_large_pools():
    """Prefix-occupied pools (how a real pool looks) at 2^24."""
    import oracle
    from paper_2407_02215_b200.workloads import microbench_leaves
    depth = 24
    for occ in (0.1, 0.9):
        leaves = microbench_leaves(depth, occ, pool_like=True).astype(np.uint32)
        c = make(depth, leaves)
        ref = oracle_nodes(depth, leaves)
        assert np.array_equal(c.nodes, ref)
        live, free = c.index()
        assert np.array_equal(live, np.flatnonzero(leaves))
        assert np.array_equal(free, np.flatnonzero(leaves == 0))
        ranks = np.random.default_rng(3).integers(0, int(ref[1]), 1 << 16)
        assert np.array_equal(c.one_to_bit_ids(ranks), oracle.decode_ones(ref, 1 << depth, ranks))


# -- drop-in behaviour of the class (reference tests/test_cbt.py) ---------------

def test_depth_bounds():
    for bad in (0, -1, 26):
        with pytest.raises(ValueError):
            Cbt(bad)
    assert Cbt(1).capacity == 2
    assert Cbt(25).capacity == 1 << 25
    assert Cbt(26, max_depth=30).capacity == 1 << 26
    with pytest.raises(ValueError):
        Cbt(31, max_depth=31)


def test_worked_example_and_errors():
    c = Cbt(4)
    for s in (0, 3, 10):
        c.set_bit(s, 1)
    with pytest.raises(AssertionError):
        c.count()
    with pytest.raises(AssertionError):
        c.one_to_bit_id(0)
    c.sum_reduce()
    assert c.count() == 3
    assert [c.one_to_bit_id(r) for r in range(3)] == [0, 3, 10]
    assert c.zero_to_bit_id(0) == 1
    assert c.get_bit(3) == 1 and c.get_bit(4) == 0
    with pytest.raises(IndexError):
        c.one_to_bit_id(3)
    with pytest.raises(IndexError):
        c.zero_to_bit_id(13)
    with pytest.raises(IndexError):
        c.set_bit(16, 1)
    with pytest.raises(ValueError):
        c.set_bit(0, 2)
    c.set_bit(3, 0)
    c.sum_reduce()
    assert [c.one_to_bit_id(r) for r in range(2)] == [0, 10]


def test_dump_format_and_raw_heap_functions():
    c = Cbt(2)
    c.set_bit(1, 1)
    c.set_bit(2, 1)
    c.sum_reduce()
    assert c.dump() == "level  0: 2\nlevel  1: 1 1\nlevel  2: 0 1 1 0"
    rng = np.random.default_rng(5)
    depth = 9
    n = 1 << depth
    nodes = np.zeros(2 * n, np.uint32)
    nodes[n:] = rng.random(n) < 0.3
    want = oracle_nodes(depth, nodes[n:])
    cbt_mod.sum_reduce_array(nodes, depth)
    assert np.array_equal(nodes, want)
    ranks = np.arange(int(nodes[1]), dtype=np.int64)
    out = np.zeros(ranks.size, np.int64)
    cbt_mod.nb_one_to_bit_ids(nodes, n, ranks, out, 0, ranks.size)
    assert np.array_equal(out, np.flatnonzero(nodes[n:]))
    assert cbt_mod.nb_zero_to_bit_id(nodes, n, 0) == int(np.flatnonzero(nodes[n:] == 0)[0])


def test_held_leaf_view_stays_live_like_the_reference():
    """The reference's ``leaves`` / ``nodes`` are live views of the heap: a caller may keep
    the array and write it again after a reduction (cbt.py:30-57).  The host mirror must
    not drop such writes, nor may a refresh from the device overwrite them."""
    c = Cbt(6)
    lv = c.leaves
    lv[3] = 1
    c.sum_reduce()
    lv[40] = 1                      # written through the view held across a device operation
    c.sum_reduce()
    assert c.count() == 2 and c.one_to_bit_id(1) == 40
    nd = c.nodes                    # held heap view: internal nodes refresh in place
    assert nd[1] == 2 and nd[64 + 3] == 1 and nd[64 + 40] == 1
    lv[41] = 1
    assert c.get_bit(41) == 1       # a read in between must not lose the write either
    c.sum_reduce()
    assert c.count() == 3 and nd[1] == 3 and c.zero_to_bit_id(0) == 0
    assert [int(x) for x in c.one_to_bit_ids([0, 1, 2])] == [3, 40, 41]
    lv[3] = 0
    c.sum_reduce()
    assert c.count() == 2 and c.one_to_bit_id(0) == 40


def test_held_view_of_a_pool_cbt_survives_an_engine_update():
    """Writes made through a held view after the engine changed the device bitfield are
    merged into the newer device state, not replaced by it and not replacing it."""
    from paper_2407_02215_b200 import halfedge
    from paper_2407_02215_b200.pipeline import ParallelEngine, SplitAll
    from paper_2407_02215_b200.state import initialize
    st = initialize(halfedge.single_triangle(), 5)
    lv = st.cbt.leaves
    assert int(lv.sum()) == 3
    with ParallelEngine() as eng:
        s = eng.update(st, SplitAll())
    live = s.live_after
    free = int(np.flatnonzero(st.cbt.nodes[32:] == 0)[-1])
    lv[free] = 1                    # held view, written after the update
    st.cbt.sum_reduce()
    assert st.cbt.count() == live + 1 and st.cbt.get_bit(free) == 1
    assert int(lv.sum()) == live + 1   # the view shows the device's leaves plus the write
