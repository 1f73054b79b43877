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


def test_index_both_lists_on_nearly_empty_and_nearly_full_blocks():
    """k_index_all: lists of a block with 0..7 entries (no 16-byte aligned interior for the bulk store: head and
    tail entries go by scalar stores), next to full, empty and half-full blocks, at every alignment."""
    depth = 20
    n = 1 << depth
    rng = np.random.default_rng(2024)
    leaves = np.zeros(n, np.uint32)
    for b in range(n // 1024):
        kind = b % 6
        blk = leaves[b * 1024:(b + 1) * 1024]
        if kind == 0:
            blk[rng.choice(1024, rng.integers(0, 8), replace=False)] = 1          # 0..7 live slots
        elif kind == 1:
            blk[:] = 1
            blk[rng.choice(1024, rng.integers(0, 8), replace=False)] = 0          # 0..7 free slots
        elif kind == 2:
            blk[:] = rng.random(1024) < 0.5
        elif kind == 3:
            blk[:] = 1
        elif kind == 5:
            blk[rng.integers(0, 1024)] = 1
    c = make(depth, leaves)
    live, free = c.index()
    assert np.array_equal(live, np.flatnonzero(leaves))
    assert np.array_equal(free, np.flatnonzero(leaves == 0))


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


# -- the two ways k_sum_reduce builds the levels above the tile roots ----------------

def _heap_on_device(bits, counters, depth):
    import torch
    from paper_2407_02215_b200 import _lib
    nodes = torch.empty(2 << depth, dtype=torch.int32, device=bits.device)
    _lib.check(_lib.load().cbtm_export_nodes(_lib.ptr(bits), _lib.ptr(counters), depth, _lib.ptr(nodes),
                                             _lib.stream_handle(bits.device)), "cbtm_export_nodes")
    return nodes


def _consistent(nodes, depth):
    """every internal node == sum of its children, on the device"""
    n = 1 << depth
    inner = nodes[1:n].to(int)
    kids = nodes[2:2 * n].to(int).view(-1, 2).sum(dim=1)
    return bool((inner == kids).all())


@pytest.mark.parametrize("depth", [10, 17, 18, 19, 21, 24, 26, 28])
def test_sum_reduce_rebuild_and_delta_paths_agree_with_the_oracle(depth):
    """k_sum_reduce: an unstamped tree (fresh, zeroed or garbage counters) is rebuilt by the last CTA
    and stamped; a stamped tree takes per-tile atomic deltas -- after arbitrary changes of the
    bitfield, repeatedly, from one tile to 2048.  Every level against the oracle's heap up to 2^24,
    against the sum-of-children property and the popcount above."""
    import torch
    from paper_2407_02215_b200 import _lib
    L = _lib.load()
    dev = torch.device("cuda", 0)
    n = 1 << depth
    gen = torch.Generator(device=dev)
    gen.manual_seed(4242 + depth)
    words = max(16, n // 64)
    lut = torch.tensor([bin(i).count("1") for i in range(256)], dtype=torch.int64, device=dev)

    def popcount(b):
        return int(sum(int(lut[b[lo:lo + (1 << 22)].view(torch.uint8).to(torch.int64)].sum())
                       for lo in range(0, b.numel(), 1 << 22)))

    def random_bits(density_and):
        b = torch.randint(-2 ** 63, 2 ** 63 - 1, (words,), dtype=torch.int64, device=dev, generator=gen)
        for _ in range(density_and):
            b &= torch.randint(-2 ** 63, 2 ** 63 - 1, (words,), dtype=torch.int64, device=dev, generator=gen)
        if n < 64 * words:       # tiny pools: only the low n bits exist
            b[n // 64:] = 0
        return b

    ws = torch.zeros(1024, dtype=torch.uint8, device=dev)
    stream = _lib.stream_handle(dev)
    bits = random_bits(0)
    counters = torch.randint(0, 2 ** 31 - 1, (L.cbtm_counter_words(depth),), dtype=torch.int32, device=dev, generator=gen)
    counters[0] = 12345                     # garbage everywhere, no stamp

    def reduce_and_check(tag):
        _lib.check(L.cbtm_sum_reduce(_lib.ptr(bits), _lib.ptr(counters), depth, _lib.ptr(ws), 1024, stream), tag)
        nodes = _heap_on_device(bits, counters, depth)
        assert int(nodes[1]) == popcount(bits), tag
        assert _consistent(nodes, depth), tag
        assert int(ws.view(torch.int32)[0]) == 0 and int(ws.view(torch.int32)[1]) == 0, tag   # the rebuild ticket is left at zero
        if depth <= 24:
            import oracle
            host = np.zeros(2 * n, np.uint32)
            host[n:] = np.unpackbits(bits.cpu().numpy().view(np.uint8), bitorder="little")[:n]
            oracle.sum_reduce_nodes(host, depth, threads=8)
            assert np.array_equal(nodes.cpu().numpy().view(np.uint32), host), tag
        return nodes

    reduce_and_check("rebuild from garbage counters")
    stamp = int(counters[0])
    assert stamp != 12345 and stamp != 0
    for round_, density in enumerate((0, 3, 1, 0)):
        bits.copy_(random_bits(density))                      # a completely different bitfield
        if round_ == 2:
            bits[:bits.numel() // 3] = 0                      # a long empty prefix
        reduce_and_check(f"delta round {round_}")
        assert int(counters[0]) == stamp
    bits[::5] ^= 0x0F0F                                       # sparse changes
    reduce_and_check("delta after sparse flips")
    counters.zero_()                                          # a caller reset the counters: rebuild again
    reduce_and_check("rebuild from zeroed counters")
    assert int(counters[0]) == stamp


def _counter_tree_consistent(bits, counters, depth):
    """leaf counters == popcount of their 1024-slot block, every counter above == sum of its children
    (the packed tree itself, without expanding it to the reference's heap)"""
    import torch
    lc = depth - 10
    lut = torch.tensor([bin(i).count("1") for i in range(256)], dtype=torch.int32, device=bits.device)
    leaf = counters[1 << lc:2 << lc]
    by = bits.view(torch.uint8)
    step = 1 << 26                                            # bytes per chunk
    for lo in range(0, by.numel(), step):
        want = lut[by[lo:lo + step].to(torch.int64)].view(-1, 128).sum(dim=1, dtype=torch.int32)
        if not torch.equal(want, leaf[lo // 128:lo // 128 + want.numel()]):
            return False
    inner = counters[1:1 << lc]
    kids = counters[2:2 << lc].view(-1, 2).sum(dim=1, dtype=torch.int32)
    return bool(torch.equal(inner, kids))


def test_sum_reduce_at_the_largest_pool_and_on_a_16_byte_aligned_bitfield():
    """2^30 slots (the ABI's limit): 8192 tiles, the rebuild path takes its first two levels through L2
    because the shared-memory heap holds 2048 roots; then the delta path.  And a bitfield that is
    16- but not 32-byte aligned (the ABI's contract) goes through the 128-bit-load variant."""
    import torch
    from paper_2407_02215_b200 import _lib
    L = _lib.load()
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(99)
    ws = torch.zeros(1024, dtype=torch.uint8, device=dev)
    stream = _lib.stream_handle(dev)
    for depth, shift_words in ((30, 0), (22, 2), (30, 2)):
        words = (1 << depth) // 64
        store = torch.randint(-2 ** 63, 2 ** 63 - 1, (words + 4,), dtype=torch.int64, device=dev, generator=gen)
        if store.data_ptr() % 32:
            store = store[2:]                                 # (torch allocations are 512-byte aligned anyway)
        bits = store[shift_words:shift_words + words]
        assert bits.data_ptr() % 32 == (16 if shift_words else 0)
        counters = torch.randint(0, 2 ** 31 - 1, (L.cbtm_counter_words(depth),), dtype=torch.int32, device=dev,
                                 generator=gen)
        counters[0] = 777
        _lib.check(L.cbtm_sum_reduce(_lib.ptr(bits), _lib.ptr(counters), depth, _lib.ptr(ws), 1024, stream), "rebuild")
        assert _counter_tree_consistent(bits, counters, depth), (depth, shift_words, "rebuild")
        assert int(ws.view(torch.int32)[0]) == 0
        bits[::3] ^= 0x00FF00FF00FF                           # change a third of the words, everywhere
        bits[: words // 5] = -1
        _lib.check(L.cbtm_sum_reduce(_lib.ptr(bits), _lib.ptr(counters), depth, _lib.ptr(ws), 1024, stream), "delta")
        assert _counter_tree_consistent(bits, counters, depth), (depth, shift_words, "delta")
        if shift_words:
            # ranked decode: the 16-byte aligned bitfield takes the word-by-word leaf search, an aligned
            # copy the sector-by-sector one (256-bit loads) -- same slots
            twin = bits.clone()
            assert twin.data_ptr() % 32 == 0
            ones = int(counters[1])
            for fn, limit in ((L.cbtm_decode_ones, ones), (L.cbtm_decode_zeros, (1 << depth) - ones)):
                ranks = torch.randint(0, limit, (1 << 16,), dtype=torch.int64, device=dev, generator=gen)
                ranks[:2] = torch.tensor([0, limit - 1], device=dev)
                a = torch.empty(ranks.numel(), dtype=torch.int32, device=dev)
                b = torch.empty_like(a)
                _lib.check(fn(_lib.ptr(bits), _lib.ptr(counters), depth, _lib.ptr(ranks), ranks.numel(), _lib.ptr(a), stream), "decode")
                _lib.check(fn(_lib.ptr(twin), _lib.ptr(counters), depth, _lib.ptr(ranks), ranks.numel(), _lib.ptr(b), stream), "decode")
                assert torch.equal(a, b) and int(a.min()) >= 0
            del twin
        del store, bits, counters
        torch.cuda.empty_cache()


def test_sum_reduce_rejects_misaligned_counters():
    import torch
    from paper_2407_02215_b200 import _lib
    L = _lib.load()
    dev = torch.device("cuda", 0)
    bits = torch.zeros(1 << 10, dtype=torch.int64, device=dev)
    counters = torch.zeros(L.cbtm_counter_words(16) + 4, dtype=torch.int32, device=dev)
    ws = torch.zeros(1024, dtype=torch.uint8, device=dev)
    out = torch.zeros(8, dtype=torch.int32, device=dev)
    bad = counters.data_ptr() + 4
    assert L.cbtm_sum_reduce(bits.data_ptr(), bad, 16, ws.data_ptr(), 1024, 0) == 6           # CBTM_E_ALIGN
    assert L.cbtm_decode_ones(bits.data_ptr(), bad, 16, None, 8, out.data_ptr(), 0) == 6
    assert L.cbtm_index(bits.data_ptr(), bad, 16, out.data_ptr(), None, None, 0) == 6
