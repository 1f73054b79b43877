"""GPU, BASELINE full sizes: where the oracle cannot follow array for array in
seconds, parity goes through size-independent properties.

* Config 3 (Earth sweep, 2^26 pool): without reservation pressure the id-level
  evolution does not depend on the pool size, so per-frame counters, the final
  live-id set and the id-level neighbour map must equal the oracle's run on a
  2^22 pool (the oracle itself is pinned to the reference at that size, see
  tests/golden/earth_sweep_d22_short.json); plus the structural validators.
* Config 4 (CBT, 2^28 leaves): root == popcount, compacted lists are exactly the
  sorted positions of set / unset bits (checked on device), ranked decode of
  sampled ranks agrees with the lists.
"""

import numpy as np
import pytest

from paper_2407_02215_b200 import _lib, workloads
from paper_2407_02215_b200.cbt import Cbt
from paper_2407_02215_b200.pipeline import ParallelEngine
from paper_2407_02215_b200.state import initialize, pointer_violations

pytestmark = pytest.mark.gpu


def test_config3_earth_sweep_2_26_matches_small_pool_oracle():
    import oracle
    from oracle import OraclePool, OracleVerdict
    seq = workloads.earth_sweep(depth=26, frames=64)
    prms = seq.params()
    st = initialize(seq.mesh, 26)
    with ParallelEngine() as eng:
        rows = eng.run_lod_sequence(st, prms)
    assert all(r.splits_rejected_oom == 0 and r.merges_rejected_oom == 0 and r.poison == 0 for r in rows)
    assert max(r.live_after for r in rows) > 60000

    op = OraclePool(seq.mesh, 22)
    threads = oracle.max_threads()
    for f in range(seq.n_frames):
        s, _ = op.update(OracleVerdict.lod(seq.mesh, prms[f]), threads=threads, fast_setup=True)
        r = rows[f]
        assert (r.splits_rejected_oom, r.merges_rejected_oom, r.splits_applied, r.merges_applied,
                r.split_allocs, r.merge_allocs, r.live_before, r.live_after) == tuple(int(x) for x in s), f

    # final state, id level
    live = st.live_slots()
    ids = st.ids
    o_live = op.live_slots()
    assert set(int(ids[s]) for s in live) == set(int(op.ids[s]) for s in o_live)
    gpu_map = st.neighbor_id_map()

    def name(q):
        return int(op.ids[q]) if q >= 0 else -1
    ora_map = {int(op.ids[s]): (name(int(op.nexts[s])), name(int(op.prevs[s])), name(int(op.twins[s])))
               for s in o_live}
    assert gpu_map == ora_map
    assert pointer_violations(st) == []
    dev = st.validate_device()
    assert dev["live"] == len(live)
    assert (dev["bad_ids"], dev["too_deep"], dev["dangling"], dev["no_reciprocal"], dev["depth_gaps"]) == (0,) * 5


def test_config4_cbt_2_28_properties():
    import torch
    depth = 28
    n = 1 << depth
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(28010)
    c = Cbt(depth, max_depth=30)
    # occupancy ~ 0.25: AND of two random words
    words = (torch.randint(-2 ** 63, 2 ** 63 - 1, (n // 64,), dtype=torch.int64, device=dev, generator=gen)
             & torch.randint(-2 ** 63, 2 ** 63 - 1, (n // 64,), dtype=torch.int64, device=dev, generator=gen))
    c._bits.copy_(words)
    c._device_changed(dirty=True)
    c.sum_reduce()
    # root == popcount of the field (byte LUT on device)
    lut = torch.tensor([bin(i).count("1") for i in range(256)], dtype=torch.int64, device=dev)
    popcount = int(lut[words.view(torch.uint8).to(torch.int64)].sum().item())
    assert c.count() == popcount
    L = _lib.load()
    live = torch.empty(popcount, dtype=torch.int32, device=dev)
    free = torch.empty(n - popcount, dtype=torch.int32, device=dev)
    rc = L.cbtm_index(_lib.ptr(c._bits), _lib.ptr(c._counters), depth, _lib.ptr(live), _lib.ptr(free), 0,
                      _lib.stream_handle(dev))
    _lib.check(rc, "cbtm_index")
    # sortedness + membership: every listed live slot has its bit set, every free slot not
    assert bool((live[1:] > live[:-1]).all()) and bool((free[1:] > free[:-1]).all())

    def bit_of(slots):
        s = slots.to(torch.int64)
        return (words[s >> 6] >> (s & 63)) & 1
    assert bool((bit_of(live) == 1).all()) and bool((bit_of(free) == 0).all())
    assert int(live[0]) >= 0 and int(live[-1]) < n and int(free[-1]) < n
    # ranked decode agrees with the lists on sampled ranks
    ranks = torch.randint(0, popcount, (1 << 16,), device=dev)
    assert np.array_equal(c.one_to_bit_ids(ranks.cpu().numpy()), live[ranks].cpu().numpy())
    zr = torch.randint(0, n - popcount, (1 << 16,), device=dev)
    assert np.array_equal(c.zero_to_bit_ids(zr.cpu().numpy()), free[zr].cpu().numpy())


def test_maximum_pool_2_30_equals_2_24_slot_for_slot():
    """The largest pool the ABI allows (2^30 slots: 56 GB of records + 12 GB of scratch, int32 slot
    indices and uint32 counters at their limits).  Without reservation pressure every decision of a
    frame -- admission, free ranks, slot placement -- is independent of how many untouched free slots
    lie behind the ones in use, so the run must equal the same sequence on a 2^24 pool slot for slot:
    counters, active list, records at the live slots, and the common prefix of the CBT."""
    import torch
    free_bytes, _ = torch.cuda.mem_get_info()
    if free_bytes < 80 * 2 ** 30:
        pytest.skip("needs ~70 GB of device memory")
    seq = workloads.earth_sweep(depth=30, frames=24)
    prms = seq.params()[:24]
    big = initialize(seq.mesh, 30)
    small = initialize(seq.mesh, 24)
    with ParallelEngine() as eng:
        rows_big = eng.run_lod_sequence(big, prms)
        rows_small = eng.run_lod_sequence(small, prms)
    assert [r.csv_row(no_timing=True) for r in rows_big] == [r.csv_row(no_timing=True) for r in rows_small]
    assert all(r.poison == 0 for r in rows_big) and rows_big[-1].live_after > 20000
    n = rows_big[-1].live_before          # the active list both pools hold is the last frame's
    assert torch.equal(big.d_cache_live[:n], small.d_cache_live[:n])
    cap = small.capacity
    for k in ("ids", "nexts", "prevs", "twins", "commands", "reserved"):
        assert torch.equal(getattr(big, "d_" + k)[:cap], getattr(small, "d_" + k)[:cap]), k
    assert torch.equal(big.d_bits[:cap // 64], small.d_bits)
    assert not bool(big.d_bits[cap // 64:].any())                    # nothing beyond the small pool was touched
    assert int(big.d_counters[1].item()) == int(small.d_counters[1].item()) == rows_big[-1].live_after
    dev = big.validate_device()
    assert (dev["bad_ids"], dev["too_deep"], dev["dangling"], dev["no_reciprocal"], dev["depth_gaps"]) == (0,) * 5
    del big
    torch.cuda.empty_cache()
