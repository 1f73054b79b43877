"""CPU: libcbtm.so loads without a GPU, exports every symbol include/cbtm.h
declares, and its size queries / argument checks behave.  No compute calls."""

import ctypes as C
import os
import re

import pytest

from paper_2407_02215_b200 import _lib
from paper_2407_02215_b200 import build as cuda_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "cbtm.h")) as fh:
        text = fh.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cbtm_[a-z_0-9]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    cuda_build.build()
    return _lib.load()


def test_header_and_binding_agree(lib):
    names = declared_symbols()
    assert len(names) >= 19
    assert set(names) == set(_lib.SIGNATURES), "python binding out of sync with include/cbtm.h"
    raw = C.CDLL(_lib.LIB_PATH)
    for name in names:
        assert hasattr(raw, name), f"libcbtm.so does not export {name}"


def test_size_queries(lib):
    assert lib.cbtm_abi_version() == 2
    assert lib.cbtm_bitfield_words(4) == 16          # one 128-byte line minimum
    assert lib.cbtm_bitfield_words(26) == (1 << 26) // 64
    assert lib.cbtm_counter_words(10) == 2
    assert lib.cbtm_counter_words(26) == 2 << 16     # heap over 2^16 leaf blocks
    assert lib.cbtm_workspace_bytes(0) == 0 and lib.cbtm_workspace_bytes(31) == 0
    w20, w26 = lib.cbtm_workspace_bytes(20), lib.cbtm_workspace_bytes(26)
    assert 11 << 20 < w20 < 13 << 20                  # ~11 bytes of scratch per slot
    assert 11 << 26 < w26 < (11 << 26) + (16 << 20)


def test_contract_violations_are_reported_before_launch(lib):
    assert lib.cbtm_sum_reduce(None, None, 40, None, 0, 0) == 1      # CBTM_E_DEPTH
    assert lib.cbtm_sum_reduce(None, None, 10, None, 0, 0) == 2      # CBTM_E_NULL
    assert lib.cbtm_decode_ones(None, None, 10, None, 4, None, 0) == 2
    assert lib.cbtm_update(None, None, 0) == 2
    pool = _lib.CPool()
    pool.depth = 99
    assert lib.cbtm_update_begin(C.byref(pool), 0) == 1


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2407_02215_b200 import Cbt, halfedge, initialize
    with pytest.raises(_lib.CbtmError):
        Cbt(4)
    with pytest.raises(_lib.CbtmError):
        initialize(halfedge.single_quad(), 8)
    with pytest.raises(_lib.CbtmError):   # the device mesh ingest has no host fallback either
        halfedge.from_polygons_device(*_quad_polygons())


def _quad_polygons():
    from paper_2407_02215_b200 import halfedge
    m = halfedge.single_quad()
    return m.positions, [[int(v) for v in m.vert]]


def test_new_entry_points_check_their_arguments(lib):
    """Contract violations of the round-1c entry points are reported before anything is launched."""
    assert lib.cbtm_wait_frame(None, 1, 1000) == 2                       # CBTM_E_NULL
    import numpy as np
    stats = np.zeros(_lib.STATS_WORDS, dtype=np.int64)
    assert lib.cbtm_wait_frame(stats.ctypes.data, 1, 2_000_000) == 7     # CBTM_E_TIMEOUT after 2 ms
    stats[_lib.STAT_SEQ] = 5
    assert lib.cbtm_wait_frame(stats.ctypes.data, 5, 1000) == 0          # already there: no spinning
    assert lib.cbtm_run_lod_sequence_batch(None, 1, None, None, 1, None, 0) == 2
    pools = (_lib.CPool * 1)()
    ptrs = (C.c_void_p * 1)(1)
    assert lib.cbtm_run_lod_sequence_batch(pools, 0, ptrs, ptrs, 1, None, 0) == 5    # CBTM_E_RANGE
    assert lib.cbtm_run_lod_sequence_batch(pools, _lib.MAX_BATCH + 1, ptrs, ptrs, 1, None, 0) == 5
    assert lib.cbtm_mesh_workspace_bytes(0) == 0 and lib.cbtm_mesh_workspace_bytes(240) > 0
    assert lib.cbtm_mesh_from_polygons(*([None] * 2), 1, 3, 3, *([None] * 8), 0, 0) == 2
    assert lib.cbtm_export_live_triangles(None, None, None, 0, None, 0) == 2
    assert lib.cbtm_update_linger(None, None, None, 1, 1000, 0) == 2
    assert lib.cbtm_run_epochs(None, None, 1, None, 0) == 2
    assert lib.cbtm_post_request(None, 1, None) == 2
    mailbox = np.zeros(64, dtype=np.int64)
    prm = np.arange(23, dtype=np.float64)
    assert lib.cbtm_post_request(mailbox.ctypes.data, 7, prm.ctypes.data) == 0
    assert mailbox[0] == 7 and np.array_equal(mailbox[8:31].view(np.float64), prm)


def test_batch_api_validates_before_touching_the_gpu():
    from paper_2407_02215_b200.pipeline import run_lod_sequence_batch
    assert run_lod_sequence_batch([], []) == []
    with pytest.raises(ValueError):
        run_lod_sequence_batch([object()], [])
