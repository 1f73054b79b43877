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
    assert lib.cbtm_abi_version() == 1
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
