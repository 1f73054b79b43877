"""ctypes binding of libcbtm.so (include/cbtm.h) plus device-memory plumbing.

PyTorch is used for what it is good at here -- owning device buffers, streams
and host<->device copies.  Every computation goes through the C ABI.  There is
NO CPU fallback: if the library is missing or no CUDA device is present, the
product path raises.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# (CBTM_LIB: another build of the same library -- a debug build with timing probes, an older build for an
# A/B measurement; still the CUDA library, there is no other implementation to fall back to)
LIB_PATH = os.environ.get("CBTM_LIB") or os.path.join(_HERE, "libcbtm.so")

PRM_WORDS = 23
STATS_WORDS = 32
STAT_PHASE_NS = 16
STAT_FRAME = 11
STAT_SEQ = 31
STAT_DONE = 30
PHASE_NAMES = ("index", "classify_admit_scatter", "agree", "reserve", "apply", "reduce_publish")
MIN_DEPTH = 1
MAX_DEPTH_ABI = 30
MAX_BATCH = 8

POOL_FULL_FREE_CACHE = 1
POOL_STAGED_LAUNCHES = 2
POOL_DESCEND_FREE_RANKS = 4
POOL_WIDE_GRID = 8
POOL_FINAL_ROW = 16

VERDICT_CONST, VERDICT_UNIFORM, VERDICT_LOD, VERDICT_EXPLICIT = 0, 1, 2, 3

STAT_NAMES = ("oom_splits", "oom_merges", "split_freed", "merge_freed",
              "split_alloc", "merge_alloc", "live_before", "live_after",
              "reserved", "allocated", "poison", "frame", "peak_depth")

_ERRORS = {1: "depth out of range", 2: "required pointer is NULL",
           3: "workspace too small", 4: "unknown verdict mode",
           5: "argument out of range", 6: "buffer not 16-byte aligned",
           7: "timed out waiting for the frame's stats"}


class CbtmError(RuntimeError):
    """A C-ABI call failed (contract violation or CUDA error)."""


class CPool(C.Structure):
    _fields_ = [
        ("ids", C.c_void_p), ("nexts", C.c_void_p), ("prevs", C.c_void_p),
        ("twins", C.c_void_p), ("commands", C.c_void_p),
        ("reserved", C.c_void_p), ("cache_live", C.c_void_p),
        ("cache_free", C.c_void_p), ("counter", C.c_void_p),
        ("bits", C.c_void_p), ("counters", C.c_void_p), ("stats", C.c_void_p),
        ("dispatch", C.c_void_p), ("workspace", C.c_void_p),
        ("workspace_bytes", C.c_size_t), ("depth", C.c_int32),
        ("rank", C.c_int32), ("max_depth", C.c_int32), ("flags", C.c_uint32),
    ]


class CVerdict(C.Structure):
    _fields_ = [
        ("mode", C.c_int32), ("value", C.c_int32),
        ("explicit_verdicts", C.c_void_p), ("root_tris", C.c_void_p),
        ("prm", C.c_double * PRM_WORDS),
    ]


# name -> (restype, argtypes); mirrors include/cbtm.h one to one
_P, _I, _I64, _SZ, _UP = C.c_void_p, C.c_int, C.c_int64, C.c_size_t, C.c_size_t
SIGNATURES = {
    "cbtm_abi_version": (C.c_int, []),
    "cbtm_bitfield_words": (_SZ, [_I]),
    "cbtm_counter_words": (_SZ, [_I]),
    "cbtm_workspace_bytes": (_SZ, [_I]),
    "cbtm_cbt_workspace_bytes": (_SZ, [_I]),
    "cbtm_sum_reduce": (C.c_int, [_P, _P, _I, _P, _SZ, _UP]),
    "cbtm_decode_ones": (C.c_int, [_P, _P, _I, _P, _I64, _P, _UP]),
    "cbtm_decode_zeros": (C.c_int, [_P, _P, _I, _P, _I64, _P, _UP]),
    "cbtm_index": (C.c_int, [_P, _P, _I, _P, _P, _P, _UP]),
    "cbtm_import_leaves": (C.c_int, [_P, _I, _P, _UP]),
    "cbtm_export_nodes": (C.c_int, [_P, _P, _I, _P, _UP]),
    "cbtm_initialize": (C.c_int, [C.POINTER(CPool), _P, _P, _P, C.c_int32, _UP]),
    "cbtm_mesh_workspace_bytes": (_SZ, [_I64]),
    "cbtm_mesh_from_polygons": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _UP]),
    "cbtm_root_triangles": (C.c_int, [_P, _P, _P, C.c_int32, _P, _UP]),
    "cbtm_classify": (C.c_int, [C.POINTER(CPool), C.POINTER(CVerdict), _P, _UP]),
    "cbtm_decode_triangles": (C.c_int, [_P, _I64, C.c_int32, _P, _P, _UP]),
    "cbtm_export_live_triangles": (C.c_int, [C.POINTER(CPool), _P, _P, _I64, _P, _UP]),
    "cbtm_validate": (C.c_int, [C.POINTER(CPool), C.c_int32, _P, _UP]),
    "cbtm_update": (C.c_int, [C.POINTER(CPool), C.POINTER(CVerdict), _UP]),
    "cbtm_update_begin": (C.c_int, [C.POINTER(CPool), _UP]),
    "cbtm_update_finish": (C.c_int, [C.POINTER(CPool), C.POINTER(CVerdict), _UP]),
    "cbtm_run_lod_sequence": (C.c_int, [C.POINTER(CPool), _P, _P, C.c_int32, _P, _UP]),
    "cbtm_update_linger": (C.c_int, [C.POINTER(CPool), C.POINTER(CVerdict), _P, _I64, _I64, _UP]),
    "cbtm_post_request": (C.c_int, [_P, _I64, _P]),
    "cbtm_run_epochs": (C.c_int, [C.POINTER(CPool), C.POINTER(CVerdict), C.c_int32, _P, _UP]),
    "cbtm_wait_frame": (C.c_int, [_P, _I64, C.c_uint64]),
    "cbtm_wait_frame_done": (C.c_int, [_P, _I64, C.c_uint64]),
    "cbtm_update_wait": (C.c_int, [C.POINTER(CPool), C.POINTER(CVerdict), _P, C.c_uint64, _UP]),
    "cbtm_run_lod_sequence_batch": (C.c_int, [C.POINTER(CPool), C.c_int32, _P, _P, C.c_int32, _P, _UP]),
}

_lib = None


def load():
    """The loaded library.  Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CbtmError(
                f"{LIB_PATH} is missing: build it with "
                "`python -m paper_2407_02215_b200.build` (needs nvcc). "
                "There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)  # AttributeError if the symbol is missing
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    if rc > 0:
        raise CbtmError(f"{what}: contract violation: {_ERRORS.get(rc, rc)}")
    raise CbtmError(f"{what}: CUDA error {-rc}")


# -- device plumbing (torch) -------------------------------------------------

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as _t
        _torch = _t
    return _torch


def require_cuda(device=None):
    """A torch CUDA device, or a loud failure (no CPU fallback)."""
    t = torch()
    if not t.cuda.is_available():
        raise CbtmError(
            "no CUDA device available: the bisector update runs only on the "
            "GPU (sm_100a); there is no CPU fallback")
    load()
    if device is None:
        return t.device("cuda", t.cuda.current_device())
    return t.device(device)


def stream_handle(device) -> int:
    """cudaStream_t of torch's current stream on `device` (the raw query is a
    fraction of the cost of building a torch.cuda.Stream object every frame)."""
    t = torch()
    raw = getattr(t._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return int(raw(device.index if device.index is not None else t.cuda.current_device()))
    return int(t.cuda.current_stream(device).cuda_stream)


def ptr(tensor) -> int:
    return 0 if tensor is None else int(tensor.data_ptr())


_NP_TO_TORCH = None


def to_device(array: np.ndarray, device):
    """numpy -> device tensor (uint64/uint32 travel as int64/int32 bits)."""
    t = torch()
    a = np.ascontiguousarray(array)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    elif a.dtype == np.uint32:
        a = a.view(np.int32)
    return t.from_numpy(a).to(device)


def to_host(tensor, dtype=None) -> np.ndarray:
    a = tensor.detach().cpu().numpy()
    if dtype is not None and a.dtype != np.dtype(dtype):
        a = a.view(dtype)
    return a
