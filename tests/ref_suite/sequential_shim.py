"""`cbtmesh.sequential` for the reference's test-suite when it runs against the drop-in.

The reference's tests create BOTH pools with `sequential.initialize` and then drive one
with `ParallelEngine` (the product, on the GPU) and the other with
`sequential.apply_verdicts` (the reference's one-operation-at-a-time id-level oracle,
pkg/src/cbtmesh/sequential.py:260-285).  Here `initialize` is the product's; the oracle
functions are the real reference's, applied to a host copy of the GPU pool in the
reference's own `TriangulationState` and written back (records through the device
arrays, occupancy through the public `Cbt.leaves` / `sum_reduce` API).

TEST INFRASTRUCTURE ONLY: nothing under paper_2407_02215_b200/ imports this.
"""

from __future__ import annotations

import numpy as np

from paper_2407_02215_b200 import _lib
from paper_2407_02215_b200.state import CapacityError, TriangulationState, initialize  # noqa: F401

from .alias_plugin import load_reference_package

_RECORDS = ("ids", "nexts", "prevs", "twins")


def _ref():
    load_reference_package()
    import cbtmesh_ref.sequential as seq
    import cbtmesh_ref.state as state
    import cbtmesh_ref.cbt as cbt
    return seq, state, cbt


def to_reference_state(st: TriangulationState):
    """Host copy of a GPU pool as the reference's own TriangulationState."""
    _, rstate, rcbt = _ref()
    if st.depth > rcbt.MAX_DEPTH:
        rcbt.MAX_DEPTH = st.depth
    host = st.to_host()
    ref = rstate.TriangulationState(st.mesh, st.depth)
    ref.max_depth = st.max_depth
    for k in ("ids", "nexts", "prevs", "twins", "commands", "reserved", "counter",
              "cache_live", "cache_free"):
        getattr(ref, k)[...] = host[k]
    ref.cbt.nodes[...] = host["nodes"]
    return ref


def from_reference_state(ref, st: TriangulationState) -> None:
    for k in _RECORDS:
        getattr(st, "d_" + k).copy_(_lib.to_device(getattr(ref, k), st.device))
    st._touched()
    st.cbt.leaves[:] = ref.cbt.leaves
    st.cbt.sum_reduce()
    st._version += 1


def _on_host_copy(name):
    def call(state, *args, **kw):
        seq, rstate, _ = _ref()
        ref = to_reference_state(state)
        try:
            return getattr(seq, name)(ref, *args, **kw)
        except rstate.CapacityError as exc:      # the drop-in's exception type, as the tests import it
            raise CapacityError(str(exc)) from None
        finally:
            from_reference_state(ref, state)
    call.__name__ = name
    call.__doc__ = f"the reference's sequential.{name} on a host copy of the GPU pool"
    return call


apply_verdicts = _on_host_copy("apply_verdicts")
refine = _on_host_copy("refine")
decimate = _on_host_copy("decimate")


def merge_configuration(state, slot):
    return _ref()[0].merge_configuration(to_reference_state(state), slot)


def triangles(state):
    return _ref()[0].triangles(to_reference_state(state))
