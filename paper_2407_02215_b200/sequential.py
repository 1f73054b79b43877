"""Compatibility shim: the reference re-exports ``initialize`` and
``CapacityError`` from ``cbtmesh.sequential`` (sequential.py:13).  The
single-threaded refine/decimate engine itself is the reference's id-level test
oracle and is out of scope for the GPU build."""

from .state import CapacityError, TriangulationState, initialize  # noqa: F401

__all__ = ["initialize", "CapacityError", "TriangulationState"]
