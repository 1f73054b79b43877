"""B200-native per-frame bisector update (arXiv 2407.02215).

Drop-in for the reference ``cbtmesh`` package's CBT / tessellation-update API:
the same names (``Cbt``, ``TriangulationState``, ``initialize``,
``ParallelEngine``, ``UpdateStats``, ``HalfedgeMesh``, ``load_obj``,
``validate``) with the update path running as hand-written sm_100a CUDA
kernels behind the C ABI of ``libcbtm.so`` (include/cbtm.h).  Importing the
package does not need a GPU; using the update path does (no CPU fallback).
"""

from .cbt import Cbt
from .halfedge import HalfedgeMesh, load_obj, validate
from .pipeline import ParallelEngine, UpdateStats
from .state import TriangulationState, initialize

__version__ = "0.1.0"

__all__ = ["Cbt", "HalfedgeMesh", "load_obj", "validate", "ParallelEngine",
           "UpdateStats", "TriangulationState", "initialize", "__version__"]
