"""pytest plugin (`-p tests.ref_suite.alias_plugin`): makes `import cbtmesh` resolve to
the B200 drop-in, so that the reference's test files run UNMODIFIED against it.

    cbtmesh, cbtmesh.cbt / pipeline / state / lod / bisector / halfedge
        -> paper_2407_02215_b200 and its modules (the product under test)
    cbtmesh.sequential
        -> tests.ref_suite.sequential_shim: `initialize` is the product's; the id-level
           engine (`apply_verdicts`, `refine`, `decimate`, ...) is the REAL reference's
           sequential.py (loaded from baseline/_ref as `cbtmesh_ref`), run on a host copy
           of the state and written back.  It is the reference's own test oracle
           (out of scope for the product), never part of the product package.

The plugin is imported before the reference's conftest.py, whose first statement is
`from cbtmesh import ...`.
"""

from __future__ import annotations

import importlib
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = os.path.join(ROOT, "baseline", "_ref")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def load_reference_package():
    """The real reference as package `cbtmesh_ref` (its relative imports stay inside it)."""
    if "cbtmesh_ref" in sys.modules:
        return sys.modules["cbtmesh_ref"]
    import importlib.util
    init = os.path.join(REF, "cbtmesh", "__init__.py")
    if not os.path.exists(init):
        raise RuntimeError(f"{init} is missing: run `python baseline/install_ref.py` where /root/reference exists")
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(REF, ".numba_cache"))
    spec = importlib.util.spec_from_file_location(
        "cbtmesh_ref", init, submodule_search_locations=[os.path.join(REF, "cbtmesh")])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["cbtmesh_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def install_alias():
    import paper_2407_02215_b200 as product
    alias = types.ModuleType("cbtmesh")
    alias.__path__ = []          # a package, but every submodule is pre-registered below
    alias.__doc__ = "alias of paper_2407_02215_b200 for the reference's test-suite"
    for name in getattr(product, "__all__", []):
        setattr(alias, name, getattr(product, name))
    sys.modules["cbtmesh"] = alias
    for sub in ("cbt", "pipeline", "state", "lod", "bisector", "halfedge"):
        mod = importlib.import_module(f"paper_2407_02215_b200.{sub}")
        sys.modules[f"cbtmesh.{sub}"] = mod
        setattr(alias, sub, mod)
    shim = importlib.import_module("tests.ref_suite.sequential_shim")
    sys.modules["cbtmesh.sequential"] = shim
    alias.sequential = shim
    alias.refine, alias.decimate = shim.refine, shim.decimate
    return alias


install_alias()
