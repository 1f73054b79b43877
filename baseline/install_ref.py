"""Places the UNMODIFIED reference package (`cbtmesh`, pure Python + numba) and its
own test-suite under the git-ignored `baseline/_ref/`, from where they travel to
the GPU box with the repo snapshot.

    python baseline/install_ref.py            # no-op when /root/reference is absent

Used for two things only, never by the product package:
  * `bench.py` times the real `cbtmesh.pipeline.ParallelEngine` on the box's host
    cores beside the GPU path (cpu_baseline kind "reference");
  * `tests/test_ref_suite_gpu.py` runs the reference's own tests against the
    drop-in (import alias cbtmesh -> paper_2407_02215_b200).

Nothing is copied into the git history: `baseline/_ref/` is listed in .gitignore.
The reference is a plain source package (no build step), so instead of the
`pip install --target` of the base contract this is a tree copy of
`pkg/src/cbtmesh` and `pkg/tests`; pip would add nothing but metadata.
"""

from __future__ import annotations

import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
DEST = os.path.join(HERE, "_ref")
SOURCE = os.environ.get("CBTM_REFERENCE", "/root/reference")


def install(force: bool = False) -> str | None:
    src_pkg = os.path.join(SOURCE, "pkg", "src", "cbtmesh")
    src_tests = os.path.join(SOURCE, "pkg", "tests")
    if not os.path.isdir(src_pkg):
        return DEST if os.path.isdir(os.path.join(DEST, "cbtmesh")) else None
    if force and os.path.isdir(DEST):
        shutil.rmtree(DEST)
    os.makedirs(DEST, exist_ok=True)
    for src, name in ((src_pkg, "cbtmesh"), (src_tests, "tests")):
        dst = os.path.join(DEST, name)
        if os.path.isdir(dst):
            shutil.rmtree(dst)
        shutil.copytree(src, dst, ignore=shutil.ignore_patterns("__pycache__", "*.pyc", "*.nbi", "*.nbc"))
    return DEST


if __name__ == "__main__":
    where = install(force="--force" in sys.argv)
    print(where or "reference not available here and baseline/_ref is empty")
