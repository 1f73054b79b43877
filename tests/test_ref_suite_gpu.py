"""GPU: the reference's OWN acceptance suite (pkg/tests, shipped unmodified in the
git-ignored baseline/_ref/tests by baseline/install_ref.py) run against the drop-in
through an import alias `cbtmesh` -> `paper_2407_02215_b200` (tests/ref_suite/).

Each reference test file runs in a subprocess (its conftest.py and `from conftest import`
expect to be the rootdir) and must pass completely: the randomized equivalence against
`sequential.apply_verdicts` for threads 1/2/4/8, schedule independence, the one-level
rule, live accounting, the hypothesis properties of the CBT, LodDecide == python decide.
"""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(ROOT, "baseline", "_ref", "tests")

# file -> number of test items the reference's suite holds there (parametrized cases counted)
FILES = {
    "test_cbt.py": 16,
    "test_pipeline.py": 20,
    "test_lod.py": 18,
    "test_bisector.py": 14,
    "test_halfedge.py": 17,
    "test_sequential.py": 21,
}


def run_reference_file(name):
    if not os.path.isdir(REF_TESTS):
        pytest.fail("baseline/_ref/tests is missing: run `python baseline/install_ref.py` "
                    "(or __graft_entry__.build()) where /root/reference exists")
    env = dict(os.environ)
    env["PYTHONPATH"] = ROOT + os.pathsep + env.get("PYTHONPATH", "")
    env.setdefault("NUMBA_CACHE_DIR", os.path.join(ROOT, "baseline", "_ref", ".numba_cache"))
    cmd = [sys.executable, "-m", "pytest", os.path.join(REF_TESTS, name), "-q", "-x",
           "-p", "tests.ref_suite.alias_plugin", "-p", "no:cacheprovider",
           "--rootdir", REF_TESTS, "-c", os.devnull]
    proc = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    tail = (proc.stdout + proc.stderr)[-4000:]
    assert proc.returncode == 0, f"reference {name} failed against the drop-in:\n{tail}"
    m = re.search(r"(\d+) passed", proc.stdout)
    assert m, tail
    assert "failed" not in proc.stdout.splitlines()[-1] and "error" not in proc.stdout.splitlines()[-1], tail
    return int(m.group(1))


@pytest.mark.parametrize("name", list(FILES))
def test_reference_suite_file_passes_against_drop_in(name):
    passed = run_reference_file(name)
    if FILES[name] is not None:
        assert passed == FILES[name], f"{name}: {passed} passed, the reference holds {FILES[name]}"
