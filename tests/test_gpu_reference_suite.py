"""The reference's own test suite through the drop-in boundary.

``make -C oracle ref`` copies /root/reference/pkg/src/gridknn and pkg/tests
into the git-ignored oracle/_ref (they travel to the GPU box like the .so
files); tests/ref_suite_plugin.py routes every default / "compiled" backend
lookup of that unmodified front-end to paper_2511_10442_b200.backend.  Each
file runs in its own pytest subprocess; the only failures allowed are the
ones listed in EXPECTED, each with the documented reason.
"""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")

# test id -> why the reference's assertion does not hold for the device backend
EXPECTED = {
    "test_backends.py::test_compiled_backend_selected_by_default":
        "asserts the default backend's NAME == 'compiled'; the plugin routes the default "
        "to this backend, whose NAME is 'cuda'",
}

# timing-based checks of the reference's CPU kernels (binned >= 5x brute at
# n = 1e5 on the host cores): not a property of the device path
DESELECT = [
    "test_acceptance.py::test_criterion_6_performance_trend",
]

FILES = ["test_backends.py", "test_knn.py", "test_binning.py", "test_stepper.py",
         "test_acceptance.py", "test_core.py", "test_gravnet.py", "test_ocgraph.py",
         "test_harness.py"]


def _run(fname):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT, os.path.join(ROOT, "tests"), env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", os.path.join(REF, "tests", fname), "-q", "-rfE",
           "-p", "ref_suite_plugin", "-p", "no:cacheprovider", "--timeout", "900"]
    for d in DESELECT:
        f, t = d.split("::")
        if f == fname:
            cmd += ["--deselect", os.path.relpath(os.path.join(REF, "tests", f), ROOT) + "::" + t]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    return r.returncode, r.stdout + r.stderr


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "tests")),
                    reason="oracle/_ref not built (make -C oracle ref)")
@pytest.mark.parametrize("fname", FILES)
def test_reference_file(fname):
    rc, out = _run(fname)
    failed = set(re.findall(r"^FAILED \S*?tests/(\S+?\.py::\S+)", out, re.M))
    failed |= set(re.findall(r"^ERROR \S*?tests/(\S+?\.py::\S+)", out, re.M))
    unexpected = sorted(f for f in failed if f not in EXPECTED)
    assert not unexpected, f"{fname}: unexpected failures {unexpected}\n{out[-4000:]}"
    assert rc in (0, 1), out[-4000:]
    assert re.search(r"\d+ passed", out), out[-2000:]
    print(out.strip().splitlines()[-1])
