"""The reference's OWN test suite run against the B200 backend through the
C ABI (the drop-in boundary proven with the reference's tests, not a
mirror of them).

integration/install_into_reference.py copies the unmodified reference
build (oracle/_ref: ilans + its Cython _core, and pkg/tests), drops in the
ctypes binding INTEGRATION.md section 2 shows (``ilans/_b200.py``) and the
``Backend("b200")`` registration (reference backend.py:31-78), and derives
``test_backend_b200.py`` = TestKernelEquivalence (reference
test_backend.py:75-128) with "ext" replaced by "b200". The whole reference
suite then runs with ``ILANS_BACKEND=b200``, so every word16 call in
test_interleave.py, test_lanes.py, test_acceptance.py, test_cli.py, ...
goes to the GPU.

Deselected, with the reason: ``TestSelection::test_ext_resolves`` asserts
the exact backend list ``["pure", "ext"]``; registering b200 adds an entry.
"""

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

from paper_1402_3392_b200 import _lib

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "integration"))

DESELECT = ["tests/test_backend.py::TestSelection::test_ext_resolves"]


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if _lib.device_count() == 0:
        pytest.fail("no CUDA device: the -m gpu suite must run on a B200")


def _run(dest, *args):
    env = dict(os.environ, ILANS_BACKEND="b200", PYTHONPATH=str(dest),
               ILANS_B200_LIB=str(Path(_lib.LIB_PATH).resolve()))
    env.pop("PYTEST_ADDOPTS", None)
    return subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                           "-o", "addopts=", *args], cwd=dest, env=env, capture_output=True,
                          text=True, timeout=1500)


@pytest.fixture(scope="module")
def ref_b200(tmp_path_factory):
    from install_into_reference import install

    return install(tmp_path_factory.mktemp("ref_b200") / "pkg")


def test_kernel_equivalence_pure_vs_b200(ref_b200):
    r = _run(ref_b200, "tests/test_backend_b200.py", "-k", "TestKernelEquivalence", "-rs")
    assert r.returncode == 0, r.stdout[-6000:] + r.stderr[-3000:]
    m = re.search(r"(\d+) passed", r.stdout)
    assert m and int(m.group(1)) == 5, r.stdout[-2000:]
    assert "skipped" not in r.stdout


def test_reference_suite_passes_with_b200_active(ref_b200):
    probe = subprocess.run(
        [sys.executable, "-c", "from ilans import backend; print(backend.ACTIVE.name)"],
        cwd=ref_b200, env=dict(os.environ, ILANS_BACKEND="b200", PYTHONPATH=str(ref_b200),
                               ILANS_B200_LIB=str(Path(_lib.LIB_PATH).resolve())),
        capture_output=True, text=True)
    assert probe.stdout.strip() == "b200", probe.stderr
    args = ["tests"]
    for d in DESELECT:
        args += ["--deselect", d]
    r = _run(ref_b200, *args)
    assert r.returncode == 0, r.stdout[-8000:] + r.stderr[-3000:]
    m = re.search(r"(\d+) passed", r.stdout)
    assert m and int(m.group(1)) >= 160, r.stdout[-2000:]
