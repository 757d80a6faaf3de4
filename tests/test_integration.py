"""CPU checks of the reference-side integration:
the installer patches a copy of the unmodified reference so that
``Backend("b200")`` registers (the library loads without a GPU; calls
would need one), and the derived TestKernelEquivalence targets "b200"."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "integration"))
REF = ROOT / "oracle" / "_ref"


@pytest.fixture(scope="module")
def ref_b200(tmp_path_factory):
    if not (REF / "tests").is_dir():
        pytest.skip("oracle/_ref not built with its tests (oracle/build_ref.sh)")
    from install_into_reference import install

    return install(tmp_path_factory.mktemp("ref") / "pkg")


def test_backend_registration(ref_b200):
    from paper_1402_3392_b200 import _lib

    code = ("from ilans import backend\n"
            "print(backend.available(), backend.ACTIVE.name, backend.get('b200').name)\n")
    env = dict(os.environ, ILANS_BACKEND="b200", PYTHONPATH=str(ref_b200),
               ILANS_B200_LIB=str(Path(_lib.LIB_PATH).resolve()))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == "['pure', 'ext', 'b200'] b200 b200"
    # unchanged default without the env override: the reference's own choice
    env.pop("ILANS_BACKEND")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    assert r.stdout.strip() == "['pure', 'ext', 'b200'] ext b200", r.stderr


def test_derived_kernel_equivalence_targets_b200(ref_b200):
    src = (ref_b200 / "tests" / "test_backend_b200.py").read_text()
    assert "class TestKernelEquivalence" in src and "class TestSelection" not in src
    assert src.count('backend="b200"') == 3 and src.count('("pure", "b200")') == 2
    assert 'backend="ext"' not in src and '("pure", "ext")' not in src
    compile(src, "test_backend_b200.py", "exec")
