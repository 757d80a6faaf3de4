"""Install the B200 backend into a COPY of the reference package and derive
the reference's own test suite for it.

    python integration/install_into_reference.py DEST [--ref oracle/_ref]

* copies the built, unmodified reference package ``<ref>/ilans`` to
  ``DEST/ilans`` and its test suite ``<ref>/tests`` (copied there from
  ``pkg/tests`` by oracle/build_ref.sh) to ``DEST/tests``;
* drops ``integration/ilans_b200_binding.py`` in as ``ilans/_b200.py``;
* applies the registration a maintainer would add to
  ``ilans/backend.py`` (reference backend.py:31-78): a ``B200`` Backend next
  to ``EXT``, ``ILANS_BACKEND=b200`` in ``_pick_default``, ``"b200"`` in
  ``get()`` and ``available()``;
* writes ``DEST/tests/test_backend_b200.py``: the reference's
  ``test_backend.py`` with the compiled backend ``"ext"`` replaced by
  ``"b200"`` in ``TestKernelEquivalence`` (reference test_backend.py:75-128),
  i.e. pure == b200 on the same random tables, messages and errors.

Every edit is anchored on the reference's exact source lines and fails
loudly if the reference changed. Nothing under DEST is committed; the GPU
test (tests/test_gpu_reference_own_suite.py) builds it in a temp dir.
"""

from __future__ import annotations

import argparse
import shutil
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent

# (anchor in reference backend.py, text inserted after it)
_BACKEND_EDITS = [
    (
        '''    EXT = Backend(
        "ext",
        _core.encode_interleaved_u16,
        _core.decode_interleaved_u16,
        _core.decode_lanes_u16,
    )
''',
        '''
try:  # B200 kernels over libilans_b200.so (INTEGRATION.md section 2)
    from . import _b200
except OSError:  # library or driver missing
    B200 = None
else:
    B200 = Backend(
        "b200",
        _b200.encode_interleaved_u16,
        _b200.decode_interleaved_u16,
        _b200.decode_lanes_u16,
    )
''',
    ),
    (
        '''    if forced == "pure":
        return PURE
''',
        '''    if forced == "b200":
        if B200 is None:
            warnings.warn(
                "ILANS_BACKEND=b200 but libilans_b200.so did not load; using default",
                RuntimeWarning,
            )
            return EXT if EXT is not None else PURE
        return B200
''',
    ),
    (
        '''    if name == "pure":
        return PURE
''',
        '''    if name == "b200":
        if B200 is None:
            raise ValueError("b200 backend requested but libilans_b200.so did not load")
        return B200
''',
    ),
]
_AVAILABLE_OLD = '''    return ["pure", "ext"] if EXT is not None else ["pure"]
'''
_AVAILABLE_NEW = '''    names = ["pure", "ext"] if EXT is not None else ["pure"]
    return names + (["b200"] if B200 is not None else [])
'''


def patch_backend(src: str) -> str:
    for anchor, add in _BACKEND_EDITS:
        if src.count(anchor) != 1:
            raise SystemExit(f"reference backend.py changed: anchor not found:\n{anchor}")
        src = src.replace(anchor, anchor + add)
    if src.count(_AVAILABLE_OLD) != 1:
        raise SystemExit("reference backend.py changed: available() not found")
    return src.replace(_AVAILABLE_OLD, _AVAILABLE_NEW)


def derive_kernel_equivalence(test_backend: str) -> str:
    """TestKernelEquivalence with "ext" -> "b200" (and only that class)."""
    start = test_backend.index("@needs_ext\nclass TestKernelEquivalence")
    head, body = test_backend[:start], test_backend[start:]
    body = body.replace('backend="ext"', 'backend="b200"').replace('("pure", "ext")',
                                                                     '("pure", "b200")')
    body = body.replace("@needs_ext\nclass TestKernelEquivalence",
                        "@needs_b200\nclass TestKernelEquivalence")
    if '"ext"' in body:
        raise SystemExit("reference TestKernelEquivalence changed: unreplaced 'ext'")
    head = head.replace(
        'needs_ext = pytest.mark.skipif(backend.EXT is None, reason="ilans._core not built")',
        'needs_ext = pytest.mark.skipif(backend.EXT is None, reason="ilans._core not built")\n'
        'needs_b200 = pytest.mark.skipif(getattr(backend, "B200", None) is None,\n'
        '                                reason="libilans_b200.so not loaded")')
    # keep only the module header + the derived class (the other classes run
    # unmodified from test_backend.py itself)
    doc = ('"""Derived from the reference tests/test_backend.py by '
           'integration/install_into_reference.py:\nTestKernelEquivalence with the '
           'compiled backend "ext" replaced by "b200"."""\n')
    head_lines = head.split("\n")
    i = next(k for k, ln in enumerate(head_lines) if ln.startswith("import "))
    j = next(k for k, ln in enumerate(head_lines) if ln.startswith("class TestSelection"))
    return doc + "\n".join(head_lines[i:j]) + body


def install(dest: Path, ref: Path = ROOT / "oracle" / "_ref") -> Path:
    dest = Path(dest)
    if not (ref / "ilans" / "backend.py").exists() or not (ref / "tests").is_dir():
        raise SystemExit(f"{ref} lacks the built reference or its tests (run oracle/build_ref.sh)")
    if dest.exists():
        shutil.rmtree(dest)
    dest.mkdir(parents=True)
    shutil.copytree(ref / "ilans", dest / "ilans",
                    ignore=shutil.ignore_patterns("__pycache__"))
    shutil.copytree(ref / "tests", dest / "tests", ignore=shutil.ignore_patterns("__pycache__"))
    shutil.copy(HERE / "ilans_b200_binding.py", dest / "ilans" / "_b200.py")
    bp = dest / "ilans" / "backend.py"
    bp.write_text(patch_backend(bp.read_text()))
    tb = (dest / "tests" / "test_backend.py").read_text()
    (dest / "tests" / "test_backend_b200.py").write_text(derive_kernel_equivalence(tb))
    return dest


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("dest")
    ap.add_argument("--ref", default=str(ROOT / "oracle" / "_ref"))
    a = ap.parse_args()
    print(install(Path(a.dest), Path(a.ref)))


if __name__ == "__main__":
    main()
