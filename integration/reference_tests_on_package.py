"""Run the reference's OWN test files against this package (not just its
kernel backend): build a throw-away `ilans` package whose modules ARE
`paper_1402_3392_b200`'s (rans, interleave, lanes, mux, backend, errors,
chunked), so `from ilans.mux import ...` in the reference tests exercises
the B200 implementation.

The reference modules outside the hot path -- the generic `ans` teaching
framework, `bench`, `cli`, and the lane-simulation helpers of `lanes`
(`LaneSet`, `ballot`, `packed_load`, ...) -- are loaded from the built
reference (oracle/_ref) *inside* that package, so their relative imports
bind to this package's modules (e.g. the reference `bench.bench_data` calls
our `encode_interleaved`). They are test infrastructure here, never part of
the product.

    python integration/reference_tests_on_package.py DEST [pytest args...]
"""

from __future__ import annotations

import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
REF = ROOT / "oracle" / "_ref"

SHIM = '''"""`ilans` aliased to paper_1402_3392_b200 (test infrastructure)."""
import importlib.util as _iu
import sys as _sys
import types as _types
from pathlib import Path as _Path

_sys.path.insert(0, {root!r})
import paper_1402_3392_b200 as _p  # noqa: E402
from paper_1402_3392_b200 import backend, chunked, errors, interleave, mux, rans  # noqa: E402

for _name in ("backend", "chunked", "errors", "interleave", "mux", "rans"):
    _sys.modules[__name__ + "." + _name] = getattr(_p, _name)

_REF = _Path({ref!r}) / "ilans"


def _load_ref(name, alias=None):
    spec = _iu.spec_from_file_location(alias or (__name__ + "." + name), _REF / (name + ".py"))
    mod = _iu.module_from_spec(spec)
    _sys.modules[spec.name] = mod
    spec.loader.exec_module(mod)
    return mod


# lanes: this package's decoders / encoders over the reference's helpers
_ref_lanes = _load_ref("lanes", __name__ + "._ref_lanes")
lanes = _types.ModuleType(__name__ + ".lanes")
lanes.__dict__.update({{k: v for k, v in vars(_ref_lanes).items() if not k.startswith("__")}})
lanes.__dict__.update({{k: v for k, v in vars(_p.lanes).items() if not k.startswith("__")}})
_sys.modules[__name__ + ".lanes"] = lanes
ans = _load_ref("ans")
bench = _load_ref("bench")
cli = _load_ref("cli")

from paper_1402_3392_b200 import *  # noqa: E402,F401,F403
from paper_1402_3392_b200.errors import *  # noqa: E402,F401,F403
from paper_1402_3392_b200.interleave import Container, decode_interleaved, encode_interleaved  # noqa: E402,F401
from paper_1402_3392_b200.rans import BYTE8, WORD16, RenormVariant, SymbolTable, quantize  # noqa: E402,F401

__version__ = "0.1.0"
'''


def build(dest: Path) -> Path:
    if not (REF / "ilans" / "ans.py").exists() or not (REF / "tests").is_dir():
        raise SystemExit(f"{REF} lacks the built reference or its tests (run oracle/build_ref.sh)")
    dest = Path(dest)
    if dest.exists():
        shutil.rmtree(dest)
    (dest / "ilans").mkdir(parents=True)
    (dest / "ilans" / "__init__.py").write_text(SHIM.format(root=str(ROOT), ref=str(REF)))
    shutil.copytree(REF / "tests", dest / "tests", ignore=shutil.ignore_patterns("__pycache__"))
    return dest


def run(dest: Path, *args: str) -> subprocess.CompletedProcess:
    env = {"PYTHONPATH": str(dest), "PATH": "/usr/bin:/bin"}
    import os

    env = dict(os.environ, PYTHONPATH=str(dest))
    env.pop("ILANS_BACKEND", None)
    return subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                           "-o", "addopts=", *args], cwd=dest, env=env, capture_output=True,
                          text=True, timeout=1800)


if __name__ == "__main__":
    d = build(Path(sys.argv[1]))
    r = run(d, *(sys.argv[2:] or ["tests"]))
    print(r.stdout[-6000:])
    print(r.stderr[-2000:], file=sys.stderr)
    sys.exit(r.returncode)
