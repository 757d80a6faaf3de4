import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
for p in (str(ROOT), str(ROOT / "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden_meta():
    return json.loads((GOLDEN / "golden.json").read_text())


@pytest.fixture(scope="session")
def golden_codec():
    return np.load(GOLDEN / "codec.npz")


@pytest.fixture(scope="session")
def golden_quantize():
    return np.load(GOLDEN / "quantize.npz")


@pytest.fixture(scope="session")
def golden_chunks():
    return np.load(GOLDEN / "chunks.npz")


@pytest.fixture(scope="session")
def golden_byte8():
    return np.load(GOLDEN / "byte8.npz")


# byte8 N=2 sb=12 on the same 1 MiB input
ZIPF_1MIB_BYTE8_DIGEST = "1ea63c4d860a4650"
ZIPF_1MIB_BYTE8_STATES = (48568369, 187084597)


def zipf_probs(s: float, n: int = 256) -> np.ndarray:
    p = (np.arange(n) + 1.0) ** -s
    return p / p.sum()


# BASELINE.md section 3 known-answer digests: 1 MiB, default_rng(1).choice,
# Zipf s=1.1, numpy 2.3.x; (lanes, scale_bits) -> container sha256[:16]
ZIPF_1MIB_INPUT_SHA = "74d2a2def4b10084"
ZIPF_1MIB_DIGESTS = {
    (32, 12): "da65beaaa96dca90",
    (32, 14): "24c8af93cbf52dc5",
    (32, 15): "f38be6883bb152df",
    (1, 14): "2e0325ca5b0f5828",
    (2, 11): "75aba17650a48d4a",
}


def zipf_1mib():
    return np.random.default_rng(1).choice(256, 2**20, p=zipf_probs(1.1)).astype(np.uint8)
