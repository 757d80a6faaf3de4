"""Host-side parts of the multiplexer (no GPU): the IEM1 container format,
the round-robin schedule and schedule validation, against the reference's
fixtures (tests/golden/mux.npz) and pkg/tests/test_mux.py's format tests."""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_1402_3392_b200.errors import FormatError, ScheduleError, TrailingGarbageWarning, \
    TruncatedStreamError
from paper_1402_3392_b200.mux import MuxedContainer, _validate_schedule, round_robin_schedule

GOLDEN = Path(__file__).resolve().parent / "golden"


def test_golden_containers_parse_and_reserialize():
    meta = json.loads((GOLDEN / "mux.json").read_text())
    arrays = np.load(GOLDEN / "mux.npz")
    for case in meta["cases"]:
        k = case["case"]
        for r, run in enumerate(case["runs"]):
            blob = arrays[f"m{k}_f{r}_blob"].tobytes()
            c = MuxedContainer.from_bytes(blob)
            assert c.flush_interval == run["flush"]
            assert c.stream_lengths == case["lengths"]
            assert len(c.payload) == run["payload_bytes"]
            assert c.to_bytes() == blob
        if case["schedule"] == "round_robin":
            assert round_robin_schedule(case["lengths"]) == arrays[f"m{k}_sched"].tolist()


def test_round_robin_shape():
    assert round_robin_schedule([2, 3, 1]) == [0, 1, 2, 0, 1, 1]
    assert round_robin_schedule([0, 0]) == []
    assert round_robin_schedule([]) == []
    assert round_robin_schedule([0, 2, 0, 1]) == [1, 3, 1]


def test_schedule_validation_messages():
    with pytest.raises(ScheduleError, match="unknown stream 7"):
        _validate_schedule([0, 7, 9], [1, 0])
    with pytest.raises(ScheduleError, match="schedule has 1 steps for stream 1, which holds 2"):
        _validate_schedule([0, 1], [1, 2])
    assert _validate_schedule([1, 0, 1], [1, 2]).tolist() == [1, 0, 1]


def test_container_parse_errors():
    with pytest.raises(FormatError, match="magic"):
        MuxedContainer.from_bytes(b"XXXX" + b"\x00" * 20)
    good = MuxedContainer(None, [0], [b""], b"").to_bytes()
    bad = bytearray(good)
    bad[4] = 9
    with pytest.raises(FormatError, match="version"):
        MuxedContainer.from_bytes(bytes(bad))
    with pytest.raises(TruncatedStreamError):
        MuxedContainer.from_bytes(good[:6])
    with pytest.raises(TruncatedStreamError):
        MuxedContainer.from_bytes(good[:-2])
    with pytest.warns(TrailingGarbageWarning):
        parsed = MuxedContainer.from_bytes(MuxedContainer(None, [0], [b""], b"abc").to_bytes()
                                           + b"zz")
    assert parsed.payload == b"abc"
    assert MuxedContainer.from_bytes(MuxedContainer(None, [], [], b"").to_bytes()) \
        .flush_interval is None
