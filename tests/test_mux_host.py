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


def test_mux_c_abi_validates_before_touching_the_device():
    """ilans_mux_* check their descriptors and the schedule on the host and
    return the reference's error kinds without a device (this runs on CPU)."""
    import ctypes

    from paper_1402_3392_b200 import _lib

    st = _lib.Status()
    bad = (_lib.MuxStream * 1)()
    bad[0].kind, bad[0].nbytes, bad[0].digit_bits = _lib.MUX_RANS, 1, 12
    bad[0].scale_bits, bad[0].lower_bound, bad[0].n_sym = 2, 1 << 20, 2
    freq = np.array([1, 3], np.uint32)
    cum = np.array([0, 1, 4], np.uint32)
    sym = np.zeros(1, np.uint32)
    sched = np.zeros(1, np.int32)
    out = np.zeros(16, np.uint8)
    n = ctypes.c_int64()
    states = np.zeros(1, np.uint32)
    sbytes = np.zeros(1, np.uint64)
    segs, maxb = ctypes.c_int64(), ctypes.c_uint64()
    rc = _lib.lib.ilans_mux_encode(ctypes.byref(bad), 1, _lib.ptr(freq), 2, _lib.ptr(cum), 3,
                                   _lib.ptr(sym), _lib.ptr(sched), 1, 0, _lib.ptr(out), 16,
                                   ctypes.byref(n), _lib.ptr(states), _lib.ptr(sbytes),
                                   ctypes.byref(segs), ctypes.byref(maxb), ctypes.byref(st))
    assert rc == _lib.ERR_VALUE and b"byte-multiple" in st.message
    good = (_lib.MuxStream * 1)()
    good[0].kind, good[0].nbytes, good[0].digit_bits = _lib.MUX_RAW, 1, 8
    sched7 = np.array([7], np.int32)
    rc = _lib.lib.ilans_mux_encode(ctypes.byref(good), 1, _lib.ptr(freq), 2, _lib.ptr(cum), 3,
                                   _lib.ptr(sym), _lib.ptr(sched7), 1, 0, _lib.ptr(out), 16,
                                   ctypes.byref(n), _lib.ptr(states), _lib.ptr(sbytes),
                                   ctypes.byref(segs), ctypes.byref(maxb), ctypes.byref(st))
    assert rc == _lib.ERR_SCHEDULE and b"unknown stream 7" in st.message
    # no steps: nothing to launch, empty payload, no device needed
    rc = _lib.lib.ilans_mux_encode(ctypes.byref(good), 1, _lib.ptr(freq), 2, _lib.ptr(cum), 3,
                                   _lib.ptr(sym), _lib.ptr(sched), 0, 0, _lib.ptr(out), 16,
                                   ctypes.byref(n), _lib.ptr(states), _lib.ptr(sbytes),
                                   ctypes.byref(segs), ctypes.byref(maxb), ctypes.byref(st))
    assert rc == _lib.OK and n.value == 0 and segs.value == 0
    counts = np.array([2], np.int64)
    hoff = np.zeros(2, np.uint64)
    poff = np.zeros(2, np.uint64)
    slot = np.zeros(4, np.uint8)
    rc = _lib.lib.ilans_mux_merge(ctypes.byref(good), 1, _lib.ptr(freq), 2, _lib.ptr(cum), 3,
                                  _lib.ptr(slot), 4, _lib.ptr(out), _lib.ptr(hoff), _lib.ptr(out),
                                  _lib.ptr(poff), _lib.ptr(counts), _lib.ptr(sched), 1,
                                  _lib.ptr(out), ctypes.byref(st))
    assert rc == _lib.ERR_SCHEDULE and b"which holds 2 symbols" in st.message
