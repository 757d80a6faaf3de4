"""Pin the CPU oracle (oracle/rans_oracle.c) before trusting it.

The oracle is checked against (1) the reference suite's own known-answer
tests, (2) golden fixtures produced by the unmodified reference
(tests/golden/make_golden.py) and (3) the container digests in BASELINE.md
section 3. CPU only.
"""

import hashlib
import struct

import numpy as np
import pytest

import oracle
from conftest import ZIPF_1MIB_DIGESTS, ZIPF_1MIB_INPUT_SHA, zipf_1mib


def iec1_bytes(lanes, n, sb, freqs, states, payload):
    """IEC1 word16 container bytes, per the layout in interleave.py:10-20."""
    head = b"IEC1" + struct.pack("<BBHQ", 1, 1, lanes, n)
    table = struct.pack("<BH", sb, len(freqs)) + struct.pack(f"<{len(freqs)}H", *freqs)
    st = struct.pack(f"<{lanes}I", *[int(x) for x in states])
    return head + table + st + np.ascontiguousarray(payload, dtype="<u2").tobytes()


def test_known_answer_golden_container():
    # pkg/tests/test_interleave.py:68-80: msg [1], table [1,3] @ sb=2, N=1
    f, cum, slot = oracle.table_views([1, 3], 2)
    payload, states = oracle.encode_interleaved_u16([1], f, cum, 2, 1)
    assert states.tolist() == [87382] and len(payload) == 0
    blob = iec1_bytes(1, 1, 2, [1, 3], states, payload)
    assert blob == (b"IEC1" + b"\x01\x01\x01\x00" + b"\x01" + b"\x00" * 7
                    + b"\x02\x02\x00\x01\x00\x03\x00" + b"\x56\x55\x01\x00")
    out, consumed = oracle.decode_interleaved_u16(payload, states, slot, f, cum, 2, 1, 1)
    assert out.tolist() == [1] and consumed == 0


def test_known_answer_single_spill_extreme():
    # pkg/tests/test_rans.py:139-144 uses table [1, 0*254, m-1] @ sb=14 and a
    # state near 2^32 - 1: encoding symbol 0 (f=1) spills exactly one digit.
    # The kernel boundary has no initial-state argument, so drive the lane up
    # with ~190K pushes of symbol 255 (f = m-1 grows x by m/(m-1) each).
    sb = 14
    freqs = [1] + [0] * 254 + [(1 << sb) - 1]
    f, cum, slot = oracle.table_views(freqs, sb)
    msg = np.array([0] + [255] * 190_000, dtype=np.uint8)
    payload, states = oracle.encode_interleaved_u16(msg, f, cum, sb, 1)
    assert len(payload) == 1  # the single spill, at the f=1 symbol
    assert 65536 <= int(states[0]) < 1 << 32
    out, consumed = oracle.decode_interleaved_u16(payload, states, slot, f, cum, sb,
                                                   len(msg), 1)
    assert np.array_equal(out, msg) and consumed == 1


def test_known_answer_quantize():
    # pkg/tests/test_rans.py:49-74
    assert oracle.quantize([1, 3], 2) == [1, 3]
    assert oracle.quantize([1, 1, 1, 1], 2) == [1, 1, 1, 1]
    assert oracle.quantize([9, 9, 9, 9], 2) == [1, 1, 1, 1]
    assert oracle.quantize([10**6, 1], 14) == [16383, 1]
    for bad in (([0, 0], 4), ([1, 2], 0), ([1, 2], 17), ([1] * 300, 12), ([1] * 5, 2)):
        with pytest.raises(oracle.OracleError):
            oracle.quantize(*bad)


def test_quantize_matches_reference_fixtures(golden_quantize, golden_meta):
    for case in golden_meta["quantize"]:
        k = case["case"]
        counts = golden_quantize[f"q{k}_counts"]
        want = golden_quantize[f"q{k}_freq"].tolist()
        assert oracle.quantize(counts, case["scale_bits"]) == want, case


def test_codec_matches_reference_fixtures(golden_codec, golden_meta):
    for case in golden_meta["codec"]:
        k, lanes, sb = case["case"], case["lanes"], case["scale_bits"]
        msg = golden_codec[f"c{k}_msg"]
        freq = golden_codec[f"c{k}_freq"]
        f, cum, slot = oracle.table_views(freq, sb)
        payload, states = oracle.encode_interleaved_u16(msg, f, cum, sb, lanes)
        assert np.array_equal(payload, golden_codec[f"c{k}_payload"]), case
        assert np.array_equal(states, golden_codec[f"c{k}_states"]), case
        if case["sha256"] is not None:
            blob = iec1_bytes(lanes, len(msg), sb, freq.tolist(), states, payload)
            assert hashlib.sha256(blob).hexdigest() == case["sha256"]
        out, consumed = oracle.decode_interleaved_u16(payload, states, slot, f, cum, sb,
                                                       len(msg), lanes)
        assert np.array_equal(out, msg) and consumed == len(payload)
        if lanes <= 32:
            out2, consumed2 = oracle.decode_lanes_u16(payload, states, slot, f, cum, sb,
                                                       len(msg), lanes)
            assert np.array_equal(out2, msg) and consumed2 == len(payload)
        xs = oracle.decode_final_states(payload, states, slot, f, cum, sb, len(msg), lanes)
        assert (xs == 65536).all()


def test_chunk_framing_matches_reference_per_chunk(golden_chunks, golden_meta):
    for case in golden_meta["chunks"]:
        k, sb, chunk = case["case"], case["scale_bits"], case["chunk"]
        msg = golden_chunks[f"k{k}_msg"]
        f, cum, slot = oracle.table_views(golden_chunks[f"k{k}_freq"], sb)
        payload, offs, states = oracle.encode_chunks_u16(msg, chunk, f, cum, sb, 32)
        assert np.array_equal(payload, golden_chunks[f"k{k}_payload"])
        assert np.array_equal(offs, golden_chunks[f"k{k}_offsets"])
        assert np.array_equal(states, golden_chunks[f"k{k}_states"])
        out = oracle.decode_chunks_u16(payload, offs, states, slot, f, cum, sb, len(msg),
                                       chunk, 32)
        assert np.array_equal(out, msg)


def test_baseline_md_digests():
    msg = zipf_1mib()
    assert hashlib.sha256(msg.tobytes()).hexdigest()[:16] == ZIPF_1MIB_INPUT_SHA
    counts, alpha = oracle.histogram(msg)
    assert np.array_equal(counts[:alpha], np.bincount(msg, minlength=int(msg.max()) + 1))
    for (lanes, sb), digest in ZIPF_1MIB_DIGESTS.items():
        freqs = oracle.quantize(counts[:alpha], sb)
        f, cum, _ = oracle.table_views(freqs, sb)
        payload, states = oracle.encode_interleaved_u16(msg, f, cum, sb, lanes)
        blob = iec1_bytes(lanes, len(msg), sb, freqs, states, payload)
        assert hashlib.sha256(blob).hexdigest()[:16] == digest, (lanes, sb)


def iec1_byte8_bytes(lanes, n, sb, freqs, states, payload):
    head = b"IEC1" + struct.pack("<BBHQ", 1, 0, lanes, n)
    table = struct.pack("<BH", sb, len(freqs)) + struct.pack(f"<{len(freqs)}H", *freqs)
    st = struct.pack(f"<{lanes}I", *[int(x) for x in states])
    return head + table + st + np.ascontiguousarray(payload, dtype=np.uint8).tobytes()


def test_byte8_matches_reference_fixtures(golden_byte8, golden_meta):
    for case in golden_meta["byte8"]:
        k, lanes, sb = case["case"], case["lanes"], case["scale_bits"]
        msg = golden_byte8[f"b{k}_msg"]
        freq = golden_byte8[f"b{k}_freq"]
        f, cum, slot = oracle.table_views(freq, sb)
        payload, states = oracle.encode_interleaved_u8(msg, f, cum, sb, lanes)
        assert np.array_equal(payload, golden_byte8[f"b{k}_payload"]), case
        assert np.array_equal(states, golden_byte8[f"b{k}_states"]), case
        if case["sha256"] is not None:
            blob = iec1_byte8_bytes(lanes, len(msg), sb, freq.tolist(), states, payload)
            assert hashlib.sha256(blob).hexdigest() == case["sha256"]
        out, used = oracle.decode_interleaved_u8(payload, states, slot, f, cum, sb, len(msg),
                                                 lanes)
        assert np.array_equal(out, msg) and used == len(payload)


def test_byte8_baseline_md_digest():
    from conftest import ZIPF_1MIB_BYTE8_DIGEST, ZIPF_1MIB_BYTE8_STATES

    msg = zipf_1mib()
    counts, alpha = oracle.histogram(msg)
    freqs = oracle.quantize(counts[:alpha], 12)
    f, cum, slot = oracle.table_views(freqs, 12)
    payload, states = oracle.encode_interleaved_u8(msg, f, cum, 12, 2)
    assert tuple(states.tolist()) == ZIPF_1MIB_BYTE8_STATES
    blob = iec1_byte8_bytes(2, len(msg), 12, freqs, states, payload)
    assert hashlib.sha256(blob).hexdigest()[:16] == ZIPF_1MIB_BYTE8_DIGEST
    with pytest.raises(oracle.OracleError) as e:
        oracle.decode_interleaved_u8(payload[:-5], states, slot, f, cum, 12, len(msg), 2)
    assert e.value.kind == "truncated"


def test_truncation_and_unencodable():
    f, cum, slot = oracle.table_views([1, 3], 2)
    msg = np.array([0, 1, 1, 0, 1] * 400, dtype=np.uint8)
    payload, states = oracle.encode_interleaved_u16(msg, f, cum, 2, 4)
    with pytest.raises(oracle.OracleError) as e:
        oracle.decode_interleaved_u16(payload[: len(payload) // 3], states, slot, f, cum, 2,
                                      len(msg), 4)
    assert e.value.kind == "truncated"
    with pytest.raises(oracle.OracleError) as e:
        oracle.decode_lanes_u16(payload[:-1], states, slot, f, cum, 2, len(msg), 4)
    assert e.value.kind == "truncated"
    f0, cum0, _ = oracle.table_views([4, 0], 2)
    with pytest.raises(oracle.OracleError) as e:
        oracle.encode_interleaved_u16([0, 1, 0], f0, cum0, 2, 2)
    assert e.value.kind == "unencodable"


def test_reference_build_agrees_when_present():
    """When oracle/_ref holds the compiled reference, oracle == reference ext."""
    ref = oracle.reference_ilans()
    if ref is None:
        pytest.skip("oracle/_ref not built (bash oracle/build_ref.sh)")
    from ilans import backend as ref_backend
    from ilans.rans import SymbolTable

    ext = ref_backend.get("ext")
    rng = np.random.default_rng(5)
    for _ in range(20):
        n_sym = int(rng.integers(2, 257))
        sb = int(rng.integers(max(1, (n_sym - 1).bit_length()), 17))
        counts = rng.integers(0, 500, size=n_sym)
        counts[0] += 1
        t = SymbolTable.from_counts(counts.tolist(), sb)
        lanes = int(rng.integers(1, 40))
        msg = rng.choice(n_sym, size=int(rng.integers(0, 5000)),
                         p=t.freq_u32 / t.total).astype(np.uint8)
        a = ext.encode_interleaved_u16(msg, t.freq_u32, t.cum_u32, sb, lanes)
        b = oracle.encode_interleaved_u16(msg, t.freq_u32, t.cum_u32, sb, lanes)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
