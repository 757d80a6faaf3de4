"""The reference suite's own checks, pointed at the B200 path.

Mirrors pkg/tests/test_acceptance.py (criteria 2, 3, 5),
pkg/tests/test_interleave.py (TestRoundTrips, TestSizeInvariance,
TestNegatives), pkg/tests/test_lanes.py (TestFullCodec) and
pkg/tests/test_backend.py (TestKernelEquivalence, with the oracle standing
in for the reference's pure backend) -- same generators, seeds and
assertions, the API imported from paper_1402_3392_b200 instead of ilans.
"""

import warnings

import numpy as np
import pytest

import oracle
from paper_1402_3392_b200 import _lib, backend
from paper_1402_3392_b200.errors import (
    FormatError,
    TrailingGarbageWarning,
    TruncatedStreamError,
    UnencodableSymbolError,
    UnsupportedVariantError,
)
from paper_1402_3392_b200.interleave import (
    Container,
    decode_interleaved,
    decode_interleaved_steps,
    encode_interleaved,
)
from paper_1402_3392_b200.lanes import (
    MAX_LANES,
    decode_lanes_full,
    decode_lanes_steps,
    encode_lanes_full,
)
from paper_1402_3392_b200.rans import BYTE8, WORD16, RenormStats, SymbolTable

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if _lib.device_count() == 0:
        pytest.fail("no CUDA device: the -m gpu suite must run on a B200")


def random_table(rng, max_n=64, max_scale=14):
    n = int(rng.integers(2, max_n + 1))
    scale_bits = int(rng.integers(max(1, (n - 1).bit_length()), max_scale + 1))
    counts = rng.integers(0, 900, size=n)
    counts[int(rng.integers(0, n))] += 1
    return SymbolTable.from_counts(counts.tolist(), scale_bits)


def random_message(rng, table, n):
    probs = table.freq_u32 / table.total
    return rng.choice(table.alphabet_size, size=n, p=probs).astype(np.uint8)


def toy_table():
    return SymbolTable([1, 3], scale_bits=2)


# ------------------------------------------------------ test_acceptance ---
def test_criterion_2_serial_lane_lockstep():
    rng = np.random.default_rng(2026)
    lane_counts = (1, 2, 4, 8, 16, 32)
    messages = 0
    for lanes in lane_counts:
        lengths = [0, 1, max(0, lanes - 1), lanes, lanes + 1, 2 * lanes + 1, 97]
        lengths += [int(rng.integers(2, 3000)) for _ in range(9)]
        lengths.append(100_000 if lanes in (8, 32) else int(rng.integers(3000, 20_000)))
        for n in lengths:
            table = random_table(rng)
            msg = random_message(rng, table, n)
            container = encode_interleaved(msg, table, lanes, WORD16)
            for got, want in zip(decode_lanes_steps(container),
                                 decode_interleaved_steps(container), strict=True):
                assert got == want
            assert np.array_equal(decode_interleaved(container), msg)
            messages += 1
    assert messages == len(lane_counts) * 17


def test_criterion_3_single_renorm_word16():
    rng = np.random.default_rng(3)
    stats = RenormStats()
    for _ in range(20):
        table = random_table(rng)
        msg = random_message(rng, table, 50_000)
        container = encode_interleaved(msg, table, 4, WORD16, stats=stats)
        decoded = decode_interleaved(container, stats=stats)
        assert np.array_equal(decoded, msg)
    assert stats.encode_symbols >= 1_000_000
    assert stats.decode_symbols >= 1_000_000
    assert stats.max_encode_digits <= 1
    assert stats.max_decode_digits <= 1


def test_criterion_5_rate_near_entropy():
    rng = np.random.default_rng(5)
    probs = rng.dirichlet(np.ones(64))
    counts = np.maximum(1, (probs * 1_000_000).astype(np.int64))
    table = SymbolTable.from_counts(counts.tolist(), 14)
    msg = random_message(rng, table, 1_000_000)
    container = encode_interleaved(msg, table, 1, WORD16)
    used_bits = 8 * container.payload_nbytes + 32 * container.lane_count
    ideal = table.ideal_bits(msg)
    assert np.array_equal(decode_interleaved(container), msg)
    assert used_bits <= 1.02 * ideal + 64


# ------------------------------------------------------ test_interleave ---
@pytest.mark.parametrize("variant", [WORD16, BYTE8], ids=["word16", "byte8"])
@pytest.mark.parametrize("lanes", [1, 2, 3, 8, 17])
def test_round_trip(variant, lanes):
    rng = np.random.default_rng(lanes * 100 + variant.digit_bits)
    table = random_table(rng, max_n=80, max_scale=16)
    for n in (0, 1, lanes - 1, lanes, lanes + 1, 257, 4000):
        if n < 0:
            continue
        msg = random_message(rng, table, n)
        container = encode_interleaved(msg, table, lanes, variant)
        assert container.message_length == n
        assert len(container.final_states) == lanes
        assert np.array_equal(decode_interleaved(container), msg)


def test_wire_round_trip():
    rng = np.random.default_rng(77)
    for variant in (WORD16, BYTE8):
        table = random_table(rng, max_n=256, max_scale=16)
        msg = random_message(rng, table, 1000)
        container = encode_interleaved(msg, table, 4, variant)
        reparsed = Container.from_bytes(container.to_bytes())
        assert reparsed.variant == container.variant
        assert reparsed.lane_count == container.lane_count
        assert reparsed.message_length == container.message_length
        assert reparsed.table == container.table
        assert reparsed.final_states == container.final_states
        assert np.array_equal(reparsed.payload, container.payload)
        assert np.array_equal(decode_interleaved(reparsed), msg)


def test_decoder_returns_lanes_to_initial_state():
    rng = np.random.default_rng(8)
    table = random_table(rng, max_n=30)
    msg = random_message(rng, table, 500)
    container = encode_interleaved(msg, table, 4, WORD16)
    *_, (symbols, states, read_pos) = decode_interleaved_steps(container)
    assert states == (WORD16.lower_bound,) * 4
    assert read_pos == len(container.payload)


def test_stats_path_matches_kernel_path():
    rng = np.random.default_rng(10)
    table = random_table(rng, max_n=50)
    msg = random_message(rng, table, 777)
    stats = RenormStats()
    via_stats = encode_interleaved(msg, table, 3, WORD16, stats=stats)
    via_kernel = encode_interleaved(msg, table, 3, WORD16)
    assert via_stats.to_bytes() == via_kernel.to_bytes()
    assert stats.encode_symbols == 777
    assert stats.max_encode_digits <= 1


def test_payload_independent_of_lanes_up_to_state_flush():
    rng = np.random.default_rng(21)
    table = random_table(rng, max_n=200)
    msg = random_message(rng, table, 20000)
    base = encode_interleaved(msg, table, 1, WORD16)
    for lanes in (2, 4, 8, 32):
        container = encode_interleaved(msg, table, lanes, WORD16)
        assert abs(container.payload_nbytes - base.payload_nbytes) <= 4 * lanes
        assert abs(len(container.to_bytes()) - len(base.to_bytes())) <= 6 * lanes


def test_negatives():
    rng = np.random.default_rng(23)
    table = random_table(rng, max_n=256)
    msg = random_message(rng, table, 5000)
    blob = bytearray(encode_interleaved(msg, table, 4, WORD16).to_bytes())
    blob[6] = 5  # lane_count u16 low byte
    tampered = Container.from_bytes(bytes(blob))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        try:
            out = decode_interleaved(tampered)
            assert not np.array_equal(out, msg)
        except (TruncatedStreamError, FormatError):
            pass
    rng = np.random.default_rng(24)
    table = random_table(rng, max_n=64)
    msg = random_message(rng, table, 2000)
    container = encode_interleaved(msg, table, 2, WORD16)
    container.payload = container.payload[: len(container.payload) // 2]
    with pytest.raises(TruncatedStreamError):
        decode_interleaved(container)
    container = encode_interleaved([1, 0, 1, 1, 0] * 20, toy_table(), 1, WORD16)
    container.payload = np.concatenate([container.payload, np.asarray([123], dtype=np.uint16)])
    with pytest.warns(TrailingGarbageWarning):
        assert decode_interleaved(container).tolist() == [1, 0, 1, 1, 0] * 20
    with pytest.raises(UnencodableSymbolError):
        encode_interleaved([5], toy_table(), 1, WORD16)
    with pytest.raises(UnencodableSymbolError):
        encode_interleaved([1], SymbolTable([4, 0], 2), 1, WORD16)
    with pytest.raises(ValueError):
        encode_interleaved([1], toy_table(), 0, WORD16)


# ----------------------------------------------------------- test_lanes ---
def test_encoder_is_bit_identical_to_serial():
    rng = np.random.default_rng(11)
    for lane_count in (1, 2, 3, 5, 8, 17, 32):
        table = random_table(rng, max_n=256, max_scale=16)
        for n in (0, 1, lane_count - 1, lane_count, lane_count + 1, 333):
            if n < 0:
                continue
            msg = random_message(rng, table, n)
            via_steps = encode_lanes_full(msg, table, lane_count)
            via_serial = encode_interleaved(msg, table, lane_count, WORD16)
            assert via_steps.to_bytes() == via_serial.to_bytes()


def test_decode_lanes_full_matches_serial():
    rng = np.random.default_rng(12)
    for lane_count in (1, 2, 4, 16, 32):
        table = random_table(rng, max_n=256, max_scale=16)
        msg = random_message(rng, table, int(rng.integers(0, 2000)))
        container = encode_interleaved(msg, table, lane_count, WORD16)
        got = decode_lanes_full(container)
        assert np.array_equal(got, decode_interleaved(container))
        assert np.array_equal(got, msg)


def test_too_many_lanes_rejected():
    msg = list(range(2)) * 40
    container = encode_interleaved(msg, toy_table(), MAX_LANES + 1, WORD16)
    assert decode_interleaved(container).tolist() == msg  # serial is fine
    with pytest.raises(UnsupportedVariantError, match="at most 32"):
        decode_lanes_full(container)
    with pytest.raises(ValueError):
        encode_lanes_full(msg, toy_table(), MAX_LANES + 1)


# ---------------------------------------------------------- test_backend ---
def test_kernel_equivalence_vs_oracle():
    """TestKernelEquivalence (test_backend.py:75-128): b200 == the pure
    kernels' behaviour (restated by the oracle) on 30 random cases each."""
    def table_for(rng, max_n=200):
        n = int(rng.integers(2, max_n + 1))
        sb = int(rng.integers(max(1, (n - 1).bit_length()), 17))
        counts = rng.integers(0, 800, size=n)
        counts[int(rng.integers(0, n))] += 1
        return SymbolTable.from_counts(counts.tolist(), sb)

    b = backend.get("b200")
    rng = np.random.default_rng(60)
    for _ in range(30):
        table = table_for(rng)
        lanes = int(rng.integers(1, 33))
        msg = random_message(rng, table, int(rng.integers(0, 3000)))
        p1, s1 = b.encode_interleaved_u16(msg, table.freq_u32, table.cum_u32,
                                          table.scale_bits, lanes)
        p2, s2 = oracle.encode_interleaved_u16(msg, table.freq_u32, table.cum_u32,
                                               table.scale_bits, lanes)
        assert np.array_equal(p1, p2) and np.array_equal(s1, s2)
        for fn in (b.decode_interleaved_u16, b.decode_lanes_u16):
            out, used = fn(p1, s1, table.slot_u8, table.freq_u32, table.cum_u32,
                           table.scale_bits, len(msg), lanes)
            assert np.array_equal(out, msg) and used == len(p1)
