"""BYTE8 (8-bit digits, L = 2^23) on the B200 vs the reference's scalar path:
golden fixtures from the reference, the BASELINE.md config-1 digest
(byte8 N=2 sb=12, 1 MiB), lane counts past 32, truncation, lockstep steps
and the stats counters (max digits per symbol > 1 for byte8)."""

import hashlib

import numpy as np
import pytest

import oracle
import paper_1402_3392_b200 as ilb
from conftest import ZIPF_1MIB_BYTE8_DIGEST, ZIPF_1MIB_BYTE8_STATES, zipf_1mib
from paper_1402_3392_b200 import _lib
from paper_1402_3392_b200.errors import TruncatedStreamError, UnsupportedVariantError
from paper_1402_3392_b200.interleave import Container, decode_interleaved_steps
from paper_1402_3392_b200.lanes import decode_lanes_steps
from paper_1402_3392_b200.rans import BYTE8, RenormStats, SymbolTable

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if _lib.device_count() == 0:
        pytest.fail("no CUDA device: the -m gpu suite must run on a B200")


def random_table(rng, max_n=200, max_sb=16):
    n = int(rng.integers(2, max_n + 1))
    sb = int(rng.integers(max(1, (n - 1).bit_length()), max_sb + 1))
    counts = rng.integers(0, 1000, size=n)
    counts[int(rng.integers(0, n))] += 1
    return SymbolTable(oracle.quantize(counts, sb), sb)


def random_message(rng, table, n):
    return rng.choice(table.alphabet_size, size=n, p=table.freq_u32 / table.total).astype(np.uint8)


def test_byte8_matches_reference_fixtures(golden_byte8, golden_meta):
    for case in golden_meta["byte8"]:
        k, lanes, sb = case["case"], case["lanes"], case["scale_bits"]
        msg = golden_byte8[f"b{k}_msg"]
        t = SymbolTable(golden_byte8[f"b{k}_freq"].tolist(), sb)
        c = ilb.encode_interleaved(msg, t, lanes, BYTE8)
        assert np.array_equal(c.payload, golden_byte8[f"b{k}_payload"]), case
        assert c.final_states == tuple(golden_byte8[f"b{k}_states"].tolist()), case
        if case["sha256"] is not None:
            assert hashlib.sha256(c.to_bytes()).hexdigest() == case["sha256"]
        assert np.array_equal(ilb.decode_interleaved(Container.from_bytes(c.to_bytes())), msg)


def test_byte8_config1_digest():
    msg = zipf_1mib()
    counts, alpha = oracle.histogram(msg)
    t = SymbolTable.from_counts(counts[:alpha].tolist(), 12)
    c = ilb.encode_interleaved(msg, t, 2, BYTE8)
    assert c.final_states == ZIPF_1MIB_BYTE8_STATES
    assert hashlib.sha256(c.to_bytes()).hexdigest()[:16] == ZIPF_1MIB_BYTE8_DIGEST
    assert np.array_equal(ilb.decode_interleaved(c), msg)


def test_byte8_many_lanes_and_oracle_fuzz():
    rng = np.random.default_rng(88)
    for lanes in (1, 2, 7, 32, 33, 257, 2000):
        t = random_table(rng)
        msg = random_message(rng, t, int(rng.integers(0, 20000)))
        c = ilb.encode_interleaved(msg, t, lanes, BYTE8)
        p, s = oracle.encode_interleaved_u8(msg, t.freq_u32, t.cum_u32, t.scale_bits, lanes)
        assert np.array_equal(c.payload, p) and c.final_states == tuple(s.tolist())
        assert np.array_equal(ilb.decode_interleaved(c), msg)


def test_byte8_truncation_and_lane_decoder_rejects():
    rng = np.random.default_rng(5)
    t = random_table(rng)
    msg = random_message(rng, t, 3000)
    for lanes in (3, 40):
        c = ilb.encode_interleaved(msg, t, lanes, BYTE8)
        c.payload = c.payload[: len(c.payload) // 2]
        with pytest.raises(TruncatedStreamError):
            ilb.decode_interleaved(c)
    c = ilb.encode_interleaved(msg, t, 2, BYTE8)
    with pytest.raises(UnsupportedVariantError, match="unsupported by lane decoder"):
        ilb.decode_lanes_full(c)
    with pytest.raises(UnsupportedVariantError):
        next(decode_lanes_steps(c))


def test_byte8_steps_and_stats():
    rng = np.random.default_rng(9)
    t = random_table(rng, max_n=40, max_sb=14)
    msg = random_message(rng, t, 2005)
    stats = RenormStats()
    c = ilb.encode_interleaved(msg, t, 8, BYTE8, stats=stats)
    out = ilb.decode_interleaved(c, stats=stats)
    assert np.array_equal(out, msg)
    assert stats.encode_symbols == stats.decode_symbols == len(msg)
    assert stats.encode_digits == stats.decode_digits == len(c.payload)
    assert 1 <= stats.max_encode_digits <= 3 and 1 <= stats.max_decode_digits <= 3
    steps = list(decode_interleaved_steps(c))
    assert [s for syms, _, _ in steps for s in syms] == msg.tolist()
    assert steps[-1][1] == (BYTE8.lower_bound,) * 8 and steps[-1][2] == len(c.payload)
    # every group's state snapshot matches the serial oracle run to that point
    f, cum, slot = t.freq_u32, t.cum_u32, t.slot_u8
    for g in (0, 17, len(steps) - 1):
        upto = min(len(msg), (g + 1) * 8)
        _, used, xs = oracle.decode_u8_full(c.payload, c.final_states, slot, f, cum,
                                            t.scale_bits, upto, 8)
        assert steps[g][1] == tuple(int(v) for v in xs) and steps[g][2] == used


# ------------------------------------------------------- chunked byte8 ---
@pytest.mark.parametrize("n, C, lanes", [(0, 1024, 2), (1, 16, 1), (1000, 16, 3),
                                         (70_001, 4096, 2), (300_000, 65536, 32),
                                         (148 * 8 * 2 * 512 + 7, 512, 8)])
def test_chunked_byte8_matches_reference_per_chunk(n, C, lanes):
    """Chunked byte8 (ICH1 variant 0): every chunk's payload and states equal
    the reference's byte8 encode of that chunk alone (oracle restatement of
    interleave.py:155-179), the byte framing packs them back to back, the
    container round-trips through bytes and every chunk re-wraps as a
    standalone IEC1 byte8 container."""
    from paper_1402_3392_b200.chunked import ChunkedContainer, decode_chunked, encode_chunked

    rng = np.random.default_rng(n + C + lanes)
    t = random_table(rng)
    msg = random_message(rng, t, n)
    cc = encode_chunked(msg, t, lanes, C, variant=BYTE8)
    assert cc.variant == BYTE8 and cc.payload.dtype == np.uint8
    k = cc.n_chunks
    for j in range(k):
        chunk = msg[j * C:(j + 1) * C]
        p, s = oracle.encode_interleaved_u8(chunk, t.freq_u32, t.cum_u32, t.scale_bits, lanes)
        a, b = int(cc.word_offsets[j]), int(cc.word_offsets[j + 1])
        assert np.array_equal(cc.payload[a:b], p), j
        assert np.array_equal(cc.states[j], s), j
    back = ChunkedContainer.from_bytes(cc.to_bytes())
    assert back.variant == BYTE8
    assert np.array_equal(decode_chunked(back), msg)
    for j in {0, k - 1} if k else ():
        one = Container.from_bytes(cc.chunk(j).to_bytes())
        assert np.array_equal(ilb.decode_interleaved(one), msg[j * C:(j + 1) * C])


def test_chunked_byte8_device_model_and_errors():
    from paper_1402_3392_b200.chunked import ChunkedContainer, decode_chunked, encode_chunked
    from paper_1402_3392_b200.errors import UnencodableSymbolError

    msg = zipf_1mib()
    cc = encode_chunked(msg, None, 2, 65536, 12, variant=BYTE8)  # config 1 shape, chunked
    counts, alpha = oracle.histogram(msg)
    assert cc.table == SymbolTable(oracle.quantize(counts[:alpha], 12), 12)
    assert np.array_equal(decode_chunked(cc), msg)
    t = SymbolTable([2048, 2047, 0, 1], 12)
    bad = np.zeros(10_000, dtype=np.uint8)
    bad[7777] = 2
    with pytest.raises(UnencodableSymbolError):
        encode_chunked(bad, t, 4, 1024, variant=BYTE8)
    good = encode_chunked(np.zeros(10_000, dtype=np.uint8), t, 4, 1024, variant=BYTE8)
    short = ChunkedContainer(good.lane_count, good.chunk_len, good.message_length, good.table,
                             good.states, good.word_offsets.copy(), good.payload, BYTE8)
    short.word_offsets[-1] -= 1  # last chunk one byte short
    with pytest.raises(TruncatedStreamError):
        decode_chunked(short)


# --------------------------------------------- N = 32 batched fast loops ---
@pytest.mark.parametrize("sb", [8, 12, 13])
def test_byte8_n32_fast_batches_match_oracle(sb):
    """N = 32 byte8 with a fast record table (sb <= 13, every f <= m/2):
    the encoder's 16-group batches (16-byte records, two spill ballots) and
    the decoder's 16-group batches, single stream and chunked, equal the
    reference restatement; f = 1 symbols and a near-m/2 symbol included."""
    from paper_1402_3392_b200.chunked import decode_chunked, encode_chunked

    rng = np.random.default_rng(sb)
    m = 1 << sb
    n_sym = min(60, m // 4)
    freq = [1] * n_sym
    freq[0] = m // 2  # f = m/2: the fast record's bound
    freq[1] += m - sum(freq)
    t = SymbolTable(freq, sb)
    for n in (512 * 37 + 5, 65536 * 3 + 1000):
        msg = random_message(rng, t, n)
        msg[::97] = rng.integers(2, n_sym, size=len(msg[::97]))  # the f = 1 symbols
        c = ilb.encode_interleaved(msg, t, 32, BYTE8)
        p, s = oracle.encode_interleaved_u8(msg, t.freq_u32, t.cum_u32, sb, 32)
        assert np.array_equal(c.payload, p) and c.final_states == tuple(s.tolist())
        assert np.array_equal(ilb.decode_interleaved(c), msg)
        cc = encode_chunked(msg, t, 32, 16384, variant=BYTE8)
        for j in (0, cc.n_chunks - 1):
            chunk = msg[j * 16384:(j + 1) * 16384]
            p, s = oracle.encode_interleaved_u8(chunk, t.freq_u32, t.cum_u32, sb, 32)
            a, b = int(cc.word_offsets[j]), int(cc.word_offsets[j + 1])
            assert np.array_equal(cc.payload[a:b], p) and np.array_equal(cc.states[j], s)
        assert np.array_equal(decode_chunked(cc), msg)


def test_byte8_n32_fast_errors_and_stats():
    """The batched N = 32 loops: a zero-frequency symbol inside a batch names
    the symbol at the highest offending index (the reference walks down);
    a payload cut inside the batched region raises TruncatedStreamError;
    the digit maxima agree between the encode and decode kernels (a
    symbol's spills are its refills)."""
    from paper_1402_3392_b200.errors import UnencodableSymbolError

    t = SymbolTable([2048, 2047, 0, 0, 1], 12)
    msg = np.zeros(70_000, dtype=np.uint8)
    msg[100], msg[60_000] = 2, 3
    with pytest.raises(UnencodableSymbolError, match="symbol 3"):
        ilb.encode_interleaved(msg, t, 32, BYTE8)
    msg[60_000] = 1
    msg[40_000] = 2
    with pytest.raises(UnencodableSymbolError, match="symbol 2"):
        ilb.encode_interleaved(msg, t, 32, BYTE8)
    msg = zipf_1mib()
    counts, alpha = oracle.histogram(msg)
    t = SymbolTable.from_counts(counts[:alpha].tolist(), 12)
    stats = RenormStats()
    c = ilb.encode_interleaved(msg, t, 32, BYTE8, stats=stats)
    assert np.array_equal(ilb.decode_interleaved(c, stats=stats), msg)
    assert stats.max_encode_digits == stats.max_decode_digits == 2
    for cut in (len(c.payload) // 3, len(c.payload) - 1):
        short = Container(c.variant, c.lane_count, c.message_length, c.table, c.final_states,
                          c.payload[:cut])
        with pytest.raises(TruncatedStreamError):
            ilb.decode_interleaved(short)
