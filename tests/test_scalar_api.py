"""Scalar per-symbol API (host helpers, no GPU): rans.push_symbol /
pop_symbol / encode_symbol_renorm / decode_symbol_renorm / rans_coder
(reference rans.py:214-329), the raw-bit bypass (interleave.py:271-298) and
the mux's per-symbol stream decoders (mux.py:100-163). The known answers
are the reference suite's (test_rans.py:90-145, test_interleave.py:259-336)
and the cross-checks run the reference itself (oracle/_ref) when built."""

import sys
from pathlib import Path

import numpy as np
import pytest

from paper_1402_3392_b200 import mux, rans
from paper_1402_3392_b200.errors import FormatError, TruncatedStreamError
from paper_1402_3392_b200.interleave import DigitReader, decode_raw_bits, encode_raw_bits
from paper_1402_3392_b200.rans import BYTE8, WORD16, RenormStats, RenormVariant, SymbolTable

TOY = RenormVariant("toy-bit", 1, 16)
REF = Path(__file__).resolve().parents[1] / "oracle" / "_ref"


def toy_table():
    return SymbolTable([1, 3], scale_bits=2)


def random_table(rng, max_n=100, max_scale=14):
    import oracle

    n = int(rng.integers(2, max_n + 1))
    sb = int(rng.integers(max(1, (n - 1).bit_length()), max_scale + 1))
    counts = rng.integers(0, 800, size=n)
    counts[int(rng.integers(0, n))] += 1
    return SymbolTable(oracle.quantize(counts, sb), sb)


def test_push_pop_known_answers():
    assert rans.push_symbol(toy_table(), 1, 16) == 22
    assert rans.pop_symbol(toy_table(), 19) == (1, 14)


def test_golden_renorm_steps():
    sink = []
    assert rans.encode_symbol_renorm(28, 1, toy_table(), TOY, sink) == 19
    assert sink == [0]
    assert rans.decode_symbol_renorm(19, toy_table(), TOY, DigitReader([0])) == (1, 28)
    with pytest.raises(TruncatedStreamError):
        rans.decode_symbol_renorm(19, toy_table(), TOY, DigitReader([]))


def test_word16_single_spill_at_extremes():
    table = SymbolTable([1] + [0] * 254 + [(1 << 14) - 1], 14)
    sink = []
    state = rans.encode_symbol_renorm((1 << 32) - 1, 0, table, WORD16, sink)
    assert sink == [0xFFFF]
    assert WORD16.lower_bound <= state < WORD16.state_limit


def test_round_trip_both_variants():
    rng = np.random.default_rng(11)
    for variant, max_spill in ((WORD16, 1), (BYTE8, 3)):
        for _ in range(10):
            table = random_table(rng)
            msg = rng.choice(table.alphabet_size, size=400, p=table.freq_u32 / table.total).tolist()
            stats = RenormStats()
            state, sink = variant.lower_bound, []
            for s in reversed(msg):
                state = rans.encode_symbol_renorm(state, s, table, variant, sink, stats)
            reader = DigitReader(sink[::-1])
            out = []
            for _ in msg:
                s, state = rans.decode_symbol_renorm(state, table, variant, reader, stats)
                out.append(s)
            assert out == msg and state == variant.lower_bound and reader.exhausted()
            assert stats.max_encode_digits <= max_spill and stats.max_decode_digits <= max_spill


def test_rans_coder_fields():
    c = rans.rans_coder(toy_table(), TOY)
    assert (c.alphabet_size, c.lower_bound, c.radix) == (2, 16, 2)
    assert c.code(1, 16) == 22 and c.decode(19) == (1, 14)
    assert c.in_interval(16) and not c.in_interval(32)


def test_raw_bits_bypass_round_trip_and_validation():
    rng = np.random.default_rng(30)
    table = toy_table()
    msg = rng.integers(0, 2, size=200).tolist()
    sub = {i: int(rng.integers(0, 4)) for i, s in enumerate(msg) if s == 0}
    stack, state = [], WORD16.lower_bound
    for i in range(len(msg) - 1, -1, -1):
        if msg[i] == 0:
            encode_raw_bits(sub[i], 2, stack, WORD16)
        state = rans.encode_symbol_renorm(state, msg[i], table, WORD16, stack)
    reader = DigitReader(stack[::-1])
    got, got_sub = [], {}
    for i in range(len(msg)):
        s, state = rans.decode_symbol_renorm(state, table, WORD16, reader)
        got.append(s)
        if s == 0:
            got_sub[i] = decode_raw_bits(2, reader, WORD16)
    assert got == msg and got_sub == sub and reader.exhausted()
    stack = []
    encode_raw_bits(0, 0, stack, WORD16)
    assert stack == [] and decode_raw_bits(0, DigitReader([]), WORD16) == 0
    with pytest.raises(ValueError):
        encode_raw_bits(4, 2, [], WORD16)
    with pytest.raises(ValueError):
        encode_raw_bits(1, 17, [], WORD16)
    with pytest.raises(ValueError):
        encode_raw_bits(1, 2, [], TOY)
    with pytest.raises(FormatError):
        decode_raw_bits(2, DigitReader([9]), WORD16)
    with pytest.raises(TruncatedStreamError):
        decode_raw_bits(2, DigitReader([]), WORD16)


def test_mux_stream_decoders():
    t = toy_table()
    d = mux.RansStreamCodec(t, WORD16).new_decoder()
    # a segment coded by hand with the scalar helpers: [state LE u32][digits LE u16]
    msg = [1, 0, 1, 1, 0, 0, 1]
    state, digits = WORD16.lower_bound, []
    for s in reversed(msg):
        state = rans.encode_symbol_renorm(state, s, t, WORD16, digits)
    raw = state.to_bytes(4, "little") + b"".join(x.to_bytes(2, "little") for x in digits[::-1])
    pos = [0]

    def read(k):
        b = raw[pos[0]:pos[0] + k]
        pos[0] += k
        return b

    d.load_state(read)
    assert [d.decode_symbol(read) for _ in msg] == msg and pos[0] == len(raw)
    with pytest.raises(FormatError):
        d.load_state(lambda k: (1).to_bytes(4, "little"))
    r = mux.RawStreamCodec(12).new_decoder()
    r.load_state(read)
    assert r.decode_symbol(lambda k: (0xABC).to_bytes(k, "little")) == 0xABC


@pytest.mark.skipif(not (REF / "ilans").exists(), reason="oracle/_ref not built")
def test_scalar_helpers_match_the_reference():
    sys.path.insert(0, str(REF))
    from ilans import rans as ref_rans

    rng = np.random.default_rng(5)
    for _ in range(20):
        t = random_table(rng)
        rt = ref_rans.SymbolTable(list(t.freq), t.scale_bits)
        for variant, rv in ((WORD16, ref_rans.WORD16), (BYTE8, ref_rans.BYTE8)):
            for _ in range(50):
                x = int(rng.integers(variant.lower_bound, variant.state_limit))
                s = int(rng.choice(t.alphabet_size, p=t.freq_u32 / t.total))
                a, b = [], []
                assert rans.encode_symbol_renorm(x, s, t, variant, a) == \
                    ref_rans.encode_symbol_renorm(x, s, rt, rv, b)
                assert a == b
                assert rans.pop_symbol(t, x) == ref_rans.pop_symbol(rt, x)
