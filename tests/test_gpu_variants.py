"""Custom RenormVariants on the B200 (variant.cu): the reference codes every
variant other than word16 / byte8 on its scalar path (interleave.py:155-179
over rans.encode_symbol_renorm / decode_symbol_renorm). The B200 coder
must give byte-identical payloads, final states, decoded bytes, step traces,
renorm statistics and errors; the reference itself (oracle/_ref) is run
beside it as the checker."""

import sys
from pathlib import Path

import numpy as np
import pytest

import oracle
import paper_1402_3392_b200 as ilb
from paper_1402_3392_b200 import _lib
from paper_1402_3392_b200.errors import (
    FormatError,
    TruncatedStreamError,
    UnencodableSymbolError,
)
from paper_1402_3392_b200.interleave import Container, decode_interleaved_steps
from paper_1402_3392_b200.rans import RenormStats, RenormVariant, SymbolTable

pytestmark = pytest.mark.gpu
REF = Path(__file__).resolve().parents[1] / "oracle" / "_ref"


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if _lib.device_count() == 0:
        pytest.fail("no CUDA device: the -m gpu suite must run on a B200")


@pytest.fixture(scope="module")
def ref():
    if not (REF / "ilans").exists():
        pytest.skip("oracle/_ref not built")
    sys.path.insert(0, str(REF))
    import ilans

    return ilans


def cases():
    # (digit_bits, lower_bound exponent-or-value, scale_bits): powers of two
    # and L = 3 * 2^sb (refill counts then depend on the digits read)
    return [(1, 16, 2), (1, 1 << 12, 8), (4, 1 << 20, 12), (12, 1 << 20, 10), (3, 3 << 12, 12),
            (5, 5 << 10, 10), (16, 1 << 14, 14), (7, 1 << 24, 11), (2, 3 << 8, 8)]


def test_custom_variants_match_the_reference(ref):
    rng = np.random.default_rng(21)
    for bits, low, sb in cases():
        v = RenormVariant(f"v{bits}", bits, low)
        rv = ref.rans.RenormVariant(f"v{bits}", bits, low)
        for lanes in (1, 2, 5, 32, 40):
            n_sym = int(rng.integers(2, min(40, 1 << sb) + 1))
            counts = rng.integers(0, 500, size=n_sym)
            counts[0] += 1
            t = SymbolTable(oracle.quantize(counts, sb), sb)
            rt = ref.rans.SymbolTable(list(t.freq), sb)
            msg = rng.choice(n_sym, size=int(rng.integers(0, 3000)),
                             p=t.freq_u32 / t.total).astype(np.uint8)
            st, rst = RenormStats(), ref.rans.RenormStats()
            c = ilb.encode_interleaved(msg, t, lanes, v, stats=st)
            rc = ref.interleave.encode_interleaved(msg, rt, lanes, rv, stats=rst)
            assert c.final_states == tuple(rc.final_states), (bits, low, sb, lanes)
            assert np.array_equal(c.payload, rc.payload), (bits, low, sb, lanes)
            assert c.payload.dtype == rc.payload.dtype
            out = ilb.decode_interleaved(c, stats=st)
            ref.interleave.decode_interleaved(rc, stats=rst)
            assert np.array_equal(out, msg)
            assert (st.encode_symbols, st.encode_digits, st.max_encode_digits,
                    st.decode_symbols, st.decode_digits, st.max_decode_digits) == (
                rst.encode_symbols, rst.encode_digits, rst.max_encode_digits,
                rst.decode_symbols, rst.decode_digits, rst.max_decode_digits)
            steps = list(decode_interleaved_steps(c))
            rsteps = list(ref.interleave.decode_interleaved_steps(rc))
            assert steps == rsteps


def test_toy_golden_recast(ref):
    """Reference test_interleave.py TestGolden::test_single_lane_recast_toy:
    a 1-lane container of "babba" under the 1-bit toy variant equals the
    generic framework's encoder (here: the reference run beside it)."""
    toy = RenormVariant("toy-bit", 1, 16)
    t = SymbolTable([1, 3], 2)
    babba = [1, 0, 1, 1, 0]
    c = ilb.encode_interleaved(babba, t, 1, toy)
    rc = ref.interleave.encode_interleaved(babba, ref.rans.SymbolTable([1, 3], 2), 1,
                                           ref.rans.RenormVariant("toy-bit", 1, 16))
    assert c.final_states == tuple(rc.final_states) == (19,)
    assert c.payload.tolist() == rc.payload.tolist() == [0, 1, 0, 0, 0]
    assert ilb.decode_interleaved(c).tolist() == babba
    with pytest.raises(FormatError):  # custom variants have no wire encoding
        c.to_bytes()


def test_custom_variant_errors():
    v = RenormVariant("v4", 4, 1 << 12)
    t = SymbolTable([4, 0, 4], 3)
    with pytest.raises(UnencodableSymbolError):
        ilb.encode_interleaved([0, 1, 2], t, 2, v)
    t2 = SymbolTable([5, 3], 3)
    msg = np.array([0, 1] * 300, dtype=np.uint8)
    c = ilb.encode_interleaved(msg, t2, 3, v)
    c2 = Container(c.variant, c.lane_count, c.message_length, c.table, c.final_states,
                   c.payload[: len(c.payload) // 2])
    with pytest.raises(TruncatedStreamError):
        ilb.decode_interleaved(c2)
    gen = decode_interleaved_steps(c2)
    with pytest.raises(TruncatedStreamError):
        for _ in gen:
            pass
