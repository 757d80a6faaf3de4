"""Host-side logic that needs no GPU: the C ABI library loads and exports
every declared symbol, wire formats, argument checks, backend resolution,
the division magic used by the encoder, and the synthetic source."""

import re
import subprocess
import sys

import numpy as np
import pytest

import paper_1402_3392_b200 as ilb
from paper_1402_3392_b200 import _lib, backend, rans, synth
from paper_1402_3392_b200.chunked import ChunkedContainer, n_chunks_for
from paper_1402_3392_b200.errors import (
    FormatError,
    TruncatedStreamError,
    UnencodableSymbolError,
    UnsupportedVariantError,
)
from paper_1402_3392_b200.interleave import Container
from paper_1402_3392_b200.rans import BYTE8, WORD16, SymbolTable

from conftest import ROOT


def header_functions():
    text = (ROOT / "include" / "ilans_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ilans_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    names = header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(_lib.lib, name), name  # dlsym succeeds
    assert sorted(_lib.EXPORTED) == names  # every prototype is bound with argtypes
    assert _lib.lib.ilans_abi_version() == 1
    assert _lib.lib.ilans_table_bytes() > 65536


def test_header_is_plain_c_and_links(tmp_path):
    """include/ilans_b200.h is a C ABI: a C11 translation unit that includes
    it compiles and links against libilans_b200.so and runs a host-only
    entry point (no device needed)."""
    so_dir = ilb.__path__[0]
    src = tmp_path / "abi.c"
    src.write_text(
        '#include "ilans_b200.h"\n#include <stdio.h>\n'
        "int main(void) { printf(\"%d %zu\\n\", ilans_abi_version(), ilans_table_bytes());"
        " return 0; }\n")
    exe = tmp_path / "abi"
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", str(ROOT / "include"), str(src),
                    "-L", so_dir, "-lilans_b200", f"-Wl,-rpath,{so_dir}", "-o", str(exe)],
                   check=True, capture_output=True, text=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    assert out[0] == "1" and int(out[1]) == _lib.lib.ilans_table_bytes()


def test_library_is_sm100a():
    so = ilb.__path__[0] + "/libilans_b200.so"
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_fails_loudly():
    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(RuntimeError, match="CUDA"):
        rans.quantize([1, 3], 2)
    with pytest.raises(RuntimeError, match="CUDA"):
        backend.encode_interleaved_u16(np.zeros(4, np.uint8), [4], [0, 4], 2, 1)


def test_golden_container_bytes_parse():
    # pkg/tests/test_interleave.py:68-80 -- host parse of the golden bytes
    blob = (b"IEC1" + b"\x01\x01\x01\x00" + b"\x01" + b"\x00" * 7
            + b"\x02\x02\x00\x01\x00\x03\x00" + b"\x56\x55\x01\x00")
    c = Container.from_bytes(blob)
    assert c.variant == WORD16 and c.lane_count == 1 and c.message_length == 1
    assert c.table == SymbolTable([1, 3], 2)
    assert c.final_states == (87382,) and len(c.payload) == 0
    assert c.to_bytes() == blob
    assert len(blob) == c.header_nbytes + c.payload_nbytes


def test_container_validation():
    blob = bytearray(b"IEC1" + b"\x01\x01\x01\x00" + b"\x01" + b"\x00" * 7
                     + b"\x02\x02\x00\x01\x00\x03\x00" + b"\x56\x55\x01\x00")
    with pytest.raises(FormatError, match="magic"):
        Container.from_bytes(b"NOPE" + b"\x00" * 30)
    b = bytearray(blob); b[4] = 9
    with pytest.raises(FormatError, match="version"):
        Container.from_bytes(bytes(b))
    b = bytearray(blob); b[5] = 7
    with pytest.raises(FormatError, match="variant"):
        Container.from_bytes(bytes(b))
    b = bytearray(blob); b[-4:] = (256).to_bytes(4, "little")
    with pytest.raises(FormatError, match="interval"):
        Container.from_bytes(bytes(b))
    with pytest.raises(TruncatedStreamError):
        Container.from_bytes(bytes(blob[:10]))
    with pytest.raises(TruncatedStreamError):
        Container.from_bytes(bytes(blob[:20]))
    with pytest.raises(FormatError, match="odd"):
        Container.from_bytes(bytes(blob) + b"x")
    b = bytearray(blob); b[6] = 0
    with pytest.raises(FormatError, match="lane_count"):
        Container.from_bytes(bytes(b))


def test_symbol_table_contract():
    t = SymbolTable([1, 3], 2)
    assert t.cum == [0, 1, 4] and t.slot_to_symbol == [0, 1, 1, 1]
    assert t.total == 4 and t.alphabet_size == 2
    assert t.freq_u32.dtype == np.uint32 and t.cum_u32.tolist() == [0, 1, 4]
    assert rans.serialize_table(t) == b"\x02\x02\x00\x01\x00\x03\x00"
    assert rans.parse_table(b"\x02\x02\x00\x01\x00\x03\x00") == (t, 7)
    assert SymbolTable([1, 3], 2) != SymbolTable([1, 3, 0], 2)  # alphabet length matters
    for bad in (([1, 2], 2), ([], 2), ([4], 0), ([4], 17), ([-1, 5], 2), ([1] * 257, 8)):
        with pytest.raises(ValueError):
            SymbolTable(*bad)
    with pytest.raises(FormatError):
        rans.serialize_table(SymbolTable([1 << 16], 16))
    with pytest.raises(FormatError):
        rans.parse_table(b"\x02\x02\x00\x01\x00\x02\x00")
    with pytest.raises(TruncatedStreamError):
        rans.parse_table(b"\x02\x02\x00\x01")
    assert abs(SymbolTable([2, 2], 2).model_entropy_bits() - 1.0) < 1e-12
    assert SymbolTable([1, 3], 2).ideal_bits([0]) == 2.0
    with pytest.raises(UnencodableSymbolError):
        SymbolTable([4, 0], 2).ideal_bits([1])


def test_variants():
    assert WORD16.radix == 1 << 16 and WORD16.state_limit == 1 << 32
    assert BYTE8.lower_bound == 1 << 23
    assert rans.variant_by_tag("word16") is WORD16
    with pytest.raises(ValueError):
        rans.variant_by_tag("nope")
    with pytest.raises(ValueError):
        rans.RenormVariant("bad", 16, 1 << 17)  # radix * L must fit in 32 bits


def test_api_argument_checks_before_device():
    t = SymbolTable([1, 3], 2)
    with pytest.raises(ValueError):
        ilb.encode_interleaved([1], t, 0)
    with pytest.raises(ValueError):
        ilb.encode_interleaved([1], t, 1 << 16)
    with pytest.raises(UnencodableSymbolError):
        ilb.encode_interleaved([5], t, 1)
    toy = rans.RenormVariant("toy-bit", 1, 16)  # custom variants: argument checks on the host
    with pytest.raises(ValueError, match="not a multiple"):
        ilb.encode_interleaved([1], t, 1, rans.RenormVariant("odd", 1, 10))
    with pytest.raises(UnencodableSymbolError):
        ilb.encode_interleaved([7], t, 1, toy)
    c = Container(BYTE8, 2, 1, t, (1 << 23, 1 << 23), np.zeros(0, np.uint8))
    with pytest.raises(UnsupportedVariantError, match="unsupported by lane decoder"):
        ilb.decode_lanes_full(c)
    c = Container(WORD16, 33, 1, t, (1 << 16,) * 33, np.zeros(0, np.uint16))
    with pytest.raises(UnsupportedVariantError, match="at most 32"):
        ilb.decode_lanes_full(c)
    with pytest.raises(ValueError):
        ilb.encode_lanes_full([1], t, 33)


def test_backend_resolution():
    assert backend.get().name == "b200" and backend.get("auto") is backend.ACTIVE
    assert backend.get("ext") is backend.B200
    assert backend.available() == ["b200"]
    with pytest.raises(ValueError, match="unknown backend"):
        backend.get("gpu")
    with pytest.raises(ValueError, match="no CPU fallback"):
        backend.get("pure")
    code = (
        "import warnings\n"
        "with warnings.catch_warnings(record=True) as caught:\n"
        "    warnings.simplefilter('always')\n"
        "    from paper_1402_3392_b200 import backend\n"
        "assert any('ILANS_BACKEND' in str(w.message) for w in caught)\n"
        "assert backend.ACTIVE.name == 'b200'\n"
    )
    env = {"ILANS_BACKEND": "quantum", "PYTHONPATH": str(ROOT)}
    subprocess.run([sys.executable, "-c", code], check=True, env=env)


def _divmagic(d):
    l = (d - 1).bit_length()
    m = ((((1 << l) - d) << 32) // d) + 1
    return m & 0xFFFFFFFF, min(l, 1), max(l - 1, 0)


def test_division_magic_exhaustive_divisors():
    """The encoder's x / f (csrc/common.cuh div_magic) is exact for every
    f in [1, 2^16] on the numerators that matter: all x < 2^32 is too many
    to enumerate per f, so check every f on edge numerators plus random ones,
    and the multiples / neighbours of f where rounding errors would show."""
    rng = np.random.default_rng(0)
    d = np.arange(1, (1 << 16) + 1, dtype=np.uint64)
    mags = np.array([_divmagic(int(x)) for x in d], dtype=np.uint64)
    magic, sh1, sh2 = mags[:, 0], mags[:, 1], mags[:, 2]
    cands = [np.zeros_like(d), np.full_like(d, 2**32 - 1), d - 1, d, d + 1,
             (np.uint64(2**32 - 1) // d) * d, (np.uint64(2**32 - 1) // d) * d - np.uint64(1)]
    cands += [rng.integers(0, 2**32, size=len(d), dtype=np.uint64) for _ in range(24)]
    for n in cands:
        n = n & np.uint64(0xFFFFFFFF)
        t = (magic * n) >> np.uint64(32)
        q = (t + ((n - t) >> sh1)) >> sh2
        assert np.array_equal(q, n // d)


def _encfast(f, cum, sb):
    """common.cuh EncFast::make, restated."""
    m = 1 << sb
    if f == 1:
        return (1 << 32) - 1, 0, cum + m - 1
    c = (f - 1).bit_length()
    return -(-(1 << (31 + c)) // f), c - 1, cum


def test_fast_encoder_record_exact():
    """The fast encoder record (common.cuh EncFast, tables with sb <= 13 and
    every f <= m/2): q = umulhi(x, M) >> s equals x // f (x - 1 for f = 1)
    on every post-spill numerator x < f << (32 - sb) -- edges, the top of
    the range, multiples - 1 and random x, for every f and sb -- and the
    push x + bias + q (m - f) -- and its in-kernel form through the record
    word Z -- and the carry-out spill test agree with the reference formulas
    (_core.pyx:36-41)."""
    rng = np.random.default_rng(1)
    u = np.uint64
    for sb in range(1, 14):
        m, t = 1 << sb, 32 - sb
        for f in range(1, max(1, m // 2) + 1):
            cum = (m - f) // 2  # any cum in [0, m - f]
            M, s, bias = _encfast(f, cum, sb)
            assert (1 << 31) <= M < (1 << 32) and 0 <= s < 32 and bias < (1 << (sb + 1))
            X = f << t
            k = np.arange(1, 400, dtype=np.uint64) * u(f) - u(1)
            xs = np.concatenate([np.arange(max(1, X - 600), X, dtype=np.uint64), k[k < u(X)],
                                 rng.integers(1, X, 600, dtype=np.uint64),
                                 np.array([1, 65536], dtype=np.uint64)])
            xs = xs[(xs >= u(1)) & (xs < u(X))]
            q = ((xs * u(M)) >> u(32)) >> u(s)
            assert np.array_equal(q, xs - u(1) if f == 1 else xs // u(f)), (sb, f)
            x2 = (xs + u(bias) + q * u(m - f)) & u(0xFFFFFFFF)
            assert np.array_equal(x2, (xs // u(f)) * u(m) + xs % u(f) + u(cum)), (sb, f)
            # the record word Z = (m - f) << t | bias << 5 | s and the kernel's
            # forms of the push and of the spill test (encode.cu fast loop)
            Z = (m - f) << t | bias << 5 | s
            assert Z < (1 << 32) and (Z & 31) == s
            x3 = (xs + u(Z >> 5) + u(m - f) * ((q - u(1 << (t - 5))) & u(0xFFFFFFFF))) \
                & u(0xFFFFFFFF)
            assert np.array_equal(x3, x2), (sb, f)
            xx = np.concatenate([np.arange(max(0, X - 3000), min(1 << 32, X + 3000), dtype=np.uint64),
                                 rng.integers(0, 1 << 32, 300, dtype=np.uint64)])
            xm = xx & u(((1 << 32) - 1) ^ ((1 << t) - 1))
            assert np.array_equal(xm + u(Z) >= u(1 << 32), xx >= u(X)), (sb, f)


@pytest.mark.parametrize("sb", [14, 15])
def test_fast_encoder_record12_exact(sb):
    """sb = 14 and 15 take the 12-byte fast record (common.cuh EncFast12):
    Y = f << t | (m - f) gives the spill test (x | (2^t - 1)) >= Y and the
    complement, Z = s | bias << 16 the shift and the bias; checked for every
    f <= m/2 (cum at both ends of its range, so bias = cum + m - 1 of f = 1
    reaches 2m - 2) on edge, top-of-range and random numerators."""
    rng = np.random.default_rng(2)
    u = np.uint64
    m, t = 1 << sb, 32 - sb
    for f in range(1, m // 2 + 1):
        for cum in (m - f, (m - f) // 3):
            M, s, bias = _encfast(f, cum, sb)
            Y, Z = (f << t) | (m - f), s | bias << 16
            assert Z < (1 << 32) and (Z & 31) == s and (Y & ((1 << t) - 1)) == m - f
            X = f << t
            xs = np.concatenate([np.arange(max(1, X - 64), X, dtype=np.uint64),
                                 rng.integers(1, X, 64, dtype=np.uint64)])
            q = ((xs * u(M)) >> u(32)) >> u(Z & 31)
            x2 = (q * u(Y & ((1 << t) - 1)) + xs + u(Z >> 16)) & u(0xFFFFFFFF)
            assert np.array_equal(x2, (xs // u(f)) * u(m) + xs % u(f) + u(cum)), (sb, f)
        xx = np.concatenate([np.arange(max(0, X - 40), X + 40, dtype=np.uint64),
                             rng.integers(0, 1 << 32, 32, dtype=np.uint64)])
        assert np.array_equal((xx | u((1 << t) - 1)) >= u(Y), xx >= u(X)), (sb, f)


@pytest.mark.parametrize("sb", [1, 5, 11, 12, 13, 14, 15, 16])
def test_quad_encoder_record_exact(sb):
    """The 16-byte fast record of the N = 32 encoder (common.cuh EncQuad,
    any sb, every f <= m/2): {M, Y = f << t | s, m - f, bias}. The spill test
    (x | (2^t - 1)) >= Y is x >= f << t, q = umulhi(x, M) >> (Y & 31) is x // f
    (x - 1 for f = 1) and (m - f) q + x + bias is the reference push
    (_core.pyx:36-41) -- for every f at sb <= 13 and for the edges plus a
    sample of f above, cum at both ends of its range, on edge, top-of-range
    and random post-spill numerators."""
    rng = np.random.default_rng(3)
    u = np.uint64
    m, t = 1 << sb, 32 - sb
    fs = np.arange(1, max(1, m // 2) + 1)
    if len(fs) > 4096:
        fs = np.unique(np.concatenate([fs[:512], fs[-512:], rng.choice(fs, 2048, replace=False)]))
    for f in map(int, fs):
        X = f << t
        for cum in (m - f, (m - f) // 3, 0):
            M, s, bias = _encfast(f, cum, sb)
            Y = (f << t) | s
            assert Y < (1 << 32) and (Y & 31) == s and s < (1 << t) - 1
            xs = np.concatenate([np.arange(max(1, X - 64), X, dtype=np.uint64),
                                 rng.integers(1, X, 64, dtype=np.uint64)])
            q = ((xs * u(M)) >> u(32)) >> u(Y & 31)
            x2 = (u(m - f) * q + xs + u(bias)) & u(0xFFFFFFFF)
            assert np.array_equal(x2, (xs // u(f)) * u(m) + xs % u(f) + u(cum)), (sb, f)
        xx = np.concatenate([np.arange(max(0, X - 40), min(1 << 32, X + 40), dtype=np.uint64),
                             rng.integers(0, 1 << 32, 32, dtype=np.uint64)])
        assert np.array_equal((xx | u((1 << t) - 1)) >= u(Y), xx >= u(X)), (sb, f)


@pytest.mark.parametrize("sb", [1, 2, 8, 12, 14, 16])
def test_quadx_encoder_record_exact(sb):
    """The 16-byte record for tables with a symbol above m/2 (common.cuh
    EncQuadX, every f < m): {magic, Y = f << t | l, m - f, cum} with divmagic's
    33-bit magic. (x | 2^t - 1) >= Y is the spill test, q = (umulhi(x, magic)
    + x) >> (Y & 31) (a 33-bit sum) is x // f and (m - f) q + x + cum the
    reference push (_core.pyx:36-41), for f above and below m/2."""
    rng = np.random.default_rng(4)
    u = np.uint64
    m, t = 1 << sb, 32 - sb
    fs = np.arange(1, m)
    if len(fs) > 3000:
        fs = np.unique(np.concatenate([fs[:300], fs[-1500:], rng.choice(fs, 1200, replace=False)]))
    for f in map(int, fs):
        l = (f - 1).bit_length()
        magic = ((1 << (32 + l)) // f) + 1 - (1 << 32)
        Y = (f << t) | l
        assert 0 <= magic < (1 << 32) and Y < (1 << 32) and (Y & 31) == l and Y >= (1 << t)
        X = f << t
        xs = np.concatenate([np.arange(max(0, X - 48), X, dtype=np.uint64),
                             rng.integers(0, X, 48, dtype=np.uint64)])
        q = (((xs * u(magic)) >> u(32)) + xs) >> u(Y & 31)
        assert np.array_equal(q, xs // u(f)), (sb, f)
        for cum in (0, m - f):
            x2 = (u(m - f) * q + xs + u(cum)) & u(0xFFFFFFFF)
            assert np.array_equal(x2, (xs // u(f)) * u(m) + xs % u(f) + u(cum)), (sb, f)
        xx = np.concatenate([np.arange(max(0, X - 40), min(1 << 32, X + 40), dtype=np.uint64),
                             rng.integers(0, 1 << 32, 32, dtype=np.uint64)])
        assert np.array_equal((xx | u((1 << t) - 1)) >= u(Y), xx >= u(X)), (sb, f)


def test_synth_host_deterministic_and_zipf():
    a = synth.synth_host(1 << 16, 1.1, seed=7)
    b = synth.synth_host(1 << 16, 1.1, seed=7)
    c = synth.synth_host(1 << 15, 1.1, seed=7, first=1 << 15)
    assert np.array_equal(a, b) and np.array_equal(a[1 << 15:], c)
    h = np.bincount(a, minlength=256) / len(a)
    assert abs(synth.entropy_bits(h) - synth.entropy_bits(synth.zipf_probs(1.1))) < 0.05


def test_chunked_container_wire_round_trip():
    rng = np.random.default_rng(3)
    t = SymbolTable([1000, 3000, 96], 12)
    n, C, N = 5000, 1024, 4
    k = n_chunks_for(n, C)
    words = rng.integers(0, C, size=k).astype(np.uint64)
    offs = np.zeros(k + 1, np.uint64)
    np.cumsum(words, out=offs[1:])
    cc = ChunkedContainer(N, C, n, t, rng.integers(1 << 16, 1 << 32, size=(k, N), dtype=np.uint64
                                                   ).astype(np.uint32), offs,
                          rng.integers(0, 1 << 16, size=int(offs[-1])).astype(np.uint16))
    back = ChunkedContainer.from_bytes(cc.to_bytes())
    assert back.table == t and back.lane_count == N and back.chunk_len == C
    assert np.array_equal(back.states, cc.states) and np.array_equal(back.payload, cc.payload)
    assert np.array_equal(back.word_offsets, cc.word_offsets)
    one = back.chunk(2)
    assert one.message_length == C and len(one.payload) == int(words[2])
    assert back.chunk(k - 1).message_length == n - (k - 1) * C
    with pytest.raises(FormatError):
        ChunkedContainer.from_bytes(b"IEC1" + cc.to_bytes()[4:])
    with pytest.raises(TruncatedStreamError):
        ChunkedContainer.from_bytes(cc.to_bytes()[:-2])
