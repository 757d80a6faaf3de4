"""rANS model objects: renorm variants, the quantized symbol table, quantize.

API-compatible with the reference module (pkg/src/ilans/rans.py). The
numeric work -- quantize (rans.py:171-211) and, in the chunked pipeline,
the histogram and every lookup table -- runs on the B200 through
libilans_b200.so. SymbolTable keeps the reference's host-side fields
(freq / cum lists, slot view) because callers read them; the device builds
its own tables from the same frequencies.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass
from functools import cached_property

import numpy as np

from . import _lib
from .errors import FormatError, TruncatedStreamError, UnencodableSymbolError

MAX_ALPHABET = 256
MAX_SCALE_BITS = 16

__all__ = [
    "RenormVariant",
    "BYTE8",
    "WORD16",
    "SymbolTable",
    "quantize",
    "encode_threshold",
    "RenormStats",
    "serialize_table",
    "parse_table",
    "variant_by_tag",
]


@dataclass(frozen=True)
class RenormVariant:
    """Digit width plus the lower bound L of the normalized state interval
    (reference rans.py:45-83). The B200 kernels implement WORD16 (16-bit
    digits, L = 2^16), where one spill / refill per symbol always suffices."""

    tag: str
    digit_bits: int
    lower_bound: int

    def __post_init__(self):
        if not 1 <= self.digit_bits <= 16:
            raise ValueError("digit_bits must be in [1, 16]")
        if self.lower_bound < 1:
            raise ValueError("lower_bound must be >= 1")
        if (1 << self.digit_bits) * self.lower_bound > 1 << 32:
            raise ValueError("radix * lower_bound must fit in 32 bits")

    @property
    def radix(self) -> int:
        return 1 << self.digit_bits

    @property
    def digit_mask(self) -> int:
        return self.radix - 1

    @property
    def state_limit(self) -> int:
        return self.radix * self.lower_bound

    def check_table(self, table: "SymbolTable") -> None:
        if self.lower_bound % table.total:
            raise ValueError(
                f"lower_bound {self.lower_bound} is not a multiple of the table total "
                f"{table.total}; renormalized coding would not be b-unique"
            )


BYTE8 = RenormVariant("byte8", 8, 1 << 23)
WORD16 = RenormVariant("word16", 16, 1 << 16)
_BY_TAG = {v.tag: v for v in (BYTE8, WORD16)}


def variant_by_tag(tag: str) -> RenormVariant:
    if tag not in _BY_TAG:
        raise ValueError(f"unknown renorm variant {tag!r}")
    return _BY_TAG[tag]


def quantize(counts, scale_bits: int) -> list[int]:
    """Counts -> integer frequencies summing to 2**scale_bits, bit-identical
    to the reference largest-remainder quantizer (rans.py:171-211), computed
    by the device model builder (csrc/table.cu, build_table_kernel)."""
    counts = [int(c) for c in counts]
    if not 1 <= scale_bits <= MAX_SCALE_BITS:
        raise ValueError(f"scale_bits must be in [1, {MAX_SCALE_BITS}]")
    if len(counts) > MAX_ALPHABET:
        raise ValueError(f"alphabet size must be <= {MAX_ALPHABET}")
    if any(c < 0 for c in counts):
        raise ValueError("counts must be non-negative")
    if any(c >= 1 << 64 for c in counts):
        raise ValueError("counts must fit in 64 bits")
    arr = np.ascontiguousarray(counts, dtype=np.uint64)
    out = np.zeros(max(1, len(counts)), dtype=np.uint32)
    st = _lib.Status()
    rc = _lib.lib.ilans_quantize(_lib.ptr(arr), len(counts), scale_bits, _lib.ptr(out),
                                 _lib.ctypes.byref(st))
    _lib.raise_for(rc, st, "quantize")
    return out[: len(counts)].tolist()


class SymbolTable:
    """Quantized frequencies plus cumulative offsets and slot lookup
    (reference rans.py:99-168). Equality is (scale_bits, freq list)."""

    def __init__(self, freqs, scale_bits: int):
        if not 1 <= scale_bits <= MAX_SCALE_BITS:
            raise ValueError(f"scale_bits must be in [1, {MAX_SCALE_BITS}]")
        freqs = [int(f) for f in freqs]
        if not 1 <= len(freqs) <= MAX_ALPHABET:
            raise ValueError(f"alphabet size must be in [1, {MAX_ALPHABET}]")
        if min(freqs) < 0:
            raise ValueError("frequencies must be non-negative")
        if sum(freqs) != 1 << scale_bits:
            raise ValueError(f"frequencies must sum to {1 << scale_bits}, got {sum(freqs)}")
        self.scale_bits = scale_bits
        self.freq = freqs
        self.cum = [0, *np.cumsum(freqs).tolist()]

    @classmethod
    def from_counts(cls, counts, scale_bits: int = 14) -> "SymbolTable":
        return cls(quantize(counts, scale_bits), scale_bits)

    @property
    def total(self) -> int:
        return 1 << self.scale_bits

    @property
    def alphabet_size(self) -> int:
        return len(self.freq)

    @cached_property
    def freq_u32(self) -> np.ndarray:
        return np.asarray(self.freq, dtype=np.uint32)

    @cached_property
    def cum_u32(self) -> np.ndarray:
        return np.asarray(self.cum, dtype=np.uint32)

    @cached_property
    def slot_u8(self) -> np.ndarray:
        """Dense slot -> symbol view (rans.py:119-121) passed to decode calls."""
        return np.repeat(np.arange(self.alphabet_size, dtype=np.uint8), self.freq_u32)

    @property
    def slot_to_symbol(self) -> list[int]:
        return self.slot_u8.tolist()

    def model_entropy_bits(self) -> float:
        """Entropy of the quantized distribution, bits per symbol."""
        f = self.freq_u32[self.freq_u32 > 0].astype(np.float64) / self.total
        return float(-(f * np.log2(f)).sum())

    def ideal_bits(self, symbols) -> float:
        """Sum of -log2(f_s / m) over a message (rans.py:153-158)."""
        f = self.freq_u32[np.asarray(symbols, dtype=np.uint8)].astype(np.float64)
        if (f == 0).any():
            raise UnencodableSymbolError("message contains zero-frequency symbols")
        return float((self.scale_bits - np.log2(f)).sum())

    def __eq__(self, other):
        return (
            isinstance(other, SymbolTable)
            and self.scale_bits == other.scale_bits
            and self.freq == other.freq
        )

    __hash__ = None

    def __repr__(self):
        return f"SymbolTable(n={self.alphabet_size}, scale_bits={self.scale_bits})"


class RenormStats:
    """Spill / refill counters (reference rans.py:235-263). The B200 path
    fills them from the kernels: symbol and digit totals, and the most
    digits one symbol moved, measured by the instrumented kernel calls
    (ilans_*_u16_stats; byte8 always reports it)."""

    def __init__(self):
        self.encode_symbols = 0
        self.encode_digits = 0
        self.max_encode_digits = 0
        self.decode_symbols = 0
        self.decode_digits = 0
        self.max_decode_digits = 0

    def note_encode(self, digits: int) -> None:
        self.encode_symbols += 1
        self.encode_digits += digits
        self.max_encode_digits = max(self.max_encode_digits, digits)

    def note_decode(self, digits: int) -> None:
        self.decode_symbols += 1
        self.decode_digits += digits
        self.max_decode_digits = max(self.max_decode_digits, digits)

    def __repr__(self):
        return (
            f"RenormStats(enc {self.encode_symbols} syms / {self.encode_digits} digits, "
            f"max {self.max_encode_digits}; dec {self.decode_symbols} syms / "
            f"{self.decode_digits} digits, max {self.max_decode_digits})"
        )


def encode_threshold(table: SymbolTable, variant: RenormVariant, symbol: int) -> int:
    """Exclusive upper state bound before pushing ``symbol`` (rans.py:229-232)."""
    return table.freq[symbol] * (variant.state_limit >> table.scale_bits)


# ---------------------------------------------------------------------------
# Scalar per-symbol helpers (reference rans.py:214-329). These are the
# reference's building blocks for custom coders (raw-bit bypass, the mux's
# per-stream decoders, user code): one exact integer state transition per
# call on Python ints. No bulk path of this package calls them -- message
# coding runs in the B200 kernels -- and they are tested against the
# reference's own known answers (tests/test_host.py).
# ---------------------------------------------------------------------------
def push_symbol(table: SymbolTable, symbol: int, state: int) -> int:
    """Bare rANS push, no renormalisation (rans.py:214-219)."""
    f = table.freq[symbol]
    if f == 0:
        raise UnencodableSymbolError(f"symbol {symbol} has frequency 0")
    q, r = divmod(state, f)
    return (q << table.scale_bits) + table.cum[symbol] + r


def pop_symbol(table: SymbolTable, state: int) -> tuple[int, int]:
    """Bare rANS pop, no renormalisation (rans.py:222-226)."""
    slot = state & (table.total - 1)
    symbol = table.slot_to_symbol[slot]
    return symbol, table.freq[symbol] * (state >> table.scale_bits) + slot - table.cum[symbol]


def encode_symbol_renorm(state: int, symbol: int, table: SymbolTable, variant: RenormVariant,
                         sink: list, stats: RenormStats | None = None) -> int:
    """Spill digits to ``sink`` (emission order) until ``state`` is below the
    symbol's threshold f * (state_limit >> sb), then push (rans.py:266-290)."""
    f = table.freq[symbol]
    if f == 0:
        raise UnencodableSymbolError(f"symbol {symbol} has frequency 0")
    limit = f * (variant.state_limit >> table.scale_bits)
    spilled = 0
    while state >= limit:
        sink.append(state & variant.digit_mask)
        state >>= variant.digit_bits
        spilled += 1
    if stats is not None:
        stats.note_encode(spilled)
    return push_symbol(table, symbol, state)


def decode_symbol_renorm(state: int, table: SymbolTable, variant: RenormVariant, source,
                         stats: RenormStats | None = None) -> tuple[int, int]:
    """Pop one symbol, then refill digits from ``source`` (anything with
    ``.read()``) until the state is back in [L, R*L) (rans.py:293-314)."""
    symbol, state = pop_symbol(table, state)
    low = variant.lower_bound
    # a valid pop never lands on 0; more refills than a state has digits
    # (+ 2) only happen on corrupt input
    max_refills = (low.bit_length() + variant.digit_bits - 1) // variant.digit_bits + 2
    refills = 0
    while state < low:
        state = (state << variant.digit_bits) | source.read()
        refills += 1
        if refills > max_refills:
            raise FormatError("renormalization does not terminate; corrupt stream")
    if stats is not None:
        stats.note_decode(refills)
    return symbol, state


@dataclass(frozen=True)
class Coder:
    """A code / decode pair with its normalisation interval -- the fields of
    the reference's generic ``ans.Coder`` (ans.py:41-67) that rans_coder
    fills; the generic teaching framework itself is out of scope."""

    alphabet_size: int
    code: object
    decode: object
    lower_bound: int
    radix: int

    def __post_init__(self):
        if self.radix < 2:
            raise ValueError("radix must be >= 2")
        if self.lower_bound < 1:
            raise ValueError("lower_bound must be >= 1")
        if self.alphabet_size < 1:
            raise ValueError("alphabet_size must be >= 1")

    def in_interval(self, state: int) -> bool:
        return self.lower_bound <= state < self.radix * self.lower_bound

    @property
    def max_digits_per_symbol(self) -> int:
        # a normalised state reaches 0 after this many divisions by radix
        # (ans.py:64-67), so no symbol can need more spills
        return math.ceil(math.log(self.radix * self.lower_bound, self.radix)) + 1


def rans_coder(table: SymbolTable, variant: RenormVariant) -> Coder:
    """A table + variant as a Coder (rans.py:317-329)."""
    variant.check_table(table)
    return Coder(alphabet_size=table.alphabet_size,
                 code=lambda s, x: push_symbol(table, s, x),
                 decode=lambda x: pop_symbol(table, x),
                 lower_bound=variant.lower_bound, radix=variant.radix)


def serialize_table(table: SymbolTable) -> bytes:
    """scale_bits u8, alphabet u16 LE, then u16 LE frequencies (rans.py:332-338)."""
    if max(table.freq) > 0xFFFF:
        raise FormatError("frequency 65536 does not fit the u16 table field")
    return struct.pack("<BH", table.scale_bits, table.alphabet_size) + table.freq_u32.astype(
        "<u2"
    ).tobytes()


def parse_table(buf: bytes, offset: int = 0) -> tuple[SymbolTable, int]:
    """Inverse of serialize_table (rans.py:341-355)."""
    if len(buf) < offset + 3:
        raise TruncatedStreamError("table header truncated")
    scale_bits, n = struct.unpack_from("<BH", buf, offset)
    offset += 3
    if len(buf) < offset + 2 * n:
        raise TruncatedStreamError("frequency table truncated")
    freqs = np.frombuffer(buf, dtype="<u2", count=n, offset=offset).tolist()
    offset += 2 * n
    try:
        table = SymbolTable(freqs, scale_bits)
    except ValueError as exc:
        raise FormatError(f"invalid frequency table: {exc}") from exc
    return table, offset
