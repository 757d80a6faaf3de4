"""Multiplexing of independently coded streams (reference pkg/src/ilans/mux.py).

Same names, wire format (IEM1) and exceptions as the reference. The
reference builds the muxed payload by running one decoder per stream along
the schedule and teeing every byte it reads; here the B200 computes the same
byte order directly (libilans_b200.so ``ilans_mux_*``, csrc/mux.cu):

* ``mux_with_flush`` / ``encode_multistream`` -- every segment is coded by
  its own device thread, each symbol's byte count comes from the encoder
  (the digits spilled while pushing a symbol are the ones refilled after
  popping it), a stable sort of the schedule plus an exclusive scan give
  every step's offset, and one thread per symbol copies its bytes there;
* ``mux`` (pre-encoded buffers) -- one device thread per stream replays its
  decoder over its own payload for the per-symbol counts, then the same
  scan + scatter;
* ``demux_decode`` -- sequential by construction (each step's read offset
  depends on every earlier step's read size), but consecutive steps on
  distinct streams decode together: one warp walks the schedule in windows
  of up to 32 steps.

Streams are ``RansStreamCodec`` (rANS over a SymbolTable, byte-multiple
digits: BYTE8, WORD16 or a custom RenormVariant with 8/16-bit digits) or
``RawStreamCodec`` (fixed-width little-endian values). The reference's
coder interface is duck-typed (any object with encode_segment /
new_decoder); the B200 kernels know these two coder types, so other coder
types raise TypeError. ``new_decoder()`` returns the reference's per-symbol
scalar decoders (host helpers; containers decode on the GPU).
"""

from __future__ import annotations

import ctypes
import struct
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import (
    FormatError,
    ScheduleError,
    TrailingGarbageWarning,
    TruncatedStreamError,
    UnencodableSymbolError,
)
from .rans import WORD16, RenormVariant, SymbolTable

MUX_MAGIC = b"IEM1"
MUX_VERSION = 1
_FIXED = struct.Struct("<BIH")     # version, flush interval (0 = none), stream count
_PREAMBLE = struct.Struct("<QH")   # symbol count, header length
_PLEN = struct.Struct("<Q")

__all__ = [
    "RansStreamCodec",
    "RawStreamCodec",
    "StreamBuffer",
    "MuxedContainer",
    "MuxBudget",
    "round_robin_schedule",
    "encode_multistream",
    "mux",
    "mux_with_flush",
    "demux_decode",
    "MUX_MAGIC",
]


# ------------------------------------------------------------ stream coders
class RansStreamCodec:
    """rANS stream coder (reference mux.py:82-104): segments start from
    x = L, the final state is the segment's 4-byte LE state, digits are
    little-endian ``digit_bits / 8``-byte groups in read order."""

    def __init__(self, table: SymbolTable, variant: RenormVariant = WORD16):
        if variant.digit_bits % 8:
            raise ValueError("mux streams need byte-multiple digit widths")
        variant.check_table(table)
        self.table = table
        self.variant = variant
        self.digit_nbytes = variant.digit_bits // 8

    def encode_segment(self, symbols) -> tuple[bytes, bytes]:
        """One segment from a fresh state: (state bytes, payload bytes)."""
        (buf,) = encode_multistream([symbols], [self])
        return buf.header, buf.payload

    def new_decoder(self):
        """Per-symbol decoder of this stream's segments (reference
        mux.py:100-128): load_state(read) / decode_symbol(read), the
        duck-typed interface of the reference's coder objects. A scalar host
        helper for callers that walk a schedule themselves; demux_decode
        decodes whole containers on the B200."""
        return _RansStreamDecoder(self)


class _RansStreamDecoder:
    def __init__(self, codec: RansStreamCodec):
        self._codec = codec
        self._state = None

    def load_state(self, read) -> None:
        state = int.from_bytes(read(4), "little")
        v = self._codec.variant
        if not v.lower_bound <= state < v.state_limit:
            raise FormatError(f"stream state {state} outside the coder interval")
        self._state = state

    def decode_symbol(self, read) -> int:
        from .rans import pop_symbol

        c = self._codec
        low, bits, nb = c.variant.lower_bound, c.variant.digit_bits, c.digit_nbytes
        symbol, state = pop_symbol(c.table, self._state)
        while state < low:
            state = (state << bits) | int.from_bytes(read(nb), "little")
        self._state = state
        return symbol


class RawStreamCodec:
    """Uncompressed fixed-width values, no coding state (reference
    mux.py:131-163)."""

    def __init__(self, width_bits: int):
        if not 1 <= width_bits <= 32:
            raise ValueError("width_bits must be in [1, 32]")
        self.width_bits = width_bits
        self.value_nbytes = (width_bits + 7) // 8

    def encode_segment(self, values) -> tuple[bytes, bytes]:
        (buf,) = encode_multistream([values], [self])
        return buf.header, buf.payload

    def new_decoder(self):
        """Per-value decoder (reference mux.py:150-163); stateless."""
        return _RawStreamDecoder(self.value_nbytes)


class _RawStreamDecoder:
    def __init__(self, nbytes: int):
        self._nbytes = nbytes

    def load_state(self, read) -> None:
        pass  # stateless: reloading at a segment boundary costs nothing

    def decode_symbol(self, read) -> int:
        return int.from_bytes(read(self._nbytes), "little")


# ------------------------------------------------------------ containers
@dataclass
class StreamBuffer:
    """One stream encoded on its own: preamble header + private payload."""

    header: bytes
    payload: bytes
    symbol_count: int


@dataclass
class MuxedContainer:
    """IEM1: magic, version u8, flush interval u32 (0 = none), stream count
    u16, per stream (symbol count u64, header length u16, header), payload
    length u64, payload; little-endian (reference mux.py:175-232)."""

    flush_interval: int | None
    stream_lengths: list[int]
    stream_headers: list[bytes]
    payload: bytes

    def to_bytes(self) -> bytes:
        parts = [MUX_MAGIC, _FIXED.pack(MUX_VERSION, self.flush_interval or 0,
                                        len(self.stream_lengths))]
        for n, header in zip(self.stream_lengths, self.stream_headers):
            parts.append(_PREAMBLE.pack(n, len(header)))
            parts.append(bytes(header))
        parts.append(_PLEN.pack(len(self.payload)))
        parts.append(bytes(self.payload))
        return b"".join(parts)

    @classmethod
    def from_bytes(cls, raw: bytes) -> "MuxedContainer":
        raw = bytes(raw)
        head = len(MUX_MAGIC) + _FIXED.size
        if len(raw) < head:
            raise TruncatedStreamError("mux container shorter than fixed header")
        if raw[: len(MUX_MAGIC)] != MUX_MAGIC:
            raise FormatError("bad magic; not an ilans mux container")
        version, flush, count = _FIXED.unpack_from(raw, len(MUX_MAGIC))
        if version != MUX_VERSION:
            raise FormatError(f"unsupported mux container version {version}")
        pos = head
        lengths: list[int] = []
        headers: list[bytes] = []
        for _ in range(count):
            if pos + _PREAMBLE.size > len(raw):
                raise TruncatedStreamError("stream preamble truncated")
            n, hlen = _PREAMBLE.unpack_from(raw, pos)
            pos += _PREAMBLE.size
            if pos + hlen > len(raw):
                raise TruncatedStreamError("stream header truncated")
            lengths.append(n)
            headers.append(raw[pos: pos + hlen])
            pos += hlen
        if pos + _PLEN.size > len(raw):
            raise TruncatedStreamError("payload length truncated")
        (plen,) = _PLEN.unpack_from(raw, pos)
        pos += _PLEN.size
        if pos + plen > len(raw):
            raise TruncatedStreamError("muxed payload truncated")
        extra = len(raw) - pos - plen
        if extra:
            warnings.warn(f"{extra} bytes after muxed payload", TrailingGarbageWarning,
                          stacklevel=2)
        return cls(flush or None, lengths, headers, raw[pos: pos + plen])


@dataclass
class MuxBudget:
    """Encoder-side buffering report from mux_with_flush."""

    flush_interval: int | None
    max_buffered: int
    segment_count: int
    payload_bytes: int


# ------------------------------------------------------------ schedules
def round_robin_schedule(lengths) -> list[int]:
    """Cycle over the streams, skipping exhausted ones (reference
    mux.py:244-256): step order is (round, stream)."""
    n = np.asarray([int(x) for x in lengths], dtype=np.int64)
    if n.size == 0 or n.sum() == 0:
        return []
    sid = np.repeat(np.arange(n.size, dtype=np.int64), np.maximum(n, 0))
    starts = np.repeat(np.cumsum(np.maximum(n, 0)) - np.maximum(n, 0), np.maximum(n, 0))
    rnd = np.arange(sid.size, dtype=np.int64) - starts
    return sid[np.lexsort((sid, rnd))].tolist()


def _schedule_array(schedule) -> np.ndarray:
    if not isinstance(schedule, (np.ndarray, list, tuple)):
        schedule = list(schedule)
    return np.asarray(schedule, dtype=np.int64).reshape(-1)


def _validate_schedule(schedule, lengths) -> np.ndarray:
    """Every id names a stream and every stream gets exactly its symbol
    count (reference mux.py:259-269, same messages and order)."""
    sched = _schedule_array(schedule)
    k = len(lengths)
    unknown = (sched < 0) | (sched >= k)
    if unknown.any():
        raise ScheduleError(f"schedule references unknown stream {int(sched[unknown][0])}")
    counts = np.bincount(sched, minlength=k) if sched.size else np.zeros(k, np.int64)
    for j, n in enumerate(lengths):
        if int(counts[j]) != int(n):
            raise ScheduleError(
                f"schedule has {int(counts[j])} steps for stream {j}, which holds {int(n)} symbols"
            )
    return sched.astype(np.int32)


# ------------------------------------------------------------ device marshalling
class _Streams:
    """ilans_mux_stream descriptors + the concatenated tables they index."""

    def __init__(self, coders, need_slot: bool):
        k = len(coders)
        self.desc = (_lib.MuxStream * max(k, 1))()
        freq, cum, slot = [], [], []
        nf = nc = ns = 0
        seen: dict[int, tuple[int, int, int]] = {}
        for j, c in enumerate(coders):
            d = self.desc[j]
            if isinstance(c, RawStreamCodec):
                d.kind, d.nbytes, d.digit_bits = _lib.MUX_RAW, c.value_nbytes, c.width_bits
                continue
            if not isinstance(c, RansStreamCodec):
                raise TypeError(
                    f"stream {j}: the B200 mux takes RansStreamCodec or RawStreamCodec coders, "
                    f"not {type(c).__name__}"
                )
            t = c.table
            if id(t) not in seen:
                seen[id(t)] = (nf, nc, ns)
                freq.append(t.freq_u32)
                cum.append(t.cum_u32)
                nf += t.alphabet_size
                nc += t.alphabet_size + 1
                if need_slot:
                    slot.append(t.slot_u8)
                    ns += t.total
            d.kind, d.nbytes = _lib.MUX_RANS, c.digit_nbytes
            d.digit_bits, d.scale_bits = c.variant.digit_bits, t.scale_bits
            d.lower_bound, d.n_sym = c.variant.lower_bound, t.alphabet_size
            d.freq_off, d.cum_off, d.slot_off = seen[id(t)]
        self.k = k
        self.freq = np.concatenate(freq) if freq else np.zeros(1, np.uint32)
        self.cum = np.concatenate(cum) if cum else np.zeros(1, np.uint32)
        self.slot = np.concatenate(slot) if slot else np.zeros(1, np.uint8)
        self.nf, self.nc, self.ns = nf, nc, ns

    def table_args(self, with_slot: bool):
        a = [ctypes.byref(self.desc), self.k, _lib.ptr(self.freq), self.nf, _lib.ptr(self.cum),
             self.nc]
        if with_slot:
            a += [_lib.ptr(self.slot), self.ns]
        return a


def _stream_values(j: int, msg, coder) -> np.ndarray:
    """A message as u32 values, with the reference's range errors: raw values
    must fit width_bits (ValueError), rANS symbols must index the table."""
    a = np.asarray(msg if isinstance(msg, np.ndarray) else list(msg)).reshape(-1)
    if a.size and not np.issubdtype(a.dtype, np.integer):
        a = a.astype(np.int64)
    a = a.astype(np.int64, copy=False)
    if isinstance(coder, RawStreamCodec):
        bad = (a < 0) | (a >= (1 << coder.width_bits))
        if bad.any():
            raise ValueError(
                f"value {int(a[bad][0])} does not fit in {coder.width_bits} bits"
            )
    elif isinstance(coder, RansStreamCodec):
        bad = (a < 0) | (a >= coder.table.alphabet_size)
        if bad.any():
            raise IndexError(f"stream {j}: symbol {int(a[bad][-1])} outside the table's alphabet")
    return a.astype(np.uint32)


def _encode(messages, coders, sched: np.ndarray, flush_interval: int | None):
    """Device encode + merge: (payload, headers, per-stream bytes, segments,
    max_buffered)."""
    streams = _Streams(coders, need_slot=False)
    values = [_stream_values(j, m, c) for j, (m, c) in enumerate(zip(messages, coders))]
    symbols = np.concatenate(values) if values else np.zeros(0, np.uint32)
    if symbols.size == 0:
        symbols = np.zeros(1, np.uint32)
    t = int(sched.size)
    sched_buf = sched if t else np.zeros(1, np.int32)
    k = len(coders)
    out = np.empty(max(8 * t, 1), dtype=np.uint8)
    plen = ctypes.c_int64(0)
    states = np.zeros(max(k, 1), np.uint32)
    sbytes = np.zeros(max(k, 1), np.uint64)
    segs = ctypes.c_int64(0)
    maxb = ctypes.c_uint64(0)
    st = _lib.Status()
    rc = _lib.lib.ilans_mux_encode(
        *streams.table_args(False), _lib.ptr(symbols), _lib.ptr(sched_buf), t,
        int(flush_interval or 0), _lib.ptr(out), out.size, ctypes.byref(plen), _lib.ptr(states),
        _lib.ptr(sbytes), ctypes.byref(segs), ctypes.byref(maxb), ctypes.byref(st))
    if rc == _lib.ERR_UNENCODABLE:
        raise UnencodableSymbolError(f"symbol {st.symbol} has frequency 0")
    _lib.raise_for(rc, st, "mux encode")
    headers = [int(states[j]).to_bytes(4, "little") if isinstance(c, RansStreamCodec) else b""
               for j, c in enumerate(coders)]
    return (out[: plen.value].tobytes(), headers, sbytes[:k].astype(np.int64),
            int(segs.value), int(maxb.value))


# ------------------------------------------------------------ pipeline
def encode_multistream(messages, coders) -> list[StreamBuffer]:
    """Encode every stream independently, one segment each (reference
    mux.py:272-280)."""
    if len(messages) != len(coders):
        raise ValueError("one coder per message")
    lengths = [len(m) for m in messages]
    sched = np.repeat(np.arange(len(lengths), dtype=np.int32), lengths).astype(np.int32)
    payload, headers, sbytes, _, _ = _encode(messages, coders, sched, None)
    ends = np.cumsum(sbytes)
    starts = ends - sbytes
    return [StreamBuffer(headers[j], payload[int(starts[j]): int(ends[j])], lengths[j])
            for j in range(len(coders))]


def mux(buffers, coders, schedule) -> bytes:
    """Merge pre-encoded single-segment buffers in the schedule's decode
    order (reference mux.py:283-313): exactly sum(len(b.payload)) bytes."""
    if len(buffers) != len(coders):
        raise ValueError("one coder per buffer")
    counts = [int(b.symbol_count) for b in buffers]
    sched = _validate_schedule(schedule, counts)
    streams = _Streams(coders, need_slot=True)
    k = len(buffers)
    headers = [bytes(b.header) for b in buffers]
    payloads = [bytes(b.payload) for b in buffers]
    hoff = np.zeros(k + 1, np.uint64)
    poff = np.zeros(k + 1, np.uint64)
    hoff[1:] = np.cumsum([len(h) for h in headers])
    poff[1:] = np.cumsum([len(p) for p in payloads])
    hcat = np.frombuffer(b"".join(headers) or b"\0", dtype=np.uint8)
    pcat = np.frombuffer(b"".join(payloads) or b"\0", dtype=np.uint8)
    cnt = np.asarray(counts or [0], dtype=np.int64)
    out = np.empty(max(int(poff[-1]), 1), dtype=np.uint8)
    t = int(sched.size)
    sched_buf = sched if t else np.zeros(1, np.int32)
    st = _lib.Status()
    rc = _lib.lib.ilans_mux_merge(
        *streams.table_args(True), _lib.ptr(hcat), _lib.ptr(hoff), _lib.ptr(pcat),
        _lib.ptr(poff), _lib.ptr(cnt), _lib.ptr(sched_buf), t, _lib.ptr(out), ctypes.byref(st))
    _lib.raise_for(rc, st, "mux merge")
    return out[: int(poff[-1])].tobytes()


def mux_with_flush(messages, coders, schedule=None,
                   flush_interval: int | None = None) -> tuple[MuxedContainer, MuxBudget]:
    """Segment every stream at epochs of ``flush_interval`` schedule steps,
    encode and merge (reference mux.py:329-433). Segment 0's state is the
    stream header; later segments carry theirs inline. With
    flush_interval=None the payload equals mux(encode_multistream(...))."""
    if len(messages) != len(coders):
        raise ValueError("one coder per message")
    lengths = [len(m) for m in messages]
    if schedule is None:
        schedule = round_robin_schedule(lengths)
    sched = _validate_schedule(schedule, lengths)
    if flush_interval is not None and flush_interval < 1:
        raise ValueError("flush_interval must be >= 1")
    payload, headers, _, segments, max_buffered = _encode(messages, coders, sched,
                                                          flush_interval)
    container = MuxedContainer(flush_interval, lengths, headers, payload)
    return container, MuxBudget(flush_interval, max_buffered, segments, len(payload))


def demux_decode(muxed, coders, schedule=None) -> list[list[int]]:
    """Decode every stream out of a MuxedContainer (or its bytes) with the
    schedule it was muxed with (reference mux.py:436-475)."""
    c = muxed if isinstance(muxed, MuxedContainer) else MuxedContainer.from_bytes(muxed)
    if len(c.stream_lengths) != len(coders):
        raise ValueError("one coder per stream")
    lengths = [int(n) for n in c.stream_lengths]
    if schedule is None:
        schedule = round_robin_schedule(lengths)
    sched = _validate_schedule(schedule, lengths)
    streams = _Streams(coders, need_slot=True)
    k = len(coders)
    headers = [bytes(h) for h in c.stream_headers]
    hoff = np.zeros(k + 1, np.uint64)
    hoff[1:] = np.cumsum([len(h) for h in headers])
    hcat = np.frombuffer(b"".join(headers) or b"\0", dtype=np.uint8)
    payload = bytes(c.payload)
    pbuf = np.frombuffer(payload or b"\0", dtype=np.uint8)
    t = int(sched.size)
    sched_buf = sched if t else np.zeros(1, np.int32)
    out = np.empty(max(t, 1), dtype=np.uint32)
    unread = ctypes.c_int64(0)
    flush = int(c.flush_interval or 0)
    st = _lib.Status()
    rc = _lib.lib.ilans_mux_demux(
        *streams.table_args(True), _lib.ptr(hcat), _lib.ptr(hoff), _lib.ptr(pbuf), len(payload),
        _lib.ptr(sched_buf), t, flush, None, _lib.ptr(out), ctypes.byref(unread),
        ctypes.byref(st))
    _lib.raise_for(rc, st, "demux")
    if unread.value:
        warnings.warn(f"{unread.value} unread bytes after demux", TrailingGarbageWarning,
                      stacklevel=2)
    values = out[:t]  # stream by stream (the device's stable sort of the schedule)
    ends = np.cumsum(lengths)
    return [values[e - n: e].tolist() for n, e in zip(lengths, ends)]
