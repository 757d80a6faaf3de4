"""Chunk framing and the HBM-resident codec pipeline.

A message is cut into fixed-size chunks (boundaries depend only on the
chunk length, never on the GPU count); chunk k is an independent N-lane
word16 stream under ONE global table, so its payload and final states are
exactly the reference's ``encode_interleaved(msg[kC:(k+1)C], table, N,
WORD16)`` and it re-wraps as a standalone IEC1 ``Container``
(``ChunkedContainer.chunk(k)``).

``DeviceCodec`` keeps everything in HBM: histogram -> (optional NCCL
all-reduce) -> quantize + tables -> one encode launch over all chunks ->
framing (offset scan + payload compaction); decode is one launch over all
chunks. Torch provides device memory and the stream; all compute is
libilans_b200.so.

ICH1 wire format (little-endian), the on-disk form of a chunked stream:

    0   4      magic "ICH1"
    4   1      version (1)
    5   1      variant (1 = word16, 0 = byte8; the IEC1 codes, interleave.py:10-20)
    6   2      lane_count N (u16)
    8   8      message_length (u64)
    16  8      chunk_len C (u64)
    24  3+2n   table (rans.serialize_table)
    -   4K     payload digits per chunk (u32), K = ceil(len / C)
    -   4KN    final lane states, chunk-major (u32)
    -   rest   payloads back to back (u16 LE digits for word16, bytes for byte8)
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib, rans
from .errors import FormatError, TruncatedStreamError
from .interleave import Container, _as_symbols
from .rans import BYTE8, WORD16, RenormVariant, SymbolTable

CHUNK_MAGIC = b"ICH1"
DEFAULT_CHUNK = 64 * 1024

__all__ = ["ChunkedContainer", "DeviceCodec", "encode_chunked", "decode_chunked"]


def n_chunks_for(n: int, chunk_len: int) -> int:
    return 0 if n == 0 else -(-n // chunk_len)


def _check_chunking(chunk_len: int, lane_count: int) -> None:
    if chunk_len <= 0 or chunk_len % 16:
        raise ValueError("chunk_len must be a positive multiple of 16")
    if not 1 <= lane_count <= 32:
        raise ValueError("chunked streams use 1..32 lanes (one warp per chunk)")


@dataclass
class ChunkedContainer:
    lane_count: int
    chunk_len: int
    message_length: int
    table: SymbolTable
    states: np.ndarray        # u32 [n_chunks, N]
    word_offsets: np.ndarray  # u64 [n_chunks + 1], in digits (words / bytes)
    payload: np.ndarray       # u16 (word16) or u8 (byte8) [word_offsets[-1]]
    variant: RenormVariant = WORD16

    @property
    def n_chunks(self) -> int:
        return n_chunks_for(self.message_length, self.chunk_len)

    def chunk_length(self, k: int) -> int:
        return min(self.chunk_len, self.message_length - k * self.chunk_len)

    def chunk(self, k: int) -> Container:
        """Chunk k as a standalone IEC1 container (reference-decodable)."""
        a, b = int(self.word_offsets[k]), int(self.word_offsets[k + 1])
        return Container(self.variant, self.lane_count, self.chunk_length(k), self.table,
                         tuple(self.states[k].tolist()), self.payload[a:b].copy())

    def to_bytes(self) -> bytes:
        byte8 = self.variant == BYTE8
        head = CHUNK_MAGIC + struct.pack("<BBHQQ", 1, 0 if byte8 else 1, self.lane_count,
                                         self.message_length, self.chunk_len)
        words = np.diff(self.word_offsets.astype(np.uint64)).astype("<u4")
        return (head + rans.serialize_table(self.table) + words.tobytes()
                + np.ascontiguousarray(self.states, dtype="<u4").tobytes()
                + np.ascontiguousarray(self.payload, dtype="u1" if byte8 else "<u2").tobytes())

    @classmethod
    def from_bytes(cls, raw: bytes) -> "ChunkedContainer":
        raw = bytes(raw)
        if len(raw) < 24:
            raise TruncatedStreamError("chunked container shorter than fixed header")
        if raw[:4] != CHUNK_MAGIC:
            raise FormatError("bad magic; not an ilans chunked container")
        version, variant, lanes, n, chunk_len = struct.unpack_from("<BBHQQ", raw, 4)
        if version != 1:
            raise FormatError(f"unsupported container version {version}")
        if variant not in (0, 1):
            raise FormatError(f"unknown variant byte {variant}")
        var = WORD16 if variant == 1 else BYTE8
        if not 1 <= lanes <= 32 or chunk_len == 0 or chunk_len % 16:
            raise FormatError("invalid lane_count / chunk_len")
        table, off = rans.parse_table(raw, 24)
        k = n_chunks_for(n, chunk_len)
        need = off + 4 * k + 4 * k * lanes
        if len(raw) < need:
            raise TruncatedStreamError("chunk directory truncated")
        words = np.frombuffer(raw, dtype="<u4", count=k, offset=off).astype(np.uint64)
        off += 4 * k
        states = np.frombuffer(raw, dtype="<u4", count=k * lanes, offset=off).astype(
            np.uint32).reshape(k, lanes)
        off += 4 * k * lanes
        if ((states < var.lower_bound) | (states.astype(np.uint64) >= var.state_limit)).any():
            raise FormatError("lane state outside the coder interval")
        offsets = np.zeros(k + 1, dtype=np.uint64)
        np.cumsum(words, out=offsets[1:])
        tail = raw[off:]
        if var == BYTE8:
            if len(tail) < int(offsets[-1]):
                raise TruncatedStreamError("payload truncated")
            payload = np.frombuffer(tail, dtype=np.uint8).copy()
        else:
            if len(tail) % 2:
                raise FormatError("word16 payload has odd byte length")
            if len(tail) // 2 < int(offsets[-1]):
                raise TruncatedStreamError("payload truncated")
            payload = np.frombuffer(tail, dtype="<u2").astype(np.uint16)
        return cls(lanes, chunk_len, n, table, states, offsets, payload, var)


# ---------------------------------------------------------------------------
# HBM-resident pipeline
# ---------------------------------------------------------------------------
def _torch():
    import torch  # torch: device memory, streams, NCCL plumbing only

    return torch


class DeviceCodec:
    """Chunked word16 codec resident on one GPU.

    Buffers are allocated once for ``capacity`` message bytes and reused;
    every method is asynchronous on ``stream`` (default: torch's current
    stream) except the explicit ``*_host`` read-backs.
    """

    def __init__(self, capacity: int, chunk_len: int = DEFAULT_CHUNK, lane_count: int = 32,
                 scale_bits: int = 14, device=None, stream=None):
        torch = _torch()
        _check_chunking(chunk_len, lane_count)
        if not 1 <= scale_bits <= 16:
            raise ValueError("scale_bits must be in [1, 16]")
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        self.capacity = int(capacity)
        self.chunk_len = int(chunk_len)
        self.lane_count = int(lane_count)
        self.scale_bits = int(scale_bits)
        self.stream = stream
        kmax = max(1, n_chunks_for(self.capacity, chunk_len))
        dev = self.device
        e = lambda n, dt: torch.empty(n, dtype=dt, device=dev)  # noqa: E731
        self.table = e(int(_lib.lib.ilans_table_bytes()), torch.uint8)
        self.status = e(int(_lib.lib.ilans_dstatus_bytes()), torch.uint8)
        # pinned landing buffer for stream-ordered status reads (a pageable
        # read would queue behind every copy already on the copy engine)
        self.status_host = torch.empty(int(_lib.lib.ilans_dstatus_bytes()), dtype=torch.uint8,
                                       pin_memory=True)
        self.counts = torch.zeros(256, dtype=torch.int64, device=dev)
        self.scratch = e(max(1, self.capacity) + 8, torch.int16)
        self.payload = e(max(1, self.capacity) + 8, torch.int16)
        self.chunk_words = e(kmax, torch.int32)
        self.offsets = e(kmax + 1, torch.int64)
        self.states = e(kmax * lane_count, torch.int32)
        self.consumed = e(kmax, torch.int64)
        self.final_states = e(kmax * lane_count, torch.int32)

    # -- plumbing ---------------------------------------------------------
    def _s(self) -> int:
        torch = _torch()
        s = self.stream if self.stream is not None else torch.cuda.current_stream(self.device)
        return int(s.cuda_stream)

    @staticmethod
    def _p(t) -> int:
        return int(t.data_ptr())

    # -- model ------------------------------------------------------------
    def histogram(self, d_msg, n: int, accumulate: bool = False):
        """counts[b] (+)= #{i < n : d_msg[i] == b} (int64 view of u64)."""
        self._counts_of = None if accumulate else (self._p(d_msg), int(n))
        s = self._s()
        if not accumulate:
            _lib.check_dev(_lib.lib.ilans_counts_zero_dev(self._p(self.counts), s), "counts_zero")
        _lib.check_dev(_lib.lib.ilans_histogram_u8_dev(self._p(d_msg), int(n),
                                                       self._p(self.counts), s), "histogram")
        return self.counts

    def build_table_from_counts(self):
        # a model quantized from a message's own histogram gives every byte
        # of that message f >= 1: its encode may skip the zero-frequency check
        self._covers = getattr(self, "_counts_of", None)
        _lib.check_dev(_lib.lib.ilans_table_from_counts_dev(
            self._p(self.counts), self.scale_bits, self._p(self.table), self._s()), "table")

    def build_table_from_freq(self, table: SymbolTable):
        torch = _torch()
        if table.scale_bits != self.scale_bits:
            raise ValueError("table scale_bits differs from the codec's")
        self._covers = None
        f = torch.from_numpy(table.freq_u32.view(np.int32).copy()).to(self.device,
                                                                      non_blocking=False)
        self._freq_keepalive = f
        _lib.check_dev(_lib.lib.ilans_table_from_freq_dev(
            self._p(f), table.alphabet_size, table.scale_bits, self._p(self.table), self._s()),
            "table_from_freq")

    def read_table(self) -> SymbolTable:
        """Synchronizing read-back of the device model as a SymbolTable."""
        alpha = ctypes.c_int32(0)
        sb = ctypes.c_int32(0)
        freq = np.zeros(256, dtype=np.uint32)
        st = _lib.Status()
        rc = _lib.lib.ilans_table_read_host(self._p(self.table), ctypes.byref(alpha),
                                            ctypes.byref(sb), _lib.ptr(freq), self._s(),
                                            ctypes.byref(st))
        _lib.raise_for(rc, st, "table")
        return SymbolTable(freq[: alpha.value].tolist(), sb.value)

    # -- coding -----------------------------------------------------------
    def reset_status(self):
        _lib.check_dev(_lib.lib.ilans_dstatus_reset_dev(self._p(self.status), self._s()),
                       "status")

    def check_status(self):
        st = _lib.Status()
        rc = _lib.lib.ilans_dstatus_read_host(self._p(self.status), self._s(), ctypes.byref(st))
        _lib.raise_for(rc, st, "device status")

    def copy_status(self, stream):
        """Queue a copy of the device status into status_host on ``stream``."""
        with _torch().cuda.stream(stream):
            self.status_host.copy_(self.status, non_blocking=True)

    def check_status_host(self):
        """Raise for the status last landed by copy_status (caller synced)."""
        st = _lib.Status()
        rc = _lib.lib.ilans_dstatus_parse(self._p(self.status_host), ctypes.byref(st))
        _lib.raise_for(rc, st, "device status")

    def encode(self, d_msg, n: int, frame: bool = True):
        """Encode n bytes at d_msg with the current table: one launch for all
        chunks, then (frame=True) the offset scan + payload compaction."""
        k = n_chunks_for(n, self.chunk_len)
        covered = getattr(self, "_covers", None) == (self._p(d_msg), int(n))
        self.encode_range(self._p(d_msg), n, 0, k, covered=covered)
        if frame:
            self.frame_range(n, 0, k, self._p(self.payload))

    # chunk-range pieces (for batched / pipelined use; pointers are ints)
    def _range(self, n: int, k0: int, k1: int):
        if n > self.capacity:
            raise ValueError("message larger than codec capacity")
        lo = k0 * self.chunk_len
        return lo, min(n, k1 * self.chunk_len) - lo

    def encode_range(self, msg_ptr: int, n: int, k0: int, k1: int, covered: bool = False):
        """Encode chunks [k0, k1) of the n-byte message starting at msg_ptr.
        covered=True: the current table was quantized from this message's
        own histogram (every byte has f >= 1), so the per-symbol
        zero-frequency check is skipped."""
        lo, nb = self._range(n, k0, k1)
        if nb <= 0:
            return
        fn = _lib.lib.ilans_encode_chunks_covered_dev if covered else _lib.lib.ilans_encode_chunks_dev
        _lib.check_dev(fn(
            msg_ptr + lo, nb, self.chunk_len, self.lane_count, self._p(self.table),
            self.scale_bits, self._p(self.scratch) + 2 * lo, self._p(self.chunk_words) + 4 * k0,
            self._p(self.states) + 4 * k0 * self.lane_count, self._p(self.status), self._s()),
            "encode")

    def frame_range(self, n: int, k0: int, k1: int, payload_ptr: int, stream: int | None = None):
        """Offsets for chunks [k0, k1) (continuing from offsets[k0] when
        k0 > 0) and their payloads packed at payload_ptr + 2*offset. The
        destination may be mapped pinned host memory (packing over PCIe)."""
        lo, nb = self._range(n, k0, k1)
        if nb <= 0:
            if k0 == 0:
                self.offsets[:1].zero_()
            return
        _lib.check_dev(_lib.lib.ilans_frame_chunks_dev(
            self._p(self.scratch) + 2 * lo, nb, self.chunk_len,
            self._p(self.chunk_words) + 4 * k0, self._p(self.offsets) + 8 * k0, payload_ptr,
            1 if k0 > 0 else 0, self._s() if stream is None else stream), "frame")

    def decode_range(self, out_ptr: int, n: int, k0: int, k1: int, payload_ptr: int,
                     offsets_ptr: int, states_ptr: int, final_states: bool = False,
                     stream: int | None = None):
        """Decode chunks [k0, k1) into out_ptr + k0*C. offsets_ptr/states_ptr
        point at the whole message's directory (global word offsets into
        payload_ptr)."""
        lo, nb = self._range(n, k0, k1)
        if nb <= 0:
            return
        N = self.lane_count
        _lib.check_dev(_lib.lib.ilans_decode_chunks_dev(
            payload_ptr, offsets_ptr + 8 * k0, states_ptr + 4 * k0 * N, nb, self.chunk_len, N,
            self._p(self.table), self.scale_bits, out_ptr + lo, self._p(self.consumed) + 8 * k0,
            (self._p(self.final_states) + 4 * k0 * N) if final_states else None,
            self._p(self.status), self._s() if stream is None else stream), "decode")

    def decode(self, d_out, n: int, payload=None, offsets=None, states=None,
               final_states: bool = False):
        """Decode n bytes into d_out from (payload, offsets, states) -- by
        default the codec's own framed encode output."""
        payload = self.payload if payload is None else payload
        offsets = self.offsets if offsets is None else offsets
        states = self.states if states is None else states
        _lib.check_dev(_lib.lib.ilans_decode_chunks_dev(
            self._p(payload), self._p(offsets), self._p(states), int(n), self.chunk_len,
            self.lane_count, self._p(self.table), self.scale_bits, self._p(d_out),
            self._p(self.consumed), self._p(self.final_states) if final_states else None,
            self._p(self.status), self._s()), "decode")

    def decode_slots(self, d_out, n: int, final_states: bool = False):
        """Decode n bytes into d_out straight from this codec's encode scratch
        (each chunk's words right-aligned in its slot, counts in
        chunk_words): the device-resident round trip needs no packing pass;
        the packed ICH1 payload is built when the stream leaves HBM
        (frame_range into mapped pinned host memory)."""
        _lib.check_dev(_lib.lib.ilans_decode_chunks_slots_dev(
            self._p(self.scratch), self._p(self.chunk_words), self._p(self.states), int(n),
            self.chunk_len, self.lane_count, self._p(self.table), self.scale_bits,
            self._p(d_out), self._p(self.consumed),
            self._p(self.final_states) if final_states else None, self._p(self.status),
            self._s()), "decode_slots")

    def directory(self, n: int):
        """Word offsets of the framed stream (the ICH1 directory) from the
        encoder's chunk word counts, without packing the payload."""
        k = n_chunks_for(n, self.chunk_len)
        _lib.check_dev(_lib.lib.ilans_frame_chunks_dev(
            self._p(self.scratch), int(n), self.chunk_len, self._p(self.chunk_words),
            self._p(self.offsets), None, 0, self._s()), "directory")
        return self.offsets[: k + 1]

    def decode_adler32(self, n: int, adler=None, payload=None, offsets=None, states=None,
                       slots: bool = False):
        """Decode fused with its consumer: the zlib Adler-32
        of every decoded chunk (uint32 per chunk, as int32 tensor), computed
        in registers -- the decoded bytes never reach HBM."""
        torch = _torch()
        k = n_chunks_for(n, self.chunk_len)
        if adler is None:
            adler = torch.empty(max(1, k), dtype=torch.int32, device=self.device)
        if slots:  # straight from the encode scratch (see decode_slots)
            _lib.check_dev(_lib.lib.ilans_decode_chunks_slots_adler32_dev(
                self._p(self.scratch), self._p(self.chunk_words), self._p(self.states), int(n),
                self.chunk_len, self.lane_count, self._p(self.table), self.scale_bits,
                self._p(adler), self._p(self.consumed), self._p(self.status), self._s()),
                "decode_slots_adler32")
            return adler[:k]
        payload = self.payload if payload is None else payload
        offsets = self.offsets if offsets is None else offsets
        states = self.states if states is None else states
        _lib.check_dev(_lib.lib.ilans_decode_chunks_adler32_dev(
            self._p(payload), self._p(offsets), self._p(states), int(n), self.chunk_len,
            self.lane_count, self._p(self.table), self.scale_bits, self._p(adler),
            self._p(self.consumed), self._p(self.status), self._s()), "decode_adler32")
        return adler[:k]

    def adler32(self, d_data, n: int, adler=None):
        """Per-chunk Adler-32 of n bytes already on the device (unfused)."""
        torch = _torch()
        k = n_chunks_for(n, self.chunk_len)
        if adler is None:
            adler = torch.empty(max(1, k), dtype=torch.int32, device=self.device)
        _lib.check_dev(_lib.lib.ilans_adler32_chunks_dev(
            self._p(d_data), int(n), self.chunk_len, self._p(adler), self._s()), "adler32")
        return adler[:k]

    # -- read-back --------------------------------------------------------
    def encoded_host(self, n: int, table: SymbolTable) -> ChunkedContainer:
        torch = _torch()
        k = n_chunks_for(n, self.chunk_len)
        torch.cuda.current_stream(self.device).synchronize() if self.stream is None \
            else self.stream.synchronize()
        offs = self.offsets[: k + 1].cpu().numpy().view(np.uint64).copy()
        words = int(offs[-1]) if k else 0
        payload = self.payload[:words].cpu().numpy().view(np.uint16).copy()
        states = self.states[: k * self.lane_count].cpu().numpy().view(np.uint32).reshape(
            k, self.lane_count).copy()
        if k == 0:
            offs = np.zeros(1, dtype=np.uint64)
        return ChunkedContainer(self.lane_count, self.chunk_len, n, table, states, offs, payload)


def encode_chunked(message, table: SymbolTable | None = None, lane_count: int = 32,
                   chunk_len: int = DEFAULT_CHUNK, scale_bits: int = 14,
                   variant: RenormVariant = WORD16) -> ChunkedContainer:
    """Encode host bytes as independent N-lane chunks under one table. With
    table=None the model is built on the device (histogram + quantize), as
    cli._build_table does on the host (cli.py:31-37). variant=BYTE8 codes
    every chunk with byte digits (the reference's scalar byte8 path)."""
    torch = _torch()
    _check_chunking(chunk_len, lane_count)
    if variant == BYTE8:
        return _encode_chunked_u8(message, table, lane_count, chunk_len, scale_bits)
    if variant != WORD16:
        from .errors import UnsupportedVariantError

        raise UnsupportedVariantError(f"chunked streams are word16 or byte8, not {variant.tag!r}")
    if table is not None:
        msg = _as_symbols(message, table)
        WORD16.check_table(table)
        scale_bits = table.scale_bits
    else:
        msg = np.frombuffer(message, dtype=np.uint8) if isinstance(
            message, (bytes, bytearray, memoryview)) else np.asarray(message, dtype=np.uint8)
    n = len(msg)
    codec = DeviceCodec(max(16, n), chunk_len, lane_count, scale_bits)
    d_msg = torch.empty(max(16, n), dtype=torch.uint8, device=codec.device)
    if n:
        d_msg[:n].copy_(torch.from_numpy(np.ascontiguousarray(msg)))
    if table is None:
        codec.histogram(d_msg, n)
        codec.build_table_from_counts()
        table = codec.read_table()
    else:
        codec.build_table_from_freq(table)
    codec.reset_status()
    codec.encode(d_msg, n)
    codec.check_status()
    return codec.encoded_host(n, table)


def decode_chunked(cc: ChunkedContainer) -> np.ndarray:
    """Decode a ChunkedContainer on the device (one launch for all chunks)."""
    torch = _torch()
    _check_chunking(cc.chunk_len, cc.lane_count)
    if cc.variant == BYTE8:
        return _decode_chunked_u8(cc)
    n = cc.message_length
    if n == 0:
        return np.zeros(0, dtype=np.uint8)
    k = cc.n_chunks
    if cc.states.shape != (k, cc.lane_count) or len(cc.word_offsets) != k + 1:
        raise FormatError("chunk directory does not match the message length")
    codec = DeviceCodec(n, cc.chunk_len, cc.lane_count, cc.table.scale_bits)
    dev = codec.device
    pay = torch.from_numpy(np.ascontiguousarray(cc.payload).view(np.int16)).to(dev)
    if pay.numel() == 0:
        pay = torch.zeros(8, dtype=torch.int16, device=dev)
    offs = torch.from_numpy(np.ascontiguousarray(cc.word_offsets, dtype=np.uint64).view(
        np.int64)).to(dev)
    states = torch.from_numpy(np.ascontiguousarray(cc.states, dtype=np.uint32).view(
        np.int32).reshape(-1)).to(dev)
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    codec.build_table_from_freq(cc.table)
    codec.reset_status()
    codec.decode(out, n, pay, offs, states)
    codec.check_status()
    consumed = codec.consumed[:k].cpu().numpy()
    if (consumed != np.diff(cc.word_offsets.astype(np.int64))).any():
        import warnings

        from .errors import TrailingGarbageWarning

        warnings.warn("unread digits after chunk decode", TrailingGarbageWarning, stacklevel=2)
    return out.cpu().numpy()


class _Model:
    """Device table + status blobs for the one-shot byte8 calls."""

    def __init__(self, torch, dev):
        self.torch, self.dev = torch, dev
        self.table = torch.empty(int(_lib.lib.ilans_table_bytes()), dtype=torch.uint8, device=dev)
        self.status = torch.empty(int(_lib.lib.ilans_dstatus_bytes()), dtype=torch.uint8,
                                  device=dev)
        self.s = int(torch.cuda.current_stream(dev).cuda_stream)

    def from_freq(self, table: SymbolTable):
        f = self.torch.from_numpy(table.freq_u32.view(np.int32).copy()).to(self.dev)
        self._keep = f
        _lib.check_dev(_lib.lib.ilans_table_from_freq_dev(
            int(f.data_ptr()), table.alphabet_size, table.scale_bits, int(self.table.data_ptr()),
            self.s), "table_from_freq")

    def from_message(self, d_msg, n: int, scale_bits: int) -> SymbolTable:
        counts = self.torch.zeros(256, dtype=self.torch.int64, device=self.dev)
        _lib.check_dev(_lib.lib.ilans_histogram_u8_dev(int(d_msg.data_ptr()), int(n),
                                                       int(counts.data_ptr()), self.s),
                       "histogram")
        _lib.check_dev(_lib.lib.ilans_table_from_counts_dev(
            int(counts.data_ptr()), scale_bits, int(self.table.data_ptr()), self.s), "table")
        alpha, sb = ctypes.c_int32(0), ctypes.c_int32(0)
        freq = np.zeros(256, dtype=np.uint32)
        st = _lib.Status()
        rc = _lib.lib.ilans_table_read_host(int(self.table.data_ptr()), ctypes.byref(alpha),
                                            ctypes.byref(sb), _lib.ptr(freq), self.s,
                                            ctypes.byref(st))
        _lib.raise_for(rc, st, "table")
        return SymbolTable(freq[: alpha.value].tolist(), sb.value)

    def reset(self):
        _lib.check_dev(_lib.lib.ilans_dstatus_reset_dev(int(self.status.data_ptr()), self.s),
                       "status")

    def check(self):
        st = _lib.Status()
        rc = _lib.lib.ilans_dstatus_read_host(int(self.status.data_ptr()), self.s,
                                              ctypes.byref(st))
        _lib.raise_for(rc, st, "device status")


def _encode_chunked_u8(message, table, lane_count: int, chunk_len: int,
                       scale_bits: int) -> ChunkedContainer:
    """Chunked byte8: one warp per chunk (csrc/byte8.cu), byte framing."""
    torch = _torch()
    if table is not None:
        msg = _as_symbols(message, table)
        BYTE8.check_table(table)
    else:
        msg = np.frombuffer(message, dtype=np.uint8) if isinstance(
            message, (bytes, bytearray, memoryview)) else np.asarray(message, dtype=np.uint8)
    n = len(msg)
    dev = torch.device("cuda", torch.cuda.current_device())
    m = _Model(torch, dev)
    d_msg = torch.zeros(max(16, n), dtype=torch.uint8, device=dev)
    if n:
        d_msg[:n].copy_(torch.from_numpy(np.ascontiguousarray(msg)))
    if table is None:
        table = m.from_message(d_msg, n, scale_bits)
        BYTE8.check_table(table)
    else:
        m.from_freq(table)
    k = n_chunks_for(n, chunk_len)
    cap = 3 * max(n, 1) + 16
    scratch = torch.empty(cap, dtype=torch.uint8, device=dev)
    payload = torch.empty(cap, dtype=torch.uint8, device=dev)
    nbytes = torch.zeros(max(k, 1), dtype=torch.int32, device=dev)
    offsets = torch.zeros(k + 1, dtype=torch.int64, device=dev)
    states = torch.empty(max(k, 1) * lane_count, dtype=torch.int32, device=dev)
    m.reset()
    p = lambda t: int(t.data_ptr())  # noqa: E731
    if n:
        _lib.check_dev(_lib.lib.ilans_encode_chunks_u8_dev(
            p(d_msg), n, chunk_len, lane_count, p(m.table), p(scratch), p(nbytes), p(states),
            p(m.status), m.s), "encode_chunks_u8")
        m.check()
        _lib.check_dev(_lib.lib.ilans_frame_chunks_u8_dev(
            p(scratch), n, chunk_len, p(nbytes), p(offsets), p(payload), m.s), "frame_u8")
    offs = offsets.cpu().numpy().view(np.uint64).copy()
    total = int(offs[-1]) if k else 0
    return ChunkedContainer(lane_count, chunk_len, n, table,
                            states[: k * lane_count].cpu().numpy().view(np.uint32)
                            .reshape(k, lane_count).copy(),
                            offs if k else np.zeros(1, np.uint64),
                            payload[:total].cpu().numpy().copy(), BYTE8)


def _decode_chunked_u8(cc: ChunkedContainer) -> np.ndarray:
    torch = _torch()
    n = cc.message_length
    if n == 0:
        return np.zeros(0, dtype=np.uint8)
    k = cc.n_chunks
    if cc.states.shape != (k, cc.lane_count) or len(cc.word_offsets) != k + 1:
        raise FormatError("chunk directory does not match the message length")
    dev = torch.device("cuda", torch.cuda.current_device())
    m = _Model(torch, dev)
    m.from_freq(cc.table)
    pay = torch.zeros(max(len(cc.payload), 1) + 8, dtype=torch.uint8, device=dev)
    if len(cc.payload):
        pay[: len(cc.payload)].copy_(torch.from_numpy(np.ascontiguousarray(cc.payload,
                                                                           dtype=np.uint8)))
    offs = torch.from_numpy(np.ascontiguousarray(cc.word_offsets, dtype=np.uint64)
                            .view(np.int64)).to(dev)
    states = torch.from_numpy(np.ascontiguousarray(cc.states, dtype=np.uint32).view(np.int32)
                              .reshape(-1)).to(dev)
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    consumed = torch.zeros(k, dtype=torch.int64, device=dev)
    m.reset()
    p = lambda t: int(t.data_ptr())  # noqa: E731
    _lib.check_dev(_lib.lib.ilans_decode_chunks_u8_dev(
        p(pay), p(offs), p(states), n, cc.chunk_len, cc.lane_count, p(m.table), p(out),
        p(consumed), p(m.status), m.s), "decode_chunks_u8")
    m.check()
    if (consumed.cpu().numpy() != np.diff(cc.word_offsets.astype(np.int64))).any():
        import warnings

        from .errors import TrailingGarbageWarning

        warnings.warn("unread digits after chunk decode", TrailingGarbageWarning, stacklevel=2)
    return out.cpu().numpy()


class _Slot:
    """One in-flight round trip: device buffers, pinned host buffers and the
    streams of one HostCodec slot."""

    def __init__(self, torch, dev, capacity, chunk_len, lane_count, scale_bits):
        self.s_in = torch.cuda.Stream(dev)
        self.s_comp = torch.cuda.Stream(dev)
        self.s_out = torch.cuda.Stream(dev)
        self.s_dec = [torch.cuda.Stream(dev) for _ in range(4)]
        self.codec = DeviceCodec(capacity, chunk_len, lane_count, scale_bits, dev,
                                 stream=self.s_comp)
        self.d_msg = torch.empty(max(16, capacity), dtype=torch.uint8, device=dev)
        self.d_out = torch.empty(max(16, capacity), dtype=torch.uint8, device=dev)
        k = max(1, n_chunks_for(capacity, chunk_len))
        pin = lambda n, dt: torch.empty(n, dtype=dt, pin_memory=True)  # noqa: E731
        self.h_offsets = pin(k + 1, torch.int64)
        self.h_states = pin(k * lane_count, torch.int32)
        self.h_payload = pin(max(1, capacity) + 8, torch.int16)
        self.free = None  # event: the slot's last round trip has finished on the device
        self.pending = None  # an EncodeJob whose payload downloads are not issued yet

    def streams(self):
        return (self.s_in, self.s_comp, self.s_out, *self.s_dec)


class EncodeJob:
    """An ``HostCodec.encode_async`` in flight. ``encode_async`` returns as
    soon as the work is queued; the payload downloads need the word offsets
    on the host, so they are issued by ``materialize()`` -- called by
    ``wait()`` and by a ``decode_async`` of this job -- which blocks only
    until the offsets have landed (and raises the encode's device errors).
    payload / offsets / states are views of the slot's pinned buffers."""

    def __init__(self, codec, slot, n, k, batches, ev_off, ev_status, ev_states, h2d):
        self.codec, self.slot, self.n, self.k = codec, slot, n, k
        self.batches, self.ev_off, self.ev_status = batches, ev_off, ev_status
        self.ev_states = ev_states
        self.ev_pay = None
        self.ev_done = None
        self.h2d_bytes = h2d
        self.d2h_bytes = None
        self.words = None

    def materialize(self):
        """Issue the payload downloads (once): per batch, as soon as its word
        offsets are on the host."""
        if self.ev_pay is not None:
            return self
        if self.slot.pending is self:
            self.slot.pending = None
        torch = _torch()
        slot, c = self.slot, self.slot.codec
        N = c.lane_count
        ev_pay = []
        for i, ((k0, k1), ev) in enumerate(zip(self.batches, self.ev_off)):
            ev.synchronize()
            if i == len(self.batches) - 1:  # the encode kernel is done: report its errors
                self.ev_status.synchronize()
                c.check_status_host()
            a, b = int(slot.h_offsets[k0]), int(slot.h_offsets[k1])
            with torch.cuda.stream(slot.s_out):
                slot.h_payload[a:b].copy_(c.payload[a:b], non_blocking=True)
            ev_pay.append(HostCodec._event(slot.s_out))
        self.codec._mark("enc.d2h.end", slot.s_out)
        self.ev_done = HostCodec._event(slot.s_out)
        self.ev_pay = ev_pay
        k = self.k
        self.words = int(slot.h_offsets[k]) if k else 0
        self.d2h_bytes = 8 * (k + 1) + 4 * k * N + 2 * self.words
        self.payload = slot.h_payload[: self.words]
        self.offsets = slot.h_offsets[: k + 1]
        self.states = slot.h_states[: k * N]
        return self

    def wait(self):
        """Payload, offsets and states on the host."""
        self.materialize()
        self.ev_done.synchronize()
        return self.payload, self.offsets, self.states


class DecodeJob:
    def __init__(self, slot, out, ev_done, h2d, d2h):
        self.slot, self.out, self.ev_done = slot, out, ev_done
        self.h2d_bytes, self.d2h_bytes = h2d, d2h
        self._checked = False

    def wait(self):
        self.ev_done.synchronize()
        if not self._checked:
            self.slot.codec.check_status_host()
            self._checked = True
        return self.out


class HostCodec:
    """End-to-end chunked codec over pinned host buffers: the public call a
    user makes with data in host memory. Work is split into chunk-aligned
    batches on per-slot streams so PCIe traffic overlaps the kernels:

    encode: H2D batch b (copy stream) || histogram of batch b (compute
      stream) -> [NCCL all-reduce] -> quantize + tables -> one encode launch
      -> per batch: framing (offsets + packing) -> offsets D2H; the payload
      of batch b goes D2H once its size is known on the host.
    decode: directory H2D -> per batch: payload H2D (copy) || decode (one
      of four streams: a batch alone cannot fill the GPU, a chunk is one
      warp) || decoded bytes D2H (output stream).

    ``slots`` (default 2) independent buffer sets let consecutive calls
    overlap: ``encode_async`` (never blocks) and ``decode_async`` return
    jobs, so the upload of the next message runs while the previous round
    trip's results are still coming down (PCIe is full duplex; a lone call
    leaves one direction idle while the whole message is uploaded for the
    histogram). An encode job issues its payload downloads in
    ``materialize()`` (called by ``wait()`` and by a ``decode_async`` of
    it), which waits for the word offsets. Job results are views of the
    slot's pinned buffers, valid until the slot is reused ``slots`` calls
    later. ``encode`` / ``decode`` are the blocking forms. Buffers (device
    and pinned host) are allocated once for ``capacity`` bytes per slot."""

    def __init__(self, capacity: int, chunk_len: int = DEFAULT_CHUNK, lane_count: int = 32,
                 scale_bits: int = 14, device=None, counts_allreduce=None,
                 batch_bytes: int = 32 << 20, slots: int = 2):
        torch = _torch()
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        _check_chunking(chunk_len, lane_count)
        self.device = dev
        self.capacity = int(capacity)
        self.chunk_len, self.lane_count = int(chunk_len), int(lane_count)
        self.slots = [_Slot(torch, dev, self.capacity, chunk_len, lane_count, scale_bits)
                      for _ in range(max(1, int(slots)))]
        self._next = 0
        self._last = None  # slot of the most recent encode (its device table)
        self.counts_allreduce = counts_allreduce
        self.batch_chunks = max(1, batch_bytes // chunk_len)
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        self.trace = None
        self._h2d_tail = None

    # back-compat views of the first slot
    @property
    def codec(self):
        return self.slots[0].codec

    def _batches(self, k: int):
        return [(a, min(k, a + self.batch_chunks)) for a in range(0, k, self.batch_chunks)]

    @staticmethod
    def _event(stream):
        e = _torch().cuda.Event()
        e.record(stream)
        return e

    def _mark(self, name, stream):
        """Timeline probe: with ``self.trace`` a list, record a timing event."""
        if self.trace is not None:
            e = _torch().cuda.Event(enable_timing=True)
            e.record(stream)
            self.trace.append((name, e))

    def _take_slot(self):
        torch = _torch()
        slot = self.slots[self._next]
        self._next = (self._next + 1) % len(self.slots)
        if slot.pending is not None:  # its offsets / payload buffers are about to be reused
            slot.pending.materialize()
            slot.pending = None
        cur = torch.cuda.current_stream(self.device)
        for s in slot.streams():
            s.wait_stream(cur)
            if slot.free is not None:
                s.wait_event(slot.free)
        return slot

    def encode_async(self, h_msg, n: int) -> EncodeJob:
        """Queue the encode of pinned uint8 h_msg[:n] (never blocks the host;
        the payload downloads are issued by the job's materialize())."""
        torch = _torch()
        if n > self.capacity:
            raise ValueError("message larger than codec capacity")
        slot = self._take_slot()
        c = slot.codec
        C, N = c.chunk_len, c.lane_count
        k = n_chunks_for(n, C)
        batches = self._batches(k)
        p_msg = slot.d_msg.data_ptr()
        c.reset_status()
        # phase 1: H2D per batch, histogram as each batch lands
        _lib.check_dev(_lib.lib.ilans_counts_zero_dev(c.counts.data_ptr(), c._s()), "counts")
        self._mark("enc.h2d.start", slot.s_in)
        for i, (k0, k1) in enumerate(batches):
            lo, hi = k0 * C, min(n, k1 * C)
            if i == 1 and self._h2d_tail is not None:
                # uploads are ordered: after its first batch (which fills the
                # link while the previous encode's first payload batch is
                # still coming down) this message waits for the previous
                # round trip's payload upload instead of sharing the link
                # with it (that upload is on the previous decode's critical
                # path)
                slot.s_in.wait_event(self._h2d_tail)
            with torch.cuda.stream(slot.s_in):
                slot.d_msg[lo:hi].copy_(h_msg[lo:hi], non_blocking=True)
            slot.s_comp.wait_event(self._event(slot.s_in))
            _lib.check_dev(_lib.lib.ilans_histogram_u8_dev(p_msg + lo, hi - lo,
                                                           c.counts.data_ptr(), c._s()), "hist")
        if self.counts_allreduce is not None:
            with torch.cuda.stream(slot.s_comp):
                self.counts_allreduce(c.counts)
        self._mark("enc.h2d.end", slot.s_in)
        c.build_table_from_counts()
        self._mark("enc.kernel.start", slot.s_comp)
        # phase 2: one encode launch over all chunks (a chunk is one warp's
        # sequential work, so splitting it would only serialise), then per
        # batch: pack into HBM + copy its word offsets out; as soon as a
        # batch's offsets are on the host its payload D2H is issued.
        c.encode_range(p_msg, n, 0, k, covered=True)  # model from this message's histogram
        self._mark("enc.kernel.end", slot.s_comp)
        if k == 0:
            c.frame_range(n, 0, 0, c.payload.data_ptr())
        ev_off = []
        for k0, k1 in batches:
            c.frame_range(n, k0, k1, c.payload.data_ptr())
            slot.s_out.wait_event(self._event(slot.s_comp))
            with torch.cuda.stream(slot.s_out):
                slot.h_offsets[k0 + 1: k1 + 1].copy_(c.offsets[k0 + 1: k1 + 1],
                                                     non_blocking=True)
            ev_off.append(self._event(slot.s_out))
        slot.h_offsets[:1].zero_()
        c.copy_status(slot.s_out)  # after the last frame, so after the encode kernel
        ev_status = self._event(slot.s_out)
        with torch.cuda.stream(slot.s_out):
            slot.h_states[: k * N].copy_(c.states[: k * N], non_blocking=True)
        ev_states = self._event(slot.s_out)
        self._last = slot
        self.h2d_bytes = n
        slot.pending = EncodeJob(self, slot, n, k, batches, ev_off, ev_status, ev_states, n)
        return slot.pending

    def encode(self, h_msg, n: int):
        """h_msg: pinned uint8 tensor. Returns (payload, offsets, states) as
        views of the pinned host buffers (valid until the slot is reused)."""
        job = self.encode_async(h_msg, n)
        out = job.wait()
        self.d2h_bytes = job.d2h_bytes
        return out

    def decode_async(self, src, h_out, n: int | None = None, h_offsets=None, h_states=None,
                     table: SymbolTable | None = None):
        """Queue the decode into pinned uint8 h_out. ``src`` is an EncodeJob
        of this codec (its device model; payload batches are uploaded as
        soon as their download finished) or a pinned int16 payload with
        ``h_offsets``, ``h_states`` and ``n``, decoded with ``table`` (e.g.
        a ChunkedContainer's) or, without one, with the model of the most
        recent encode."""
        torch = _torch()
        if isinstance(src, EncodeJob):
            slot, job = src.slot, src.materialize()
            n, h_payload, h_offsets, h_states = src.n, src.payload, src.offsets, src.states
            cur = torch.cuda.current_stream(self.device)
            for s in slot.streams():
                s.wait_stream(cur)
        elif table is not None:
            slot, job, h_payload = self._take_slot(), None, src
            slot.codec.build_table_from_freq(table)
            self._last = slot
        else:
            if self._last is None:
                raise RuntimeError("decode needs a device model: encode first or pass table=")
            slot, job, h_payload = self._last, None, src
            # the slot's buffers are reused in place (they hold the model):
            # issue a pending encode's payload downloads first, then order
            # every slot stream after all of its earlier work (the encode
            # kernels on s_comp, the downloads on s_out, earlier decodes)
            if slot.pending is not None:
                slot.pending.materialize()
            fence = [self._event(s) for s in slot.streams()]
            fence.append(self._event(torch.cuda.current_stream(self.device)))
            for s in slot.streams():
                for e in fence:
                    s.wait_event(e)
        c = slot.codec
        C, N = c.chunk_len, c.lane_count
        k = n_chunks_for(n, C)
        offs = h_offsets.numpy()
        words = int(offs[k]) if k else 0
        c.reset_status()
        for s in slot.s_dec:  # table + status reset happen on the compute stream
            s.wait_stream(slot.s_comp)
        with torch.cuda.stream(slot.s_in):
            if job is not None:  # the offsets are on the host already; states may not be
                slot.s_in.wait_event(job.ev_states)
            c.offsets[: k + 1].copy_(h_offsets, non_blocking=True)
            c.states[: k * N].copy_(h_states, non_blocking=True)
        p_pay, p_off = c.payload.data_ptr(), c.offsets.data_ptr()
        p_st, p_out = c.states.data_ptr(), slot.d_out.data_ptr()
        ev_dir = self._event(slot.s_in)
        self._mark("dec.h2d.start", slot.s_in)
        batches = self._batches(k)
        for i, (k0, k1) in enumerate(batches):
            a, b = int(offs[k0]), int(offs[k1])
            with torch.cuda.stream(slot.s_in):
                if job is not None:
                    slot.s_in.wait_event(job.ev_pay[i])
                c.payload[a:b].copy_(h_payload[a:b], non_blocking=True)
            s_dec = slot.s_dec[i % len(slot.s_dec)]
            s_dec.wait_event(self._event(slot.s_in))
            s_dec.wait_event(ev_dir)
            c.decode_range(p_out, n, k0, k1, p_pay, p_off, p_st, stream=s_dec.cuda_stream)
            slot.s_out.wait_event(self._event(s_dec))
            lo, hi = k0 * C, min(n, k1 * C)
            with torch.cuda.stream(slot.s_out):
                h_out[lo:hi].copy_(slot.d_out[lo:hi], non_blocking=True)
        self._mark("dec.h2d.end", slot.s_in)
        self._h2d_tail = self._event(slot.s_in)
        for s in (slot.s_in, *slot.s_dec):
            slot.s_out.wait_stream(s)
        self._mark("dec.d2h.end", slot.s_out)
        c.copy_status(slot.s_out)
        ev_done = self._event(slot.s_out)
        slot.s_comp.wait_event(ev_done)
        slot.free = ev_done
        h2d, d2h = 2 * words + 8 * (k + 1) + 4 * k * N, n
        self.h2d_bytes, self.d2h_bytes = h2d, d2h
        return DecodeJob(slot, h_out[:n], ev_done, h2d, d2h)

    def decode(self, h_payload, h_offsets, h_states, n: int, h_out,
               table: SymbolTable | None = None):
        """Decode into pinned uint8 tensor h_out (model: ``table``, else the
        most recent encode's)."""
        return self.decode_async(h_payload, h_out, n, h_offsets, h_states, table).wait()
