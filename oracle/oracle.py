"""ctypes wrapper over oracle/rans_oracle.c -- the CPU checker.

TEST INFRASTRUCTURE ONLY. Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, always as the thing results
are COMPARED AGAINST, never as the thing measured or shipped. The product
package (paper_1402_3392_b200) never imports this module.

The function signatures mirror the reference kernel boundary
(pkg/src/ilans/_core.pyx:14, :46-47, :130-131) so tests can call the oracle
and the product backend with the same arguments.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "liboracle.so"
REF_DIR = HERE / "_ref"

OK, ERR_VALUE, ERR_UNENCODABLE, ERR_TRUNCATED, ERR_FORMAT = 0, 1, 2, 3, 6
KIND_NAMES = {ERR_VALUE: "value", ERR_UNENCODABLE: "unencodable", ERR_TRUNCATED: "truncated",
              ERR_FORMAT: "format"}


class OracleError(Exception):
    def __init__(self, kind: int, msg: str = ""):
        super().__init__(f"{KIND_NAMES.get(kind, kind)}: {msg}")
        self.kind = KIND_NAMES.get(kind, str(kind))


def build() -> Path:
    src = HERE / "rans_oracle.c"
    if not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        LIB_PATH.parent.mkdir(parents=True, exist_ok=True)
        subprocess.run(
            ["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-o", str(LIB_PATH), str(src)],
            check=True,
        )
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(str(build()))
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def histogram(msg) -> tuple[np.ndarray, int]:
    """np.bincount(msg, minlength=256) as u64 plus alphabet = max + 1."""
    m = np.ascontiguousarray(msg, dtype=np.uint8)
    counts = np.zeros(256, dtype=np.uint64)
    alpha = lib().orc_histogram_u8(_p(m), ctypes.c_int64(len(m)), _p(counts))
    return counts, int(alpha)


def quantize(counts, scale_bits: int) -> list[int]:
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.uint64))
    out = np.zeros(max(1, len(c)), dtype=np.uint32)
    rc = lib().orc_quantize(_p(c), ctypes.c_int(len(c)), ctypes.c_int(scale_bits), _p(out))
    if rc:
        raise OracleError(rc, "quantize")
    return out[: len(c)].tolist()


def table_views(freqs, scale_bits: int):
    """(freq u32, cum u32[n+1], slot u8[m]) as rans.SymbolTable builds them
    (rans.py:115-121, :136-146)."""
    f = np.asarray(freqs, dtype=np.uint32)
    cum = np.zeros(len(f) + 1, dtype=np.uint32)
    cum[1:] = np.cumsum(f, dtype=np.uint64).astype(np.uint32)
    slot = np.repeat(np.arange(len(f), dtype=np.uint8), f.astype(np.int64))
    assert len(slot) == 1 << scale_bits
    return f, cum, slot


def encode_interleaved_u16(msg, freq, cum, scale_bits: int, n_lanes: int):
    m = np.ascontiguousarray(msg, dtype=np.uint8)
    f = np.zeros(256, dtype=np.uint32)
    f[: len(freq)] = np.asarray(freq, dtype=np.uint32)
    c = np.zeros(257, dtype=np.uint32)
    c[: len(cum)] = np.asarray(cum, dtype=np.uint32)
    scratch = np.empty(max(1, len(m)), dtype=np.uint16)
    states = np.empty(n_lanes, dtype=np.uint32)
    words = ctypes.c_int64(0)
    bad_i = ctypes.c_int64(-1)
    bad_s = ctypes.c_int(-1)
    rc = lib().orc_encode_u16(
        _p(m), ctypes.c_int64(len(m)), _p(f), _p(c), ctypes.c_int(scale_bits),
        ctypes.c_int(n_lanes), _p(scratch), _p(scratch), ctypes.byref(words), _p(states),
        ctypes.byref(bad_i), ctypes.byref(bad_s),
    )
    if rc:
        raise OracleError(rc, f"symbol {bad_s.value} has frequency 0")
    return scratch[: words.value].copy(), states


def _decode(fn, payload, states, slot_sym, freq, cum, scale_bits, msg_len, n_lanes):
    pay = np.ascontiguousarray(payload, dtype=np.uint16)
    xs = np.array(states, dtype=np.uint32)
    slot = np.ascontiguousarray(slot_sym, dtype=np.uint8)
    f = np.zeros(256, dtype=np.uint32)
    f[: len(freq)] = np.asarray(freq, dtype=np.uint32)
    c = np.zeros(257, dtype=np.uint32)
    c[: len(cum)] = np.asarray(cum, dtype=np.uint32)
    out = np.empty(msg_len, dtype=np.uint8)
    consumed = ctypes.c_int64(0)
    rc = fn(
        _p(pay), ctypes.c_int64(len(pay)), _p(xs), _p(slot), _p(f), _p(c),
        ctypes.c_int(scale_bits), ctypes.c_int64(msg_len), ctypes.c_int(n_lanes), _p(out),
        ctypes.byref(consumed),
    )
    if rc:
        raise OracleError(rc, "decode")
    return out, int(consumed.value), xs


def decode_interleaved_u16(payload, states, slot_sym, freq, cum, scale_bits, msg_len, n_lanes):
    out, consumed, _ = _decode(lib().orc_decode_u16, payload, states, slot_sym, freq, cum,
                               scale_bits, msg_len, n_lanes)
    return out, consumed


def decode_lanes_u16(payload, states, slot_sym, freq, cum, scale_bits, msg_len, n_lanes):
    out, consumed, _ = _decode(lib().orc_decode_lanes_u16, payload, states, slot_sym, freq,
                               cum, scale_bits, msg_len, n_lanes)
    return out, consumed


def decode_final_states(payload, states, slot_sym, freq, cum, scale_bits, msg_len, n_lanes):
    """Lane states after a full decode (all return to L on valid input)."""
    _, _, xs = _decode(lib().orc_decode_u16, payload, states, slot_sym, freq, cum,
                       scale_bits, msg_len, n_lanes)
    return xs


def _pad_tables(freq, cum):
    f = np.zeros(256, dtype=np.uint32)
    f[: len(freq)] = np.asarray(freq, dtype=np.uint32)
    c = np.zeros(257, dtype=np.uint32)
    c[: len(cum)] = np.asarray(cum, dtype=np.uint32)
    return f, c


def encode_interleaved_u8(msg, freq, cum, scale_bits: int, n_lanes: int):
    """BYTE8 scalar encode (interleave.py:155-165): (payload u8, states u32)."""
    m = np.ascontiguousarray(msg, dtype=np.uint8)
    f, c = _pad_tables(freq, cum)
    scratch = np.empty(max(1, 4 * len(m)), dtype=np.uint8)
    out = np.empty(max(1, 4 * len(m)), dtype=np.uint8)
    states = np.empty(n_lanes, dtype=np.uint32)
    nb = ctypes.c_int64(0)
    rc = lib().orc_encode_u8(_p(m), ctypes.c_int64(len(m)), _p(f), _p(c),
                             ctypes.c_int(scale_bits), ctypes.c_int(n_lanes), _p(scratch),
                             _p(out), ctypes.byref(nb), _p(states))
    if rc:
        raise OracleError(rc, "encode_u8")
    return out[: nb.value].copy(), states


def decode_interleaved_u8(payload, states, slot_sym, freq, cum, scale_bits, msg_len, n_lanes):
    """BYTE8 scalar decode (interleave.py:168-179): (message, digits read)."""
    out, used, _ = decode_u8_full(payload, states, slot_sym, freq, cum, scale_bits, msg_len,
                                  n_lanes)
    return out, used


def decode_u8_full(payload, states, slot_sym, freq, cum, scale_bits, msg_len, n_lanes):
    """BYTE8 scalar decode returning (message, digits read, lane states)."""
    pay = np.ascontiguousarray(payload, dtype=np.uint8)
    xs = np.array(states, dtype=np.uint32)
    slot = np.ascontiguousarray(slot_sym, dtype=np.uint8)
    f, c = _pad_tables(freq, cum)
    out = np.empty(max(1, msg_len), dtype=np.uint8)
    consumed = ctypes.c_int64(0)
    rc = lib().orc_decode_u8(_p(pay), ctypes.c_int64(len(pay)), _p(xs), _p(slot), _p(f), _p(c),
                             ctypes.c_int(scale_bits), ctypes.c_int64(msg_len),
                             ctypes.c_int(n_lanes), _p(out), ctypes.byref(consumed))
    if rc:
        raise OracleError(rc, "decode_u8")
    return out[:msg_len], int(consumed.value), xs


def encode_chunks_u16(msg, chunk_len: int, freq, cum, scale_bits: int, n_lanes: int):
    """Chunk framing oracle: per chunk an independent N-lane stream.
    Returns (payload u16[total], word_offsets u64[n_chunks+1], states u32[n_chunks, N])."""
    m = np.ascontiguousarray(msg, dtype=np.uint8)
    n = len(m)
    n_chunks = 0 if n == 0 else -(-n // chunk_len)
    f = np.zeros(256, dtype=np.uint32)
    f[: len(freq)] = np.asarray(freq, dtype=np.uint32)
    c = np.zeros(257, dtype=np.uint32)
    c[: len(cum)] = np.asarray(cum, dtype=np.uint32)
    scratch = np.empty(max(1, chunk_len), dtype=np.uint16)
    payload = np.empty(max(1, n), dtype=np.uint16)
    offsets = np.zeros(n_chunks + 1, dtype=np.uint64)
    states = np.empty((max(1, n_chunks), n_lanes), dtype=np.uint32)
    rc = lib().orc_encode_chunks_u16(
        _p(m), ctypes.c_int64(n), ctypes.c_int64(chunk_len), _p(f), _p(c),
        ctypes.c_int(scale_bits), ctypes.c_int(n_lanes), _p(scratch), _p(payload),
        _p(offsets), _p(states),
    )
    if rc:
        raise OracleError(rc, "encode_chunks")
    return payload[: int(offsets[-1])].copy(), offsets, states[:n_chunks].copy()


def decode_chunks_u16(payload, offsets, states, slot_sym, freq, cum, scale_bits, n,
                      chunk_len, n_lanes):
    pay = np.ascontiguousarray(payload, dtype=np.uint16)
    if len(pay) == 0:
        pay = np.zeros(1, dtype=np.uint16)
    offs = np.ascontiguousarray(offsets, dtype=np.uint64)
    st = np.ascontiguousarray(states, dtype=np.uint32)
    slot = np.ascontiguousarray(slot_sym, dtype=np.uint8)
    f = np.zeros(256, dtype=np.uint32)
    f[: len(freq)] = np.asarray(freq, dtype=np.uint32)
    c = np.zeros(257, dtype=np.uint32)
    c[: len(cum)] = np.asarray(cum, dtype=np.uint32)
    out = np.empty(max(1, n), dtype=np.uint8)
    rc = lib().orc_decode_chunks_u16(
        _p(pay), _p(offs), _p(st), _p(slot), _p(f), _p(c), ctypes.c_int(scale_bits),
        ctypes.c_int64(n), ctypes.c_int64(chunk_len), ctypes.c_int(n_lanes), _p(out),
    )
    if rc:
        raise OracleError(rc, "decode_chunks")
    return out[:n]


def reference_ilans():
    """Import the unmodified reference package built by oracle/build_ref.sh
    (oracle/_ref/ilans with its compiled _core), or None if absent."""
    import importlib
    import sys

    if not (REF_DIR / "ilans" / "__init__.py").exists():
        return None
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    os.environ.setdefault("ILANS_BACKEND", "ext")
    return importlib.import_module("ilans")
