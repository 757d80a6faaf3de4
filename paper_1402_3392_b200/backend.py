"""Kernel backend: the drop-in for the reference plugin boundary.

Reference: pkg/src/ilans/backend.py:16-78 -- a frozen ``Backend`` with the
three word16 kernel callables, resolved by ``get(name)`` with the default
chosen by ``ILANS_BACKEND``. Here there is exactly one backend, "b200",
whose callables have the reference signatures (_core.pyx:14, :46-47,
:130-131) and run on the B200 through libilans_b200.so. "ext" resolves to
it too (it is the compiled backend); the reference's pure-Python backend is
not shipped -- its behaviour is the test oracle (oracle/), never a runtime
fallback.
"""

from __future__ import annotations

import ctypes
import os
import warnings
import weakref
from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _lib


@dataclass(frozen=True)
class Backend:
    name: str
    encode_interleaved_u16: Callable
    decode_interleaved_u16: Callable
    decode_lanes_u16: Callable


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


# Host addresses of the model arrays: drop-in callers pass the same table
# views (SymbolTable's cached freq_u32 / cum_u32 / slot_u8) on every call,
# and a.ctypes.data costs ~1 us per array per call under the GIL.
_ptr_cache: dict[int, tuple] = {}


def _tptr(a: np.ndarray) -> int:
    # keyed by identity (a weak reference guards against a reused id) and
    # size (an in-place resize that moves the buffer changes it)
    hit = _ptr_cache.get(id(a))
    if hit is not None and hit[0]() is a and hit[2] == a.size:
        return hit[1]
    p = a.ctypes.data
    if len(_ptr_cache) > 64:
        _ptr_cache.clear()
    try:
        _ptr_cache[id(a)] = (weakref.ref(a), p, a.size)
    except TypeError:  # not weak-referenceable: no caching
        pass
    return p


def encode_interleaved_u16(msg, freq, cum, scale_bits: int, n_lanes: int):
    """Backward interleaved encode on the B200. Returns (payload u16 array in
    decoder read order, final lane states u32 array) -- contract of
    _pure.encode_interleaved_u16 (_pure.py:15-39)."""
    m = np.ascontiguousarray(msg, dtype=np.uint8)
    f = _u32(freq)
    c = _u32(cum)
    if len(c) < len(f) + 1:
        raise ValueError("cum must have len(freq) + 1 entries")
    payload = np.empty(max(1, len(m)), dtype=np.uint16)
    states = np.empty(n_lanes, dtype=np.uint32) if n_lanes > 0 else np.empty(0, np.uint32)
    words = ctypes.c_int64(0)
    st = _lib.Status()
    rc = _lib.lib.ilans_encode_interleaved_u16(
        _lib.ptr(m), len(m), _tptr(f), len(f), _tptr(c), int(scale_bits), int(n_lanes),
        _lib.ptr(payload), ctypes.byref(words), _lib.ptr(states), ctypes.byref(st))
    _lib.raise_for(rc, st, "encode_interleaved_u16")
    return payload[: words.value].copy(), states


def encode_interleaved_u16_stats(msg, freq, cum, scale_bits: int, n_lanes: int):
    """encode_interleaved_u16 + the kernel-measured most digits one symbol
    spilled (RenormStats, rans.py:235-263): (payload, states, max_digits)."""
    m = np.ascontiguousarray(msg, dtype=np.uint8)
    f = _u32(freq)
    c = _u32(cum)
    if len(c) < len(f) + 1:
        raise ValueError("cum must have len(freq) + 1 entries")
    payload = np.empty(max(1, len(m)), dtype=np.uint16)
    states = np.empty(n_lanes, dtype=np.uint32) if n_lanes > 0 else np.empty(0, np.uint32)
    words = ctypes.c_int64(0)
    st = _lib.Status()
    rc = _lib.lib.ilans_encode_interleaved_u16_stats(
        _lib.ptr(m), len(m), _lib.ptr(f), len(f), _lib.ptr(c), int(scale_bits), int(n_lanes),
        _lib.ptr(payload), ctypes.byref(words), _lib.ptr(states), ctypes.byref(st))
    _lib.raise_for(rc, st, "encode_interleaved_u16")
    return payload[: words.value].copy(), states, int(st.max_digits)


def _decode(fn, payload, states, slot_sym, freq, cum, scale_bits, msg_len, n_lanes,
            with_stats=False):
    pay = np.ascontiguousarray(payload, dtype=np.uint16)
    xs = np.array(states, dtype=np.uint32)  # copied: inputs are never mutated
    slot = np.ascontiguousarray(slot_sym, dtype=np.uint8)
    f = _u32(freq)
    c = _u32(cum)
    if len(c) < len(f) + 1:
        raise ValueError("cum must have len(freq) + 1 entries")
    if len(xs) < n_lanes:
        raise ValueError("one state per lane required")
    out = np.empty(max(1, msg_len), dtype=np.uint8)
    consumed = ctypes.c_int64(0)
    st = _lib.Status()
    rc = fn(_lib.ptr(pay), len(pay), _lib.ptr(xs), _tptr(slot), len(slot), _tptr(f),
            _tptr(c), len(f), int(scale_bits), int(msg_len), int(n_lanes), _lib.ptr(out),
            ctypes.byref(consumed), ctypes.byref(st))
    _lib.raise_for(rc, st, "decode")
    if with_stats:
        return out[:msg_len], int(consumed.value), int(st.max_digits)
    return out[:msg_len], int(consumed.value)


_dec_serial = _lib.lib.ilans_decode_interleaved_u16
_dec_lanes = _lib.lib.ilans_decode_lanes_u16


def decode_interleaved_u16(payload, states, slot_sym, freq, cum, scale_bits, msg_len, n_lanes):
    """Forward interleaved decode on the B200. Returns (message u8 array,
    words read) -- contract of _pure.decode_interleaved_u16 (_pure.py:42-66)."""
    return _decode(_dec_serial, payload, states, slot_sym, freq, cum, scale_bits, msg_len,
                   n_lanes)


def decode_interleaved_u16_stats(payload, states, slot_sym, freq, cum, scale_bits, msg_len,
                                 n_lanes):
    """decode_interleaved_u16 + the kernel-measured most digits one symbol
    refilled: (message, words read, max_digits)."""
    return _decode(_lib.lib.ilans_decode_interleaved_u16_stats, payload, states, slot_sym, freq,
                   cum, scale_bits, msg_len, n_lanes, with_stats=True)


def decode_lanes_u16(payload, states, slot_sym, freq, cum, scale_bits, msg_len, n_lanes):
    """Group-at-a-time lane decode on the B200; byte-identical to
    decode_interleaved_u16 (_pure.py:69-101). At most 32 lanes."""
    if n_lanes > 32:
        raise ValueError("at most 32 lanes")
    return _decode(_dec_lanes, payload, states, slot_sym, freq, cum, scale_bits, msg_len,
                   n_lanes)


# ---------------------------------------------------------------------------
# BYTE8 (8-bit digits, L = 2^23): the reference runs this variant on its
# scalar Python path (interleave.py:155-179); here it is a GPU kernel too.
# Not part of the reference Backend (whose fields are the word16 kernels),
# so these return one extra value: the most digits moved for one symbol
# (what RenormStats.max_*_digits records).
# ---------------------------------------------------------------------------
def encode_interleaved_u8(msg, freq, cum, scale_bits: int, n_lanes: int):
    """Backward byte8 encode on the B200 -> (payload u8, states u32, max spills)."""
    m = np.ascontiguousarray(msg, dtype=np.uint8)
    f = _u32(freq)
    c = _u32(cum)
    if len(c) < len(f) + 1:
        raise ValueError("cum must have len(freq) + 1 entries")
    payload = np.empty(max(1, 3 * len(m)), dtype=np.uint8)
    states = np.empty(n_lanes, dtype=np.uint32)
    nbytes = ctypes.c_int64(0)
    st = _lib.Status()
    rc = _lib.lib.ilans_encode_interleaved_u8(
        _lib.ptr(m), len(m), _lib.ptr(f), len(f), _lib.ptr(c), int(scale_bits), int(n_lanes),
        _lib.ptr(payload), ctypes.byref(nbytes), _lib.ptr(states), ctypes.byref(st))
    _lib.raise_for(rc, st, "encode_interleaved_u8")
    return payload[: nbytes.value].copy(), states, int(st.max_digits)


def decode_interleaved_u8(payload, states, slot_sym, freq, cum, scale_bits, msg_len, n_lanes):
    """Forward byte8 decode on the B200 -> (message u8, digits read, max refills)."""
    pay = np.ascontiguousarray(payload, dtype=np.uint8)
    xs = np.array(states, dtype=np.uint32)
    slot = np.ascontiguousarray(slot_sym, dtype=np.uint8)
    f = _u32(freq)
    c = _u32(cum)
    out = np.empty(max(1, msg_len), dtype=np.uint8)
    consumed = ctypes.c_int64(0)
    st = _lib.Status()
    rc = _lib.lib.ilans_decode_interleaved_u8(
        _lib.ptr(pay), len(pay), _lib.ptr(xs), _lib.ptr(slot), len(slot), _lib.ptr(f),
        _lib.ptr(c), len(f), int(scale_bits), int(msg_len), int(n_lanes), _lib.ptr(out),
        ctypes.byref(consumed), ctypes.byref(st))
    _lib.raise_for(rc, st, "decode_u8")
    return out[:msg_len], int(consumed.value), int(st.max_digits)


def decode_trace_u16(payload, states, slot_sym, freq, cum, scale_bits, msg_len, n_lanes,
                     byte8: bool = False):
    """Instrumented device decode (ilans_decode_trace_u16): returns
    (msg, trace_states [groups, N], trace_pos [groups], groups_done,
    consumed, error) where error is the exception the plain decode would
    raise (TruncatedStreamError) or None; everything up to the failing group
    is filled in, so step generators can yield before raising. byte8=True
    traces the byte8 decoder (ilans_decode_trace_u8) instead."""
    pay = np.ascontiguousarray(payload, dtype=np.uint8 if byte8 else np.uint16)
    xs = np.array(states, dtype=np.uint32)
    slot = np.ascontiguousarray(slot_sym, dtype=np.uint8)
    f = _u32(freq)
    c = _u32(cum)
    groups = -(-msg_len // n_lanes) if msg_len else 0
    out = np.zeros(max(1, msg_len), dtype=np.uint8)
    tstates = np.zeros((max(1, groups), n_lanes), dtype=np.uint32)
    tpos = np.zeros(max(1, groups), dtype=np.uint64)
    done = ctypes.c_int64(0)
    consumed = ctypes.c_int64(0)
    st = _lib.Status()
    fn = _lib.lib.ilans_decode_trace_u8 if byte8 else _lib.lib.ilans_decode_trace_u16
    rc = fn(
        _lib.ptr(pay), len(pay), _lib.ptr(xs), _lib.ptr(slot), len(slot), _lib.ptr(f),
        _lib.ptr(c), len(f), int(scale_bits), int(msg_len), int(n_lanes), _lib.ptr(out),
        _lib.ptr(tstates), _lib.ptr(tpos), ctypes.byref(done), ctypes.byref(consumed),
        ctypes.byref(st))
    err = None
    if rc in (_lib.ERR_TRUNCATED, _lib.ERR_FORMAT):
        try:
            _lib.raise_for(rc, st, "decode")
        except Exception as exc:  # noqa: BLE001 -- handed back to the generator
            err = exc
    else:
        _lib.raise_for(rc, st, "decode")
    g = int(done.value)
    return out[:msg_len], tstates[:g], tpos[:g], g, int(consumed.value), err


B200 = Backend("b200", encode_interleaved_u16, decode_interleaved_u16, decode_lanes_u16)
EXT = B200  # the compiled backend, under the reference's name for it
PURE = None  # not shipped: the pure-Python kernels are the test oracle


def _pick_default() -> Backend:
    forced = os.environ.get("ILANS_BACKEND", "").strip().lower()
    if forced in ("", "b200", "ext", "auto"):
        return B200
    warnings.warn(
        f"ILANS_BACKEND={forced!r} is not available in ilans-b200; using 'b200'",
        RuntimeWarning,
    )
    return B200


ACTIVE = _pick_default()


def get(name: str | None = None) -> Backend:
    """Resolve a backend by name; None / "auto" mean the import-time default."""
    if name is None or name == "auto":
        return ACTIVE
    if name in ("b200", "ext"):
        return B200
    if name == "pure":
        raise ValueError("the pure-Python backend is not part of ilans-b200 (no CPU fallback)")
    raise ValueError(f"unknown backend {name!r}")


def available() -> list[str]:
    return ["b200"]


# ---------------------------------------------------------------------------
# Any RenormVariant (the reference's scalar path for variants other than
# word16 / byte8, interleave.py:155-179): digits as one array element each.
# ---------------------------------------------------------------------------
def _digit_dtype(variant):
    return np.uint16 if variant.digit_bits > 8 else np.uint8


def encode_interleaved_var(msg, table, n_lanes: int, variant):
    """Backward encode with ``variant``'s digits on the B200 -> (payload in
    read order (u8 for digits <= 8 bits, else u16), states, max digits)."""
    m = np.ascontiguousarray(msg, dtype=np.uint8)
    f, c = table.freq_u32, table.cum_u32
    kmax = -(-table.scale_bits // variant.digit_bits) + 1
    digits = np.empty(max(1, len(m) * kmax), dtype=np.uint16)
    states = np.empty(n_lanes, dtype=np.uint32)
    count = ctypes.c_int64(0)
    st = _lib.Status()
    rc = _lib.lib.ilans_encode_interleaved_var(
        _lib.ptr(m), len(m), _lib.ptr(f), len(f), _lib.ptr(c), int(table.scale_bits),
        int(n_lanes), int(variant.digit_bits), int(variant.lower_bound), _lib.ptr(digits),
        len(digits), ctypes.byref(count), _lib.ptr(states), ctypes.byref(st))
    if rc == _lib.ERR_UNSUPPORTED:
        from .errors import UnsupportedVariantError

        raise UnsupportedVariantError(st.message.decode(errors="replace"))
    _lib.raise_for(rc, st, "encode_interleaved_var")
    return digits[: count.value].astype(_digit_dtype(variant)), states, int(st.max_digits)


def decode_interleaved_var(payload, states, table, msg_len: int, n_lanes: int, variant,
                           trace: bool = False):
    """Forward decode with ``variant``'s digits on the B200 -> (message,
    digits read, max digits); trace=True -> (message, trace states [groups,
    N], read position per group, groups done, digits read, error or None)
    for the step generator."""
    pay = np.ascontiguousarray(payload, dtype=np.uint16)
    xs = np.array(states, dtype=np.uint32)
    f, c, slot = table.freq_u32, table.cum_u32, table.slot_u8
    out = np.zeros(max(1, msg_len), dtype=np.uint8)
    consumed = ctypes.c_int64(0)
    st = _lib.Status()
    groups = -(-msg_len // n_lanes) if msg_len else 0
    tstates = np.zeros((max(1, groups), n_lanes), dtype=np.uint32) if trace else None
    tpos = np.zeros(max(1, groups), dtype=np.uint64) if trace else None
    done = ctypes.c_int64(0)
    rc = _lib.lib.ilans_decode_interleaved_var(
        _lib.ptr(pay), len(pay), _lib.ptr(xs), _lib.ptr(slot), len(slot), _lib.ptr(f), _lib.ptr(c),
        len(f), int(table.scale_bits), int(msg_len), int(n_lanes), int(variant.digit_bits),
        int(variant.lower_bound), _lib.ptr(out), ctypes.byref(consumed),
        _lib.ptr(tstates) if trace else None, _lib.ptr(tpos) if trace else None,
        ctypes.byref(done) if trace else None, ctypes.byref(st))
    if rc == _lib.ERR_UNSUPPORTED:
        from .errors import UnsupportedVariantError

        raise UnsupportedVariantError(st.message.decode(errors="replace"))
    if trace:
        err = None
        if rc in (_lib.ERR_TRUNCATED, _lib.ERR_FORMAT):
            try:
                _lib.raise_for(rc, st, "decode")
            except Exception as exc:  # noqa: BLE001 -- handed back to the generator
                err = exc
        else:
            _lib.raise_for(rc, st, "decode")
        return out[:msg_len], tstates, tpos, int(done.value), int(st.consumed), err
    _lib.raise_for(rc, st, "decode_interleaved_var")
    return out[:msg_len], int(consumed.value), int(st.max_digits)

