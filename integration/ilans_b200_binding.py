"""ctypes binding of libilans_b200.so: the B200 word16 kernels.

This is the reference-side module a maintainer adds as
``pkg/src/ilans/_b200.py``; it replaces the three
Cython kernels of ``pkg/src/ilans/_core.pyx`` (encode_interleaved_u16 :14,
decode_interleaved_u16 :46-47, decode_lanes_u16 :130-131) with the C ABI of
``include/ilans_b200.h`` (ilans_encode_interleaved_u16,
ilans_decode_interleaved_u16, ilans_decode_lanes_u16). Same signatures,
same return values, same exception types. ``integration/install_into_reference.py``
installs it into a copy of the reference and registers ``Backend("b200")``.
"""
import atexit
import ctypes
import os

import numpy as np

from .errors import TruncatedStreamError, UnencodableSymbolError

_lib = ctypes.CDLL(os.environ.get("ILANS_B200_LIB", "libilans_b200.so"))
# the library's per-thread contexts skip CUDA teardown once the process exits
atexit.register(_lib.ilans_process_exiting)


class _Status(ctypes.Structure):  # ilans_status (include/ilans_b200.h)
    _fields_ = [("code", ctypes.c_int32), ("cuda_error", ctypes.c_int32),
                ("stream", ctypes.c_int64), ("index", ctypes.c_int64),
                ("symbol", ctypes.c_int32), ("max_digits", ctypes.c_int32),
                ("consumed", ctypes.c_int64), ("message", ctypes.c_char * 128)]


_P, _I32, _I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
_lib.ilans_encode_interleaved_u16.argtypes = [_P, _I64, _P, _I32, _P, _I32, _I32, _P, _P, _P,
                                              ctypes.POINTER(_Status)]
for _f in (_lib.ilans_decode_interleaved_u16, _lib.ilans_decode_lanes_u16):
    _f.argtypes = [_P, _I64, _P, _P, _I64, _P, _P, _I32, _I32, _I64, _I32, _P, _P,
                   ctypes.POINTER(_Status)]


def _raise(rc, st):
    if rc == 0:
        return
    msg = st.message.decode(errors="replace")
    if rc == 3:
        raise TruncatedStreamError(msg)
    if rc == 2:
        raise UnencodableSymbolError(msg)
    if rc == 1:
        raise ValueError(msg)
    raise RuntimeError(f"ilans_b200 error {rc}: {msg}")


def _p(a):
    return a.ctypes.data


def encode_interleaved_u16(msg, freq, cum, scale_bits, n_lanes):
    m = np.ascontiguousarray(msg, np.uint8)
    f = np.ascontiguousarray(freq, np.uint32)
    c = np.ascontiguousarray(cum, np.uint32)
    out = np.empty(max(1, len(m)), np.uint16)  # word16: at most one word per symbol
    states = np.empty(n_lanes, np.uint32)
    words, st = ctypes.c_int64(), _Status()
    _raise(_lib.ilans_encode_interleaved_u16(_p(m), len(m), _p(f), len(f), _p(c), scale_bits,
                                             n_lanes, _p(out), ctypes.byref(words), _p(states),
                                             ctypes.byref(st)), st)
    return out[:words.value].copy(), states


def _decode(fn, payload, states, slot_sym, freq, cum, scale_bits, msg_len, n_lanes):
    p = np.ascontiguousarray(payload, np.uint16)
    x = np.array(states, np.uint32)
    s = np.ascontiguousarray(slot_sym, np.uint8)
    f = np.ascontiguousarray(freq, np.uint32)
    c = np.ascontiguousarray(cum, np.uint32)
    out = np.empty(max(1, msg_len), np.uint8)
    used, st = ctypes.c_int64(), _Status()
    _raise(fn(_p(p), len(p), _p(x), _p(s), len(s), _p(f), _p(c), len(f), scale_bits, msg_len,
              n_lanes, _p(out), ctypes.byref(used), ctypes.byref(st)), st)
    return out[:msg_len], used.value


def decode_interleaved_u16(payload, states, slot_sym, freq, cum, scale_bits, msg_len, n_lanes):
    return _decode(_lib.ilans_decode_interleaved_u16, payload, states, slot_sym, freq, cum,
                   scale_bits, msg_len, n_lanes)


def decode_lanes_u16(payload, states, slot_sym, freq, cum, scale_bits, msg_len, n_lanes):
    return _decode(_lib.ilans_decode_lanes_u16, payload, states, slot_sym, freq, cum,
                   scale_bits, msg_len, n_lanes)
