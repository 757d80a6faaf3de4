"""ctypes binding of libilans_b200.so (include/ilans_b200.h).

This is the ONLY compute path of the package: every encode / decode /
histogram / quantize call ends in an sm_100a kernel of libilans_b200.so.
There is no CPU fallback. If the library is missing, importing this module
raises ImportError; if no CUDA device is visible, each call raises
RuntimeError (ILANS_ERR_CUDA).
"""

from __future__ import annotations

import atexit
import ctypes
import os
from pathlib import Path

import numpy as np

from .errors import (
    FormatError,
    ScheduleError,
    TruncatedStreamError,
    UnencodableSymbolError,
    UnsupportedVariantError,
)

LIB_PATH = Path(os.environ.get("ILANS_B200_LIB", Path(__file__).resolve().parent / "libilans_b200.so"))

(OK, ERR_VALUE, ERR_UNENCODABLE, ERR_TRUNCATED, ERR_UNSUPPORTED, ERR_CUDA, ERR_FORMAT,
 ERR_SCHEDULE) = range(8)
MUX_RANS, MUX_RAW = 0, 1


class Status(ctypes.Structure):
    _fields_ = [
        ("code", ctypes.c_int32),
        ("cuda_error", ctypes.c_int32),
        ("stream", ctypes.c_int64),
        ("index", ctypes.c_int64),
        ("symbol", ctypes.c_int32),
        ("max_digits", ctypes.c_int32),
        ("consumed", ctypes.c_int64),
        ("message", ctypes.c_char * 128),
    ]


class MuxStream(ctypes.Structure):
    """ilans_mux_stream: one multiplexed stream's coder parameters."""

    _fields_ = [
        ("kind", ctypes.c_int32),
        ("nbytes", ctypes.c_int32),
        ("digit_bits", ctypes.c_int32),
        ("scale_bits", ctypes.c_int32),
        ("lower_bound", ctypes.c_uint32),
        ("n_sym", ctypes.c_int32),
        ("freq_off", ctypes.c_int64),
        ("cum_off", ctypes.c_int64),
        ("slot_off", ctypes.c_int64),
    ]


def _load() -> ctypes.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is not built; run `python paper_1402_3392_b200/build.py` "
            "(the B200 codec has no CPU fallback)"
        )
    return ctypes.CDLL(str(LIB_PATH))


lib = _load()

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_st = ctypes.POINTER(Status)

# (name, restype, argtypes) -- one row per prototype in include/ilans_b200.h
PROTOTYPES = [
    ("ilans_abi_version", ctypes.c_int, []),
    ("ilans_device_count", ctypes.c_int, []),
    ("ilans_set_device", ctypes.c_int, [ctypes.c_int, _st]),
    ("ilans_launch_count", ctypes.c_uint64, []),
    ("ilans_process_exiting", None, []),
    ("ilans_encode_interleaved_u16", ctypes.c_int,
     [_vp, _i64, _vp, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _st]),
    ("ilans_decode_interleaved_u16", ctypes.c_int,
     [_vp, _i64, _vp, _vp, _i64, _vp, _vp, _i32, _i32, _i64, _i32, _vp, _vp, _st]),
    ("ilans_decode_lanes_u16", ctypes.c_int,
     [_vp, _i64, _vp, _vp, _i64, _vp, _vp, _i32, _i32, _i64, _i32, _vp, _vp, _st]),
    ("ilans_encode_interleaved_u16_stats", ctypes.c_int,
     [_vp, _i64, _vp, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _st]),
    ("ilans_decode_interleaved_u16_stats", ctypes.c_int,
     [_vp, _i64, _vp, _vp, _i64, _vp, _vp, _i32, _i32, _i64, _i32, _vp, _vp, _st]),
    ("ilans_encode_interleaved_var", ctypes.c_int,
     [_vp, _i64, _vp, _i32, _vp, _i32, _i32, _i32, ctypes.c_uint32, _vp, _i64, _vp, _vp, _st]),
    ("ilans_decode_interleaved_var", ctypes.c_int,
     [_vp, _i64, _vp, _vp, _i64, _vp, _vp, _i32, _i32, _i64, _i32, _i32, ctypes.c_uint32, _vp,
      _vp, _vp, _vp, _vp, _st]),
    ("ilans_decode_trace_u16", ctypes.c_int,
     [_vp, _i64, _vp, _vp, _i64, _vp, _vp, _i32, _i32, _i64, _i32, _vp, _vp, _vp, _vp, _vp,
      _st]),
    ("ilans_encode_interleaved_u8", ctypes.c_int,
     [_vp, _i64, _vp, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _st]),
    ("ilans_decode_interleaved_u8", ctypes.c_int,
     [_vp, _i64, _vp, _vp, _i64, _vp, _vp, _i32, _i32, _i64, _i32, _vp, _vp, _st]),
    ("ilans_decode_trace_u8", ctypes.c_int,
     [_vp, _i64, _vp, _vp, _i64, _vp, _vp, _i32, _i32, _i64, _i32, _vp, _vp, _vp, _vp, _vp,
      _st]),
    ("ilans_quantize", ctypes.c_int, [_vp, _i32, _i32, _vp, _st]),
    ("ilans_histogram_u8", ctypes.c_int, [_vp, _i64, _vp, _vp, _st]),
    ("ilans_table_bytes", ctypes.c_size_t, []),
    ("ilans_dstatus_bytes", ctypes.c_size_t, []),
    ("ilans_counts_zero_dev", ctypes.c_int, [_vp, _vp]),
    ("ilans_histogram_u8_dev", ctypes.c_int, [_vp, _i64, _vp, _vp]),
    ("ilans_table_from_counts_dev", ctypes.c_int, [_vp, _i32, _vp, _vp]),
    ("ilans_table_from_freq_dev", ctypes.c_int, [_vp, _i32, _i32, _vp, _vp]),
    ("ilans_table_read_host", ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _st]),
    ("ilans_dstatus_reset_dev", ctypes.c_int, [_vp, _vp]),
    ("ilans_dstatus_read_host", ctypes.c_int, [_vp, _vp, _st]),
    ("ilans_dstatus_parse", ctypes.c_int, [_vp, _st]),
    ("ilans_encode_chunks_dev", ctypes.c_int,
     [_vp, _i64, _i64, _i32, _vp, _i32, _vp, _vp, _vp, _vp, _vp]),
    ("ilans_encode_chunks_covered_dev", ctypes.c_int,
     [_vp, _i64, _i64, _i32, _vp, _i32, _vp, _vp, _vp, _vp, _vp]),
    ("ilans_frame_chunks_dev", ctypes.c_int, [_vp, _i64, _i64, _vp, _vp, _vp, _i32, _vp]),
    ("ilans_decode_chunks_dev", ctypes.c_int,
     [_vp, _vp, _vp, _i64, _i64, _i32, _vp, _i32, _vp, _vp, _vp, _vp, _vp]),
    ("ilans_decode_chunks_slots_dev", ctypes.c_int,
     [_vp, _vp, _vp, _i64, _i64, _i32, _vp, _i32, _vp, _vp, _vp, _vp, _vp]),
    ("ilans_decode_chunks_slots_adler32_dev", ctypes.c_int,
     [_vp, _vp, _vp, _i64, _i64, _i32, _vp, _i32, _vp, _vp, _vp, _vp]),
    ("ilans_decode_chunks_adler32_dev", ctypes.c_int,
     [_vp, _vp, _vp, _i64, _i64, _i32, _vp, _i32, _vp, _vp, _vp, _vp]),
    ("ilans_adler32_chunks_dev", ctypes.c_int, [_vp, _i64, _i64, _vp, _vp]),
    ("ilans_encode_chunks_u8_dev", ctypes.c_int,
     [_vp, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("ilans_frame_chunks_u8_dev", ctypes.c_int, [_vp, _i64, _i64, _vp, _vp, _vp, _vp]),
    ("ilans_decode_chunks_u8_dev", ctypes.c_int,
     [_vp, _vp, _vp, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _vp]),
    ("ilans_synth_bytes_dev", ctypes.c_int, [_vp, _i64, _u64, _i64, _vp, _vp]),
    ("ilans_mux_encode", ctypes.c_int,
     [_vp, _i32, _vp, _i64, _vp, _i64, _vp, _vp, _i64, _i64, _vp, _i64, _vp, _vp, _vp, _vp,
      _vp, _st]),
    ("ilans_mux_merge", ctypes.c_int,
     [_vp, _i32, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp,
      _st]),
    ("ilans_mux_demux", ctypes.c_int,
     [_vp, _i32, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _i64, _vp, _i64, _i64, _vp,
      _vp, _vp, _st]),
]

for _name, _res, _args in PROTOTYPES:
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = [p[0] for p in PROTOTYPES]

# per-thread contexts outliving the interpreter must not call into a
# CUDA runtime that is being torn down (see ilans_process_exiting)
atexit.register(lib.ilans_process_exiting)


def raise_for(rc: int, st: Status, what: str = "") -> None:
    """Map an ilans_rc to the reference's exception types (errors.py:4-33)."""
    if rc == OK:
        return
    msg = st.message.decode(errors="replace") or what
    if rc == ERR_TRUNCATED:
        raise TruncatedStreamError(msg)
    if rc == ERR_UNENCODABLE:
        raise UnencodableSymbolError(msg)
    if rc == ERR_UNSUPPORTED:
        raise UnsupportedVariantError(msg)
    if rc == ERR_FORMAT:
        raise FormatError(msg)
    if rc == ERR_SCHEDULE:
        raise ScheduleError(msg)
    if rc == ERR_VALUE:
        raise ValueError(msg)
    raise RuntimeError(f"ilans-b200 CUDA failure in {what}: {msg}")


def check_dev(rc: int, what: str) -> None:
    """Device-pointer entry points return a bare rc (no status struct)."""
    if rc == OK:
        return
    if rc == ERR_VALUE:
        raise ValueError(f"{what}: invalid arguments")
    raise RuntimeError(f"{what}: CUDA launch failed (rc={rc})")


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def device_count() -> int:
    return int(lib.ilans_device_count())


def launch_count() -> int:
    return int(lib.ilans_launch_count())
