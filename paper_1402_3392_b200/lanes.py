"""Lane-parallel (warp) decode and encode entry points.

API-compatible with the kernel-backed parts of pkg/src/ilans/lanes.py:
decode_lanes_full (lanes.py:196-218) and encode_lanes_full (lanes.py:235-252).
On the B200 the lane model is not a simulation: a warp of 32 threads IS the
lane group, __ballot_sync is lanes.ballot, __popc(mask & lanemask_lt) is
lanes.lane_offset and the coalesced shared-ring read is lanes.packed_load
(csrc/decode.cu).
"""

from __future__ import annotations

import warnings

import numpy as np

from . import backend as backend_mod
from .errors import TrailingGarbageWarning, UnsupportedVariantError
from .interleave import Container, _as_symbols, _steps, encode_interleaved
from .rans import WORD16, SymbolTable

MAX_LANES = 32

__all__ = ["MAX_LANES", "decode_lanes_full", "decode_lanes_steps", "encode_lanes_full"]


def _check_lane_decodable(container: Container) -> None:
    if container.variant != WORD16:
        raise UnsupportedVariantError(
            f"variant {container.variant.tag!r} unsupported by lane decoder"
        )
    if container.lane_count > MAX_LANES:
        raise UnsupportedVariantError(
            f"lane decoder supports at most {MAX_LANES} lanes, "
            f"container has {container.lane_count}"
        )


def decode_lanes_full(container: Container, *, backend=None) -> np.ndarray:
    """Group-at-a-time decode; byte-identical to decode_interleaved."""
    _check_lane_decodable(container)
    table = container.table
    kern = backend_mod.get(backend)
    msg, consumed = kern.decode_lanes_u16(
        container.payload,
        np.asarray(container.final_states, dtype=np.uint32),
        table.slot_u8,
        table.freq_u32,
        table.cum_u32,
        table.scale_bits,
        container.message_length,
        container.lane_count,
    )
    if consumed != len(container.payload):
        warnings.warn(
            f"{len(container.payload) - consumed} unread digits after decode",
            TrailingGarbageWarning,
            stacklevel=2,
        )
    return msg


def decode_lanes_steps(container: Container):
    """Instrumented lane decode: yields (symbols, states, digits_read) after
    every group, in the shape of interleave.decode_interleaved_steps
    (reference lanes.py:221-232); a device trace of the warp decoder."""
    _check_lane_decodable(container)
    yield from _steps(container)


def encode_lanes_full(message, table: SymbolTable, lane_count: int) -> Container:
    """Group-form encode (tail group first, then full groups backwards);
    bit-identical to encode_interleaved. At most 32 lanes."""
    if not 1 <= lane_count <= MAX_LANES:
        raise ValueError(f"lane count must be in [1, {MAX_LANES}]")
    WORD16.check_table(table)
    _as_symbols(message, table)
    return encode_interleaved(message, table, lane_count, WORD16)
