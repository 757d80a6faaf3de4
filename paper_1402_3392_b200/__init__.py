"""ilans-b200: B200-native interleaved rANS (Giesen, arXiv:1402.3392).

Drop-in for the reference ``ilans`` word16 hot path: same public names
(SymbolTable, quantize, encode_interleaved, decode_interleaved,
decode_lanes_full, Container, backend.Backend) with every encode, decode,
histogram and quantize executed by hand-written sm_100a kernels in
libilans_b200.so. Chunked, HBM-resident and multi-GPU entry points live in
``chunked`` and ``dist``.
"""

from . import backend, interleave, lanes, mux, rans
from .errors import (
    CodecError,
    FormatError,
    NotBUniqueError,
    ScheduleError,
    TrailingGarbageWarning,
    TruncatedStreamError,
    UnencodableSymbolError,
    UnsupportedVariantError,
)
from .interleave import Container, decode_interleaved, encode_interleaved
from .lanes import decode_lanes_full, encode_lanes_full
from .rans import BYTE8, WORD16, RenormVariant, SymbolTable, quantize

__version__ = "0.1.0"
