"""Per-call cost of the drop-in plugin path (one 64 KiB chunk, N = 32):
wall time of the raw C-ABI call (backend.*_u16) and of the reference-API
wrapper (interleave.encode_interleaved / decode_interleaved). Run under
ncu --metrics gpu__time_duration.sum for the kernel share."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1402_3392_b200 import backend  # noqa: E402
from paper_1402_3392_b200.interleave import decode_interleaved, encode_interleaved  # noqa: E402
from paper_1402_3392_b200.rans import SymbolTable  # noqa: E402
from paper_1402_3392_b200.synth import synth_host  # noqa: E402

C = 65536
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
msg = synth_host(C * 8, 1.1, 1234)
counts = np.bincount(msg, minlength=256)
t = SymbolTable.from_counts(counts[: int(np.nonzero(counts)[0][-1]) + 1].tolist(), 12)
chunk = msg[:C]
f, cum, slot = t.freq_u32, t.cum_u32, t.slot_u8
p, s = backend.encode_interleaved_u16(chunk, f, cum, 12, 32)
backend.decode_interleaved_u16(p, s, slot, f, cum, 12, C, 32)


def timeit(fn):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return 1e6 * (time.perf_counter() - t0) / reps


r = {
    "raw_encode_us": timeit(lambda: backend.encode_interleaved_u16(chunk, f, cum, 12, 32)),
    "raw_decode_us": timeit(lambda: backend.decode_interleaved_u16(p, s, slot, f, cum, 12, C, 32)),
}
c = encode_interleaved(chunk, t, 32)
r["api_encode_us"] = timeit(lambda: encode_interleaved(chunk, t, 32))
r["api_decode_us"] = timeit(lambda: decode_interleaved(c))
print(r)
