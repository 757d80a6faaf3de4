"""Multiplexer throughput: B200 mux_with_flush / mux / demux_decode vs the
reference's pure-Python mux.py, same workload (run on the GPU box):

    python tools/mux_probe.py [streams] [symbols_per_stream] [flush]

Workload: `streams` streams, 3 of 4 word16 rANS over a Zipf(1.1) table
(sb = 12), every 4th raw 12-bit values; round-robin schedule; messages as
numpy arrays. The reference is timed on 1/16 of the symbols (it is pure
Python) and reported per symbol."""

import sys
import time

import numpy as np

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/oracle/_ref")
from paper_1402_3392_b200 import mux as bm  # noqa: E402
from paper_1402_3392_b200.rans import SymbolTable  # noqa: E402
from paper_1402_3392_b200.synth import synth_host  # noqa: E402
import ilans.mux as rm  # noqa: E402
from ilans.rans import SymbolTable as RTable  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 16
N = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
F = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
F = F or None  # 0: no flushing

src = synth_host(K * N, 1.1, seed=7)
counts = np.bincount(src, minlength=256)
freq = SymbolTable.from_counts(counts.tolist(), 12).freq
rng = np.random.default_rng(3)


def build(mod, table_cls, n):
    t = table_cls(freq, 12)
    coders, msgs = [], []
    for j in range(K):
        if j % 4 == 3:
            coders.append(mod.RawStreamCodec(12))
            msgs.append(rng.integers(0, 1 << 12, size=n))
        else:
            coders.append(mod.RansStreamCodec(t))
            msgs.append(src[j * N: j * N + n].astype(np.int64))
    return coders, msgs


def tm(f, reps=3):
    f()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        best = min(best, time.perf_counter() - t0)
    return best


coders, msgs = build(bm, SymbolTable, N)
sched = bm.round_robin_schedule([N] * K)
cont, budget = bm.mux_with_flush(msgs, coders, sched, F)
blob = cont.to_bytes()
assert [list(m) for m in msgs] == bm.demux_decode(blob, coders, sched)
bufs = bm.encode_multistream(msgs, coders)
T = K * N
e = tm(lambda: bm.mux_with_flush(msgs, coders, sched, F))
d = tm(lambda: bm.demux_decode(blob, coders, sched))
m = tm(lambda: bm.mux(bufs, coders, sched))
print(f"B200: {K} streams x {N} symbols, flush {F}: payload {len(cont.payload)} B, "
      f"{budget.segment_count} segments, max_buffered {budget.max_buffered}")
print(f"B200 mux_with_flush {T / e / 1e6:.2f} Msym/s ({e * 1e3:.1f} ms), "
      f"mux {T / m / 1e6:.2f} Msym/s, demux_decode {T / d / 1e6:.2f} Msym/s ({d * 1e3:.1f} ms)")

n_ref = max(1, N // 16)
rcoders, rmsgs = build(rm, RTable, n_ref)
rsched = rm.round_robin_schedule([n_ref] * K)
rcont, _ = rm.mux_with_flush([m.tolist() for m in rmsgs], rcoders, rsched, F)
rblob = rcont.to_bytes()
rl = [m.tolist() for m in rmsgs]
re_ = tm(lambda: rm.mux_with_flush(rl, rcoders, rsched, F), 1)
rd = tm(lambda: rm.demux_decode(rblob, rcoders, rsched), 1)
rbufs = rm.encode_multistream(rl, rcoders)
rmm = tm(lambda: rm.mux(rbufs, rcoders, rsched), 1)
Tr = K * n_ref
print(f"reference (pure Python, {Tr} symbols): mux_with_flush {Tr / re_ / 1e6:.3f} Msym/s, "
      f"mux {Tr / rmm / 1e6:.3f} Msym/s, demux_decode {Tr / rd / 1e6:.3f} Msym/s")
