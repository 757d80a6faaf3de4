"""Golden fixtures for the stream multiplexer, from the UNMODIFIED reference.

Run in the dev container (the only place /root/reference exists):

    python tests/golden/make_mux_golden.py

Writes tests/golden/mux.npz + mux.json. Every case runs the reference's own
``ilans.mux`` (pure Python, pkg/src/ilans/mux.py) on seeded messages:
per-stream buffers from encode_multistream, the merged payload from mux, and
the serialized container + MuxBudget of mux_with_flush for several flush
intervals and schedules. The B200 tests rebuild the same coders from the
JSON descriptions and must reproduce every byte.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
if not (ROOT / "oracle" / "_ref" / "ilans").exists():
    sys.path.insert(0, "/root/reference/pkg/src")
from ilans import mux as rmux  # noqa: E402
from ilans.rans import BYTE8, WORD16, RenormVariant, SymbolTable  # noqa: E402


def coder_from(desc):
    if desc["kind"] == "raw":
        return rmux.RawStreamCodec(desc["width"])
    t = SymbolTable(desc["freq"], desc["sb"])
    v = RenormVariant(desc["tag"], desc["digit_bits"], desc["L"])
    return rmux.RansStreamCodec(t, v)


def random_rans(rng, variant, max_n=256, max_sb=None):
    n = int(rng.integers(2, max_n + 1))
    top = max_sb or min(16, variant.lower_bound.bit_length() - 1)
    lo = max(1, (n - 1).bit_length())
    sb = int(rng.integers(lo, max(lo, top) + 1))
    while variant.lower_bound % (1 << sb):
        sb -= 1
    counts = rng.integers(0, 500, size=n) ** int(rng.integers(1, 3))
    counts[int(rng.integers(0, n))] += 1
    t = SymbolTable.from_counts(counts.tolist(), sb)
    return {"kind": "rans", "freq": t.freq, "sb": sb, "tag": variant.tag,
            "digit_bits": variant.digit_bits, "L": variant.lower_bound}


def message_for(rng, desc, n):
    if desc["kind"] == "raw":
        return rng.integers(0, 1 << desc["width"], size=n, dtype=np.uint64).tolist()
    f = np.asarray(desc["freq"], dtype=np.float64)
    return rng.choice(len(f), size=n, p=f / f.sum()).tolist()


def main():
    rng = np.random.default_rng(14023392)
    custom = RenormVariant("custom8", 8, 1 << 16)       # byte digits, L = 2^16
    arrays, cases = {}, []
    shapes = [
        # (stream kinds, lengths, flush intervals, schedule kind)
        (["w16", "w16", "raw12"], [400, 700, 250], [None, 16, 1000], "shuffle"),
        (["w16", "w16", "raw12"], [300, 200, 100], [None, 7], "round_robin"),
        (["b8", "raw5"], [300, 120], [None, 1, 33], "shuffle"),
        (["w16"], [1000], [None, 64], "single"),
        (["w16", "raw8"], [64, 0], [None], "round_robin"),
        (["w16", "w16"], [1, 3000], [None, 256], "lopsided"),
        (["custom8", "w16", "raw32", "b8", "raw1"], [500, 300, 200, 400, 90], [None, 5, 97],
         "shuffle"),
        (["w16"] * 12 + ["raw16"] * 4, [int(x) for x in rng.integers(0, 200, size=16)],
         [None, 3, 50], "shuffle"),
        ([], [], [None], "round_robin"),
        (["w16", "b8"], [0, 0], [None, 4], "round_robin"),
    ]
    k = 0
    for kinds, lengths, flushes, skind in shapes:
        descs = []
        for kind in kinds:
            if kind == "w16":
                descs.append(random_rans(rng, WORD16))
            elif kind == "b8":
                descs.append(random_rans(rng, BYTE8, max_sb=16))
            elif kind == "custom8":
                descs.append(random_rans(rng, custom))
            else:
                descs.append({"kind": "raw", "width": int(kind[3:])})
        msgs = [message_for(rng, d, n) for d, n in zip(descs, lengths)]
        coders = [coder_from(d) for d in descs]
        if skind == "shuffle":
            sched = [j for j, n in enumerate(lengths) for _ in range(n)]
            rng.shuffle(sched)
        elif skind == "single":
            sched = [0] * lengths[0]
        elif skind == "lopsided":
            sched = [0] + [1] * lengths[1]
        else:
            sched = rmux.round_robin_schedule(lengths)
        sched = [int(s) for s in sched]
        bufs = rmux.encode_multistream(msgs, coders)
        merged = rmux.mux(bufs, coders, sched)
        runs = []
        for fl in flushes:
            cont, budget = rmux.mux_with_flush(msgs, coders, sched, fl)
            blob = cont.to_bytes()
            assert rmux.demux_decode(blob, coders, sched) == [list(m) for m in msgs]
            arrays[f"m{k}_f{len(runs)}_blob"] = np.frombuffer(blob, dtype=np.uint8)
            runs.append({"flush": fl, "max_buffered": budget.max_buffered,
                         "segment_count": budget.segment_count,
                         "payload_bytes": budget.payload_bytes})
        for j, m in enumerate(msgs):
            arrays[f"m{k}_msg{j}"] = np.asarray(m, dtype=np.uint64)
            arrays[f"m{k}_hdr{j}"] = np.frombuffer(bufs[j].header, dtype=np.uint8)
            arrays[f"m{k}_pay{j}"] = np.frombuffer(bufs[j].payload, dtype=np.uint8)
        arrays[f"m{k}_sched"] = np.asarray(sched, dtype=np.int32)
        arrays[f"m{k}_merged"] = np.frombuffer(merged, dtype=np.uint8)
        cases.append({"case": k, "streams": descs, "lengths": lengths, "runs": runs,
                      "schedule": skind})
        k += 1
    np.savez_compressed(OUT / "mux.npz", **arrays)
    (OUT / "mux.json").write_text(json.dumps({"generator": "tests/golden/make_mux_golden.py",
                                              "reference": "pkg/src/ilans/mux.py",
                                              "cases": cases}, indent=1) + "\n")
    print(f"{k} mux cases, {sum(a.nbytes for a in arrays.values())} bytes")


if __name__ == "__main__":
    main()
