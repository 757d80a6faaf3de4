"""Generate the golden parity fixtures from the UNMODIFIED reference.

Run in the dev container (the only place /root/reference exists):

    bash oracle/build_ref.sh          # reference + its compiled _core -> oracle/_ref
    python tests/golden/make_golden.py

Every array in tests/golden/*.npz is produced by the reference package
itself (ilans.encode_interleaved / decode_interleaved / quantize /
SymbolTable, backend "ext" when built, otherwise "pure" -- the two are
byte-identical per pkg/tests/test_backend.py:75-128). The tests use them to
pin the oracle (oracle/rans_oracle.c) and to check the CUDA path.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
OUT = Path(__file__).resolve().parent

sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
if not (ROOT / "oracle" / "_ref" / "ilans").exists():
    sys.path.insert(0, "/root/reference/pkg/src")
import ilans  # noqa: E402
from ilans import backend  # noqa: E402
from ilans.interleave import encode_interleaved, decode_interleaved  # noqa: E402
from ilans.rans import WORD16, SymbolTable, quantize  # noqa: E402


def random_table(rng, max_n=256, min_sb=None, max_sb=16):
    # same generator shape as pkg/tests/test_interleave.py:45-50
    n = int(rng.integers(1, max_n + 1))
    lo = max(1, (n - 1).bit_length()) if min_sb is None else max(min_sb, (n - 1).bit_length(), 1)
    sb = int(rng.integers(lo, max_sb + 1))
    counts = rng.integers(0, 1000, size=n)
    counts[int(rng.integers(0, n))] += 1
    return counts, SymbolTable.from_counts(counts.tolist(), sb)


def random_message(rng, table, n):
    probs = table.freq_u32 / table.total
    return rng.choice(table.alphabet_size, size=n, p=probs).astype(np.uint8)


def codec_cases():
    rng = np.random.default_rng(1402_3392)
    arrays, meta = {}, []
    lane_set = [1, 2, 3, 4, 5, 8, 16, 17, 31, 32, 33, 64, 100, 1000]
    k = 0
    for lanes in lane_set:
        for n in sorted({0, 1, max(0, lanes - 1), lanes, lanes + 1, 2 * lanes + 1, 97,
                         int(rng.integers(2, 5000)), int(rng.integers(5000, 30000))}):
            counts, table = random_table(rng)
            msg = random_message(rng, table, n)
            c = encode_interleaved(msg, table, lanes, WORD16)
            blob = c.to_bytes()
            out = decode_interleaved(c)
            assert np.array_equal(out, msg)
            arrays[f"c{k}_msg"] = msg
            arrays[f"c{k}_freq"] = table.freq_u32
            arrays[f"c{k}_payload"] = np.asarray(c.payload, dtype=np.uint16)
            arrays[f"c{k}_states"] = np.asarray(c.final_states, dtype=np.uint32)
            meta.append(dict(case=k, lanes=lanes, n=n, scale_bits=table.scale_bits,
                             alphabet=table.alphabet_size,
                             sha256=hashlib.sha256(blob).hexdigest(), nbytes=len(blob)))
            k += 1
    # scale-bits sweep incl. the extremes 1 and 16, single-symbol alphabets
    for sb in range(1, 17):
        for n_sym in (1, 2, min(256, 1 << sb)):
            counts = rng.integers(1, 50, size=n_sym)
            table = SymbolTable.from_counts(counts.tolist(), sb)
            msg = random_message(rng, table, 3000)
            c = encode_interleaved(msg, table, 32, WORD16)
            arrays[f"c{k}_msg"] = msg
            arrays[f"c{k}_freq"] = table.freq_u32
            arrays[f"c{k}_payload"] = np.asarray(c.payload, dtype=np.uint16)
            arrays[f"c{k}_states"] = np.asarray(c.final_states, dtype=np.uint32)
            try:
                blob = c.to_bytes()
            except ilans.FormatError:  # f = 65536 has no u16 wire field (rans.py:334-335)
                blob = None
            meta.append(dict(case=k, lanes=32, n=3000, scale_bits=sb, alphabet=n_sym,
                             sha256=None if blob is None else hashlib.sha256(blob).hexdigest(),
                             nbytes=None if blob is None else len(blob)))
            k += 1
    return arrays, meta


def quantize_cases():
    rng = np.random.default_rng(7)
    arrays, meta = {}, []
    k = 0

    def add(counts, sb):
        nonlocal k
        counts = [int(c) for c in counts]
        freqs = quantize(counts, sb)
        arrays[f"q{k}_counts"] = np.asarray(counts, dtype=np.uint64)
        arrays[f"q{k}_freq"] = np.asarray(freqs, dtype=np.uint32)
        meta.append(dict(case=k, scale_bits=sb, n=len(counts)))
        k += 1

    # the reference suite's knowns (pkg/tests/test_rans.py:49-74)
    add([1, 3], 2)
    add([1, 1, 1, 1], 2)
    add([9, 9, 9, 9], 2)
    add([10**6, 1], 14)
    for _ in range(300):
        n = int(rng.integers(1, 257))
        sb = int(rng.integers(max(1, (n - 1).bit_length()), 17))
        counts = rng.integers(0, 1000, size=n)
        counts[int(rng.integers(0, n))] += 1
        add(counts, sb)
    # skewed, many forced-to-one symbols (the diff < 0 loop, several rounds)
    for sb in (8, 9, 10, 11, 12, 14, 16):
        for _ in range(10):
            n = 256 if sb >= 8 else 1 << sb
            counts = np.ones(n, dtype=np.int64)
            counts[int(rng.integers(0, n))] = int(rng.integers(10**5, 10**9))
            add(counts, sb)
    # Zipf-shaped, huge totals (> 2^32, as the 8 GiB config produces)
    for s in (0.3, 1.05, 1.1, 1.5, 2.15, 2.97):
        p = (np.arange(256) + 1.0) ** -s
        p /= p.sum()
        for total in (2**20, 2**28, 2**33, 2**40, 2**52):
            counts = np.floor(p * total).astype(np.uint64)
            counts[0] += 1
            for sb in (11, 12, 13, 14, 15, 16):
                add(counts, sb)
    return arrays, meta


def chunk_cases():
    """Chunk framing parity: chunk k must equal reference
    encode_interleaved(msg[kC:(k+1)C], table, 32, WORD16)."""
    rng = np.random.default_rng(99)
    arrays, meta = {}, []
    p = (np.arange(256) + 1.0) ** -1.1
    p /= p.sum()
    k = 0
    for n, chunk, sb in ((300_001, 65536, 12), (100_000, 16384, 14), (65536 * 2, 65536, 15),
                         (5000, 1024, 11)):
        msg = rng.choice(256, n, p=p).astype(np.uint8)
        counts = np.bincount(msg, minlength=int(msg.max()) + 1)
        table = SymbolTable.from_counts(counts.tolist(), sb)
        payloads, states = [], []
        for off in range(0, n, chunk):
            c = encode_interleaved(msg[off:off + chunk], table, 32, WORD16)
            payloads.append(np.asarray(c.payload, dtype=np.uint16))
            states.append(np.asarray(c.final_states, dtype=np.uint32))
        offs = np.zeros(len(payloads) + 1, dtype=np.uint64)
        offs[1:] = np.cumsum([len(x) for x in payloads])
        arrays[f"k{k}_msg"] = msg
        arrays[f"k{k}_freq"] = table.freq_u32
        arrays[f"k{k}_payload"] = np.concatenate(payloads)
        arrays[f"k{k}_offsets"] = offs
        arrays[f"k{k}_states"] = np.stack(states)
        meta.append(dict(case=k, n=n, chunk=chunk, scale_bits=sb, lanes=32))
        k += 1
    return arrays, meta


def byte8_cases():
    """BYTE8 (8-bit digits, L = 2^23): the reference's scalar path."""
    from ilans.rans import BYTE8

    rng = np.random.default_rng(8)
    arrays, meta = {}, []
    k = 0
    for lanes in (1, 2, 3, 5, 8, 17, 32, 33, 100):
        for n in sorted({0, 1, max(0, lanes - 1), lanes + 1, 2 * lanes + 3, 701,
                         int(rng.integers(1000, 4000))}):
            counts, table = random_table(rng)
            msg = random_message(rng, table, n)
            c = encode_interleaved(msg, table, lanes, BYTE8)
            assert np.array_equal(decode_interleaved(c), msg)
            arrays[f"b{k}_msg"] = msg
            arrays[f"b{k}_freq"] = table.freq_u32
            arrays[f"b{k}_payload"] = np.asarray(c.payload, dtype=np.uint8)
            arrays[f"b{k}_states"] = np.asarray(c.final_states, dtype=np.uint32)
            try:
                blob = c.to_bytes()
            except ilans.FormatError:
                blob = None
            meta.append(dict(case=k, lanes=lanes, n=n, scale_bits=table.scale_bits,
                             sha256=None if blob is None else hashlib.sha256(blob).hexdigest()))
            k += 1
    return arrays, meta


def main():
    print("reference backend:", backend.ACTIVE.name, "ilans", ilans.__version__)
    info = {"generator": "tests/golden/make_golden.py", "reference_backend": backend.ACTIVE.name,
            "numpy": np.__version__}
    for name, fn in (("codec", codec_cases), ("quantize", quantize_cases), ("chunks", chunk_cases),
                     ("byte8", byte8_cases)):
        arrays, meta = fn()
        np.savez_compressed(OUT / f"{name}.npz", **arrays)
        info[name] = meta
        print(name, len(meta), "cases")
    (OUT / "golden.json").write_text(json.dumps(info, indent=1))


if __name__ == "__main__":
    main()
