"""Stream multiplexer on the B200 (paper_1402_3392_b200.mux -> csrc/mux.cu).

Parity: every byte the reference's mux.py produced for the fixtures in
tests/golden/mux.npz (tests/golden/make_mux_golden.py) -- per-stream
buffers, merged payloads, serialized flushed containers, budgets -- and the
reference's own behavioural tests (pkg/tests/test_mux.py) restated against
this API."""

import json
import warnings
from pathlib import Path

import numpy as np
import pytest

from paper_1402_3392_b200 import _lib
from paper_1402_3392_b200.errors import (
    FormatError,
    ScheduleError,
    TrailingGarbageWarning,
    TruncatedStreamError,
    UnencodableSymbolError,
)
from paper_1402_3392_b200.mux import (
    MuxedContainer,
    RansStreamCodec,
    RawStreamCodec,
    StreamBuffer,
    demux_decode,
    encode_multistream,
    mux,
    mux_with_flush,
    round_robin_schedule,
)
from paper_1402_3392_b200.rans import BYTE8, WORD16, RenormVariant, SymbolTable

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if _lib.device_count() == 0:
        pytest.fail("no CUDA device: the -m gpu suite must run on a B200")


def coder_from(desc):
    if desc["kind"] == "raw":
        return RawStreamCodec(desc["width"])
    t = SymbolTable(desc["freq"], desc["sb"])
    return RansStreamCodec(t, RenormVariant(desc["tag"], desc["digit_bits"], desc["L"]))


def golden_cases():
    meta = json.loads((GOLDEN / "mux.json").read_text())
    arrays = np.load(GOLDEN / "mux.npz")
    for case in meta["cases"]:
        k = case["case"]
        coders = [coder_from(d) for d in case["streams"]]
        msgs = [arrays[f"m{k}_msg{j}"].astype(np.int64).tolist() for j in range(len(coders))]
        yield case, arrays, coders, msgs, arrays[f"m{k}_sched"].tolist()


# ---------------------------------------------------------------- golden ---
def test_encode_multistream_matches_reference_buffers():
    for case, arrays, coders, msgs, _ in golden_cases():
        k = case["case"]
        bufs = encode_multistream(msgs, coders)
        for j, b in enumerate(bufs):
            assert b.header == arrays[f"m{k}_hdr{j}"].tobytes(), (k, j)
            assert b.payload == arrays[f"m{k}_pay{j}"].tobytes(), (k, j)
            assert b.symbol_count == len(msgs[j])


def test_mux_matches_reference_merge():
    for case, arrays, coders, msgs, sched in golden_cases():
        k = case["case"]
        bufs = [StreamBuffer(arrays[f"m{k}_hdr{j}"].tobytes(), arrays[f"m{k}_pay{j}"].tobytes(),
                             len(msgs[j])) for j in range(len(coders))]
        assert mux(bufs, coders, sched) == arrays[f"m{k}_merged"].tobytes(), k


def test_mux_with_flush_matches_reference_containers():
    for case, arrays, coders, msgs, sched in golden_cases():
        k = case["case"]
        for r, run in enumerate(case["runs"]):
            cont, budget = mux_with_flush(msgs, coders, sched, run["flush"])
            assert cont.to_bytes() == arrays[f"m{k}_f{r}_blob"].tobytes(), (k, run)
            assert budget.max_buffered == run["max_buffered"], (k, run)
            assert budget.segment_count == run["segment_count"], (k, run)
            assert budget.payload_bytes == run["payload_bytes"], (k, run)
            assert demux_decode(arrays[f"m{k}_f{r}_blob"].tobytes(), coders, sched) == msgs


# ------------------------------------------------- reference test_mux.py ---
def random_table(rng, max_n=64):
    n = int(rng.integers(2, max_n + 1))
    sb = int(rng.integers(max(1, (n - 1).bit_length()), 15))
    counts = rng.integers(0, 500, size=n)
    counts[int(rng.integers(0, n))] += 1
    return SymbolTable.from_counts(counts.tolist(), sb)


def random_message(rng, table, n):
    return rng.choice(table.alphabet_size, size=n, p=table.freq_u32 / table.total).tolist()


def shuffled(rng, lengths):
    s = [j for j, n in enumerate(lengths) for _ in range(n)]
    rng.shuffle(s)
    return s


def workload(rng, lengths=(400, 700, 250)):
    tables = [random_table(rng) for _ in range(2)]
    coders = [RansStreamCodec(tables[0]), RansStreamCodec(tables[1]), RawStreamCodec(12)]
    msgs = [random_message(rng, tables[0], lengths[0]), random_message(rng, tables[1], lengths[1]),
            rng.integers(0, 1 << 12, size=lengths[2]).tolist()]
    return msgs, coders


def test_length_identity_and_single_stream():
    rng = np.random.default_rng(40)
    msgs, coders = workload(rng)
    bufs = encode_multistream(msgs, coders)
    merged = mux(bufs, coders, round_robin_schedule([len(m) for m in msgs]))
    assert len(merged) == sum(len(b.payload) for b in bufs)
    t = random_table(rng)
    msg = random_message(rng, t, 1000)
    (buf,) = encode_multistream([msg], [RansStreamCodec(t)])
    assert mux([buf], [RansStreamCodec(t)], [0] * 1000) == buf.payload


def test_round_trips_custom_schedules_and_serialization():
    rng = np.random.default_rng(44)
    msgs, coders = workload(rng)
    sched = shuffled(rng, [len(m) for m in msgs])
    for flush in (None, 1, 16, 1 << 20):
        cont, _ = mux_with_flush(msgs, coders, sched, flush)
        assert demux_decode(cont, coders, sched) == msgs
        blob = cont.to_bytes()
        assert demux_decode(blob, coders, sched) == msgs
        parsed = MuxedContainer.from_bytes(blob)
        assert parsed.flush_interval == flush and parsed.payload == cont.payload


def test_byte8_and_custom_variants_in_the_mix():
    rng = np.random.default_rng(45)
    t = random_table(rng)
    custom = RenormVariant("c8", 8, 1 << 16)
    coders = [RansStreamCodec(t, BYTE8), RawStreamCodec(5), RansStreamCodec(t, custom),
              RawStreamCodec(32)]
    msgs = [random_message(rng, t, 300), rng.integers(0, 32, size=120).tolist(),
            random_message(rng, t, 200),
            rng.integers(0, 1 << 32, size=50, dtype=np.uint64).astype(np.int64).tolist()]
    sched = shuffled(rng, [len(m) for m in msgs])
    for flush in (None, 3):
        cont, _ = mux_with_flush(msgs, coders, sched, flush)
        assert demux_decode(cont, coders, sched) == msgs


def test_wrong_schedule_never_silently_matches():
    rng = np.random.default_rng(47)
    msgs, coders = workload(rng, (50, 50, 50))
    sched = shuffled(rng, [50, 50, 50])
    cont, _ = mux_with_flush(msgs, coders, sched)
    other = shuffled(np.random.default_rng(999), [50, 50, 50])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        try:
            out = demux_decode(cont, coders, other)
        except (TruncatedStreamError, FormatError):
            return
    assert out != msgs


def test_schedule_validation():
    rng = np.random.default_rng(48)
    msgs, coders = workload(rng, (10, 10, 10))
    with pytest.raises(ScheduleError, match="stream 1"):
        mux_with_flush(msgs, coders, [0] * 10 + [1] * 9 + [2] * 11)
    msgs, coders = workload(rng, (5, 5, 5))
    with pytest.raises(ScheduleError, match="unknown stream"):
        mux_with_flush(msgs, coders, [0, 1, 2, 7] + [0] * 4 + [1] * 4 + [2] * 4)
    t = random_table(rng)
    msg = random_message(rng, t, 40)
    (buf,) = encode_multistream([msg], [RansStreamCodec(t)])
    buf.payload += b"\x00\x00"
    with pytest.raises(ScheduleError, match="not fully consumed"):
        mux([buf], [RansStreamCodec(t)], [0] * 40)
    with pytest.raises(ValueError):
        mux_with_flush(msgs[:1], coders[:1], flush_interval=0)


def test_merge_errors_follow_reference_order():
    rng = np.random.default_rng(60)
    t = random_table(rng)
    msg = random_message(rng, t, 300)
    c = RansStreamCodec(t)
    (buf,) = encode_multistream([msg], [c])
    short = StreamBuffer(buf.header, buf.payload[: len(buf.payload) // 2], 300)
    with pytest.raises(TruncatedStreamError):
        mux([short], [c], [0] * 300)
    with pytest.raises(TruncatedStreamError):
        mux([StreamBuffer(b"\x01", buf.payload, 300)], [c], [0] * 300)
    with pytest.raises(FormatError, match="interval"):
        mux([StreamBuffer(b"\0\0\0\0", buf.payload, 300)], [c], [0] * 300)


def test_flush_bounds_buffering_and_costs_per_segment():
    rng = np.random.default_rng(53)
    t = SymbolTable.from_counts([1] * 256, 14)
    coders = [RansStreamCodec(t), RansStreamCodec(t)]
    msgs = [random_message(rng, t, 1), random_message(rng, t, 10_000)]
    sched = [0] + [1] * 10_000
    base, unbounded = mux_with_flush(msgs, coders, sched)
    flushed, bounded = mux_with_flush(msgs, coders, sched, flush_interval=256)
    assert bounded.max_buffered < unbounded.max_buffered / 10
    assert demux_decode(flushed, coders, sched) == msgs
    budgets = [mux_with_flush(msgs, coders, sched, flush_interval=f)[1] for f in (64, 256, 1024)]
    assert budgets[0].max_buffered <= budgets[1].max_buffered <= budgets[2].max_buffered
    extra = bounded.segment_count - unbounded.segment_count
    assert extra > 0 and len(flushed.payload) - len(base.payload) <= extra * 8
    assert unbounded.max_buffered == len(base.payload)


def test_codec_validation_and_errors():
    with pytest.raises(ValueError):
        RawStreamCodec(0)
    with pytest.raises(ValueError):
        RawStreamCodec(33)
    with pytest.raises(ValueError):
        RawStreamCodec(4).encode_segment([16])
    with pytest.raises(ValueError, match="byte-multiple"):
        RansStreamCodec(SymbolTable([1, 3], 2), RenormVariant("odd", 12, 1 << 20))
    with pytest.raises(UnencodableSymbolError, match="symbol 1 has frequency 0"):
        RansStreamCodec(SymbolTable([4, 0], 2)).encode_segment([0, 1, 0])
    with pytest.raises(TypeError):
        encode_multistream([[1]], [object()])


def test_corrupt_header_and_truncated_payload():
    rng = np.random.default_rng(57)
    t = random_table(rng)
    coders = [RansStreamCodec(t)]
    cont, _ = mux_with_flush([random_message(rng, t, 30)], coders)
    cont.stream_headers[0] = b"\x00\x00\x00\x00"
    with pytest.raises(FormatError, match="interval"):
        demux_decode(cont, coders)
    cont, _ = mux_with_flush([random_message(rng, t, 500)], coders)
    cont.payload = cont.payload[: len(cont.payload) // 2]
    with pytest.raises(TruncatedStreamError):
        demux_decode(cont, coders)
    cont, _ = mux_with_flush([random_message(rng, t, 500)], coders)
    cont.payload += b"zz"
    with pytest.warns(TrailingGarbageWarning):
        demux_decode(cont, coders)


def test_larger_mux_round_trip():
    """A larger workload than the reference's tests (64 streams, 200 K
    symbols, flushed every 1000 steps): device encode + merge + demux."""
    rng = np.random.default_rng(61)
    tables = [random_table(rng, 256) for _ in range(8)]
    coders = [RansStreamCodec(tables[j % 8], BYTE8 if j % 3 == 0 else WORD16)
              if j % 5 else RawStreamCodec(int(rng.integers(1, 33))) for j in range(64)]
    lengths = rng.integers(0, 6000, size=64).tolist()
    msgs = []
    for c, n in zip(coders, lengths):
        if isinstance(c, RawStreamCodec):
            msgs.append(rng.integers(0, 1 << c.width_bits, size=n, dtype=np.uint64)
                        .astype(np.int64).tolist())
        else:
            msgs.append(random_message(rng, c.table, n))
    sched = shuffled(rng, lengths)
    cont, budget = mux_with_flush(msgs, coders, sched, 1000)
    assert budget.payload_bytes == len(cont.payload)
    assert demux_decode(cont.to_bytes(), coders, sched) == msgs
    bufs = encode_multistream(msgs, coders)
    plain = mux(bufs, coders, sched)
    cont0, b0 = mux_with_flush(msgs, coders, sched)
    assert cont0.payload == plain and b0.max_buffered == len(plain)


def test_fuzz_against_reference_mux():
    """Randomized workloads against the unmodified reference mux.py (from
    oracle/_ref, the checker): containers, budgets, merged payloads and
    stream buffers byte for byte; demux round trips."""
    import os

    import oracle

    if oracle.reference_ilans() is None:
        pytest.skip("oracle/_ref not built (bash oracle/build_ref.sh)")
    from ilans import mux as rmux
    from ilans.rans import BYTE8 as RBYTE8
    from ilans.rans import WORD16 as RWORD16
    from ilans.rans import RenormVariant as RVariant
    from ilans.rans import SymbolTable as RTable

    rng = np.random.default_rng(int(os.environ.get("ILANS_FUZZ_SEED", "77")))
    variants = [(WORD16, RWORD16), (BYTE8, RBYTE8),
                (RenormVariant("c8", 8, 1 << 16), RVariant("c8", 8, 1 << 16)),
                (RenormVariant("c16", 16, 1 << 14), RVariant("c16", 16, 1 << 14))]
    for it in range(int(os.environ.get("ILANS_FUZZ_ITERS", "40"))):
        k = int(rng.integers(1, 9))
        ours, theirs, msgs = [], [], []
        for _ in range(k):
            n = int(rng.choice([0, 1, 2, 17, 100, 400]))
            if rng.random() < 0.3:
                w = int(rng.integers(1, 33))
                ours.append(RawStreamCodec(w))
                theirs.append(rmux.RawStreamCodec(w))
                msgs.append(rng.integers(0, 1 << w, size=n, dtype=np.uint64)
                            .astype(np.int64).tolist())
                continue
            v, rv = variants[int(rng.integers(0, len(variants)))]
            top = min(14, v.lower_bound.bit_length() - 1)
            n_sym = int(rng.integers(1, 65))
            sb = int(rng.integers(max(1, (n_sym - 1).bit_length()), top + 1))
            counts = rng.integers(0, 300, size=n_sym)
            counts[int(rng.integers(0, n_sym))] += 1
            t = SymbolTable.from_counts(counts.tolist(), sb)
            ours.append(RansStreamCodec(t, v))
            theirs.append(rmux.RansStreamCodec(RTable(t.freq, sb), rv))
            msgs.append(random_message(rng, t, n) if n else [])
        lengths = [len(m) for m in msgs]
        sched = shuffled(rng, lengths) if rng.random() < 0.6 else round_robin_schedule(lengths)
        flush = [None, 1, 2, 7, 50][int(rng.integers(0, 5))]
        c, b = mux_with_flush(msgs, ours, sched, flush)
        rc, rb = rmux.mux_with_flush(msgs, theirs, sched, flush)
        assert c.to_bytes() == rc.to_bytes(), (it, flush, lengths)
        assert (b.max_buffered, b.segment_count, b.payload_bytes) == \
            (rb.max_buffered, rb.segment_count, rb.payload_bytes), it
        assert demux_decode(c.to_bytes(), ours, sched) == msgs, it
        bufs = encode_multistream(msgs, ours)
        rbufs = rmux.encode_multistream(msgs, theirs)
        assert [(x.header, x.payload) for x in bufs] == [(x.header, x.payload) for x in rbufs]
        assert mux(bufs, ours, sched) == rmux.mux(rbufs, theirs, sched), it
