"""Parity of the B200 path against the oracle and the reference's golden
fixtures. Every call here goes through libilans_b200.so (C ABI) into the
sm_100a kernels; results must be bit-exact: identical tables, payloads,
final states, consumed counts and decoded bytes."""

import hashlib
import warnings

import numpy as np
import pytest

import oracle
import paper_1402_3392_b200 as ilb
from conftest import ZIPF_1MIB_DIGESTS, zipf_1mib
from paper_1402_3392_b200 import _lib, backend, rans
from paper_1402_3392_b200.errors import (
    FormatError,
    TrailingGarbageWarning,
    TruncatedStreamError,
    UnencodableSymbolError,
)
from paper_1402_3392_b200.interleave import Container
from paper_1402_3392_b200.rans import WORD16, SymbolTable

pytestmark = pytest.mark.gpu

B = backend.B200


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if _lib.device_count() == 0:
        pytest.fail("no CUDA device: the -m gpu suite must run on a B200")


def random_table(rng, max_n=256, max_sb=16):
    n = int(rng.integers(1, max_n + 1))
    sb = int(rng.integers(max(1, (n - 1).bit_length()), max_sb + 1))
    counts = rng.integers(0, 1000, size=n)
    counts[int(rng.integers(0, n))] += 1
    return SymbolTable(oracle.quantize(counts, sb), sb)


def random_message(rng, table, n):
    return rng.choice(table.alphabet_size, size=n, p=table.freq_u32 / table.total).astype(np.uint8)


# ---------------------------------------------------------------- golden ---
def test_kernels_match_reference_fixtures(golden_codec, golden_meta):
    for case in golden_meta["codec"]:
        k, lanes, sb = case["case"], case["lanes"], case["scale_bits"]
        msg = golden_codec[f"c{k}_msg"]
        t = SymbolTable(golden_codec[f"c{k}_freq"].tolist(), sb)
        payload, states = B.encode_interleaved_u16(msg, t.freq_u32, t.cum_u32, sb, lanes)
        assert np.array_equal(payload, golden_codec[f"c{k}_payload"]), case
        assert np.array_equal(states, golden_codec[f"c{k}_states"]), case
        out, consumed = B.decode_interleaved_u16(payload, states, t.slot_u8, t.freq_u32,
                                                 t.cum_u32, sb, len(msg), lanes)
        assert np.array_equal(out, msg) and consumed == len(payload), case
        if lanes <= 32:
            out2, consumed2 = B.decode_lanes_u16(payload, states, t.slot_u8, t.freq_u32,
                                                 t.cum_u32, sb, len(msg), lanes)
            assert np.array_equal(out2, msg) and consumed2 == len(payload), case
        if case["sha256"] is not None:
            c = Container(WORD16, lanes, len(msg), t, tuple(int(x) for x in states), payload)
            assert hashlib.sha256(c.to_bytes()).hexdigest() == case["sha256"]


def test_quantize_matches_reference_fixtures(golden_quantize, golden_meta):
    for case in golden_meta["quantize"]:
        k = case["case"]
        counts = golden_quantize[f"q{k}_counts"]
        want = golden_quantize[f"q{k}_freq"].tolist()
        assert rans.quantize(counts.tolist(), case["scale_bits"]) == want, case


def test_quantize_known_answers_and_errors():
    assert rans.quantize([1, 3], 2) == [1, 3]
    assert rans.quantize([9, 9, 9, 9], 2) == [1, 1, 1, 1]
    assert rans.quantize([10**6, 1], 14) == [16383, 1]
    assert rans.quantize([3, 0, 0], 4) == [16, 0, 0]
    for bad, match in ((([0, 0], 4), "positive"), (([1, 2], 0), "scale_bits"),
                       (([1] * 300, 12), "alphabet"), (([1] * 5, 2), "too large")):
        with pytest.raises(ValueError, match=match):
            rans.quantize(*bad)


def test_quantize_fuzz_vs_oracle():
    rng = np.random.default_rng(11)
    for _ in range(300):
        n = int(rng.integers(1, 257))
        sb = int(rng.integers(max(1, (n - 1).bit_length()), 17))
        kind = rng.integers(0, 3)
        if kind == 0:
            counts = rng.integers(0, 1000, size=n)
        elif kind == 1:  # forced-to-one heavy (several -1 rounds)
            counts = np.ones(n, dtype=np.int64)
            counts[int(rng.integers(0, n))] = int(rng.integers(1, 10**12))
        else:  # huge totals (> 2^32, u64 counts)
            counts = rng.integers(0, 2**40, size=n)
        counts[int(rng.integers(0, n))] += 1
        assert rans.quantize(counts.tolist(), sb) == oracle.quantize(counts, sb)


def test_baseline_md_digests_through_product_api():
    msg = zipf_1mib()
    counts, alpha = oracle.histogram(msg)
    for (lanes, sb), digest in ZIPF_1MIB_DIGESTS.items():
        t = SymbolTable.from_counts(counts[:alpha].tolist(), sb)
        c = ilb.encode_interleaved(msg, t, lanes, WORD16)
        assert hashlib.sha256(c.to_bytes()).hexdigest()[:16] == digest, (lanes, sb)
        assert np.array_equal(ilb.decode_interleaved(c), msg)
        if lanes <= 32:
            assert np.array_equal(ilb.decode_lanes_full(c), msg)


# ------------------------------------------------------------ histogram ---
def test_histogram_matches_bincount():
    from paper_1402_3392_b200 import chunked  # noqa: F401  (torch-free host path below)
    import ctypes

    rng = np.random.default_rng(5)
    cases = [np.zeros(0, np.uint8), np.array([7], np.uint8),
             rng.integers(0, 256, size=1_000_003).astype(np.uint8),
             np.full(3_000_001, 200, dtype=np.uint8),  # 1-symbol source
             (rng.random(2_000_000) < 0.8).astype(np.uint8) * 77]
    for msg in cases:
        for off in (0, 1, 5, 15):
            m = msg[off:] if len(msg) > off else msg
            counts = np.zeros(256, np.uint64)
            alpha = ctypes.c_int32(0)
            st = _lib.Status()
            rc = _lib.lib.ilans_histogram_u8(_lib.ptr(np.ascontiguousarray(m)), len(m),
                                             _lib.ptr(counts), ctypes.byref(alpha),
                                             ctypes.byref(st))
            _lib.raise_for(rc, st)
            ref, ref_alpha = oracle.histogram(m)
            assert np.array_equal(counts, ref) and alpha.value == ref_alpha


def test_histogram_device_pointers_and_flush():
    """ilans_histogram_u8_dev on offset device pointers (unaligned head and
    tail bytes around the bulk-copied body), and a 1-symbol source large
    enough that every CTA flushes its 16-bit counters mid-stream (> 1000
    ring slots per CTA)."""
    import ctypes

    import torch

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(11)
    host = rng.integers(0, 256, size=5_000_011).astype(np.uint8)
    d = torch.from_numpy(host).to(dev)
    counts = torch.zeros(256, dtype=torch.int64, device=dev)
    for off, n in ((0, len(host)), (1, 100_000), (7, 4_999_999), (13, 17), (3, 65_549)):
        counts.zero_()
        rc = _lib.lib.ilans_histogram_u8_dev(d.data_ptr() + off, n, counts.data_ptr(), None)
        assert rc == 0
        torch.cuda.synchronize()
        ref = np.bincount(host[off:off + n], minlength=256)
        assert np.array_equal(counts.cpu().numpy(), ref), (off, n)
    del d
    n = 148 * 17 * (1 << 20) + 12_345  # ~2.5 GB: > 1000 x 16 KB slots per CTA
    big = torch.full((n + 1,), 200, dtype=torch.uint8, device=dev)
    big[0] = 3
    counts.zero_()
    rc = _lib.lib.ilans_histogram_u8_dev(big.data_ptr() + 1, n, counts.data_ptr(), None)
    assert rc == 0
    torch.cuda.synchronize()
    c = counts.cpu().numpy()
    assert c[200] == n and c.sum() == n
    del big
    torch.cuda.empty_cache()


# ------------------------------------------------------- API behaviour ---
def test_round_trips_many_shapes():
    rng = np.random.default_rng(2026)
    for lanes in (1, 2, 3, 5, 8, 16, 17, 31, 32, 33, 64, 65, 100, 128, 129, 200, 256, 257,
                  1024, 1500):
        t = random_table(rng)
        for n in sorted({0, 1, lanes - 1, lanes, lanes + 1, 2 * lanes + 1, 513, 4097,
                         int(rng.integers(1000, 20000))}):
            msg = random_message(rng, t, n)
            c = ilb.encode_interleaved(msg, t, lanes, WORD16)
            ref_p, ref_s = oracle.encode_interleaved_u16(msg, t.freq_u32, t.cum_u32,
                                                         t.scale_bits, lanes)
            assert np.array_equal(c.payload, ref_p) and c.final_states == tuple(ref_s.tolist())
            assert np.array_equal(ilb.decode_interleaved(c), msg)
            if lanes <= 32:
                assert np.array_equal(ilb.decode_lanes_full(c), msg)
                assert ilb.encode_lanes_full(msg, t, lanes).to_bytes() == c.to_bytes()


def test_max_lanes_65535():
    rng = np.random.default_rng(9)
    t = random_table(rng, max_n=20)
    msg = random_message(rng, t, 200_000)
    c = ilb.encode_interleaved(msg, t, 65535, WORD16)
    ref_p, ref_s = oracle.encode_interleaved_u16(msg, t.freq_u32, t.cum_u32, t.scale_bits, 65535)
    assert np.array_equal(c.payload, ref_p) and c.final_states == tuple(ref_s.tolist())
    assert np.array_equal(ilb.decode_interleaved(c), msg)


def test_truncation_raises_like_reference():
    rng = np.random.default_rng(63)
    t = random_table(rng)
    for lanes in (1, 2, 4, 8, 16, 32, 40, 100, 200):
        msg = random_message(rng, t, 1500)
        c = ilb.encode_interleaved(msg, t, lanes, WORD16)
        if len(c.payload) == 0:
            continue
        for cut in (0, len(c.payload) // 3, len(c.payload) - 1):
            c2 = Container(c.variant, c.lane_count, c.message_length, c.table, c.final_states,
                           c.payload[:cut])
            with pytest.raises(TruncatedStreamError):
                ilb.decode_interleaved(c2)
            if lanes <= 32:
                with pytest.raises(TruncatedStreamError):
                    ilb.decode_lanes_full(c2)


def test_unencodable_symbol():
    t = SymbolTable([4, 0], 2)
    with pytest.raises(UnencodableSymbolError, match="symbol 1"):
        ilb.encode_interleaved([0, 1, 0], t, 2, WORD16)
    with pytest.raises(UnencodableSymbolError):
        ilb.encode_interleaved([0, 1, 0], t, 40, WORD16)
    with pytest.raises(UnencodableSymbolError):
        B.encode_interleaved_u16(np.array([0, 1], np.uint8), [4, 0], [0, 4, 4], 2, 1)


@pytest.mark.parametrize("sb", [2, 8, 12, 13, 14])
def test_fast_encoder_record_edges(sb):
    """Tables at the edge of the fast encoder record (common.cuh EncFast:
    sb <= 12, every f <= m/2): f = m/2 exactly and f = 1 symbols take it,
    f = m/2 + 1 falls back to the 33-bit magic; both match the oracle on
    N = 32 streams long enough for the unrolled batches."""
    from paper_1402_3392_b200.chunked import decode_chunked, encode_chunked

    m = 1 << sb
    rng = np.random.default_rng(100 + sb)
    tables = [[m // 2, m // 2], [m // 2 + 1, m // 2 - 1] if m > 2 else [1, 1]]
    if m >= 8:
        k = min(m // 2 - 1, 200)                           # many f = 1 symbols
        tables.append([1] * k + [m // 2, m // 2 - k])
        tables.append([1] * k + [m - k])
    for freq in tables:
        t = SymbolTable(freq, sb)
        msg = random_message(rng, t, 70_001)
        for lanes in (32, 16, 8, 4, 1, 31, 7, 3):  # N < 32: 512/N- or 256/N-group batches
            payload, states = B.encode_interleaved_u16(msg, t.freq_u32, t.cum_u32, sb, lanes)
            ref_p, ref_s = oracle.encode_interleaved_u16(msg, t.freq_u32, t.cum_u32, sb, lanes)
            assert np.array_equal(payload, ref_p) and np.array_equal(states, ref_s), (freq, lanes)
            out, used = B.decode_interleaved_u16(payload, states, t.slot_u8, t.freq_u32,
                                                 t.cum_u32, sb, len(msg), lanes)
            assert np.array_equal(out, msg) and used == len(payload), (freq, lanes)
        cc = encode_chunked(msg, t, 32, 4096)
        ref_p, _, ref_s = oracle.encode_chunks_u16(msg, 4096, t.freq_u32, t.cum_u32, sb, 32)
        assert np.array_equal(cc.payload, ref_p) and np.array_equal(cc.states, ref_s), freq
        assert np.array_equal(decode_chunked(cc), msg)


def test_unencodable_symbol_in_fast_batches():
    """Zero-frequency symbols deep inside the unrolled fast path: the error
    names the symbol at the highest offending index (the reference's
    backward walk meets it first, _core.pyx:33-34)."""
    t = SymbolTable([2048, 2047, 0, 0, 1], 12)
    for lanes in (32, 8, 1, 7, 3, 40, 64, 100, 200, 256):
        msg = np.zeros(70_000, dtype=np.uint8)
        msg[100], msg[60_000] = 2, 3
        with pytest.raises(UnencodableSymbolError, match="symbol 3"):
            ilb.encode_interleaved(msg, t, lanes, WORD16)
        msg[60_000] = 1
        msg[40_000] = 2
        with pytest.raises(UnencodableSymbolError, match="symbol 2"):
            ilb.encode_interleaved(msg, t, lanes, WORD16)
    # two in one group, lower sub-group first (the wide coders' S x 32 lanes)
    for lanes in (64, 100, 200, 256):
        msg = np.zeros(70_000, dtype=np.uint8)
        base = (50_000 // lanes) * lanes
        msg[base + 3], msg[base + lanes - 2] = 2, 3
        with pytest.raises(UnencodableSymbolError, match="symbol 3"):
            ilb.encode_interleaved(msg, t, lanes, WORD16)


def test_trailing_garbage_warns():
    t = SymbolTable([1, 3], 2)
    c = ilb.encode_interleaved([1, 0, 1, 1, 0] * 20, t, 1, WORD16)
    c.payload = np.concatenate([c.payload, np.asarray([123], dtype=np.uint16)])
    with pytest.warns(TrailingGarbageWarning):
        out = ilb.decode_interleaved(c)
    assert out.tolist() == [1, 0, 1, 1, 0] * 20


def test_golden_container_through_gpu():
    t = SymbolTable([1, 3], 2)
    c = ilb.encode_interleaved([1], t, 1, WORD16)
    assert c.final_states == (87382,) and len(c.payload) == 0
    assert ilb.decode_interleaved(Container.from_bytes(c.to_bytes())).tolist() == [1]


def test_wrong_lane_count_never_silently_matches():
    rng = np.random.default_rng(23)
    t = random_table(rng)
    msg = random_message(rng, t, 5000)
    blob = bytearray(ilb.encode_interleaved(msg, t, 4, WORD16).to_bytes())
    blob[6] = 5
    tampered = Container.from_bytes(bytes(blob))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        try:
            out = ilb.decode_interleaved(tampered)
        except (TruncatedStreamError, FormatError):
            return
    assert not np.array_equal(out, msg)


# -------------------------------------------------------- chunk framing ---
def test_chunked_matches_reference_per_chunk(golden_chunks, golden_meta):
    from paper_1402_3392_b200.chunked import decode_chunked, encode_chunked

    for case in golden_meta["chunks"]:
        k, sb, C = case["case"], case["scale_bits"], case["chunk"]
        msg = golden_chunks[f"k{k}_msg"]
        t = SymbolTable(golden_chunks[f"k{k}_freq"].tolist(), sb)
        cc = encode_chunked(msg, t, 32, C)
        assert np.array_equal(cc.payload, golden_chunks[f"k{k}_payload"])
        assert np.array_equal(cc.word_offsets, golden_chunks[f"k{k}_offsets"])
        assert np.array_equal(cc.states, golden_chunks[f"k{k}_states"])
        assert np.array_equal(decode_chunked(cc), msg)
        # device model build == host reference model (bincount + quantize)
        cc2 = encode_chunked(msg, None, 32, C, sb)
        assert cc2.table == SymbolTable.from_counts(
            np.bincount(msg, minlength=int(msg.max()) + 1).tolist(), sb)
        # every chunk is a standalone IEC1 container
        for j in (0, cc.n_chunks - 1):
            one = Container.from_bytes(cc.chunk(j).to_bytes())
            assert np.array_equal(ilb.decode_interleaved(one), msg[j * C:(j + 1) * C])


@pytest.mark.parametrize("sb", [12, 15])
def test_full_size_config2_properties(sb):
    """BASELINE config 2 at full size (256 MiB, 4096 x 64 KiB chunks, N=32):
    size-independent properties -- exact round trip, every chunk consumes its
    whole payload and returns all lanes to L, the device model equals
    bincount + quantize, and sampled chunks equal the oracle's encode."""
    import torch

    from paper_1402_3392_b200.chunked import DeviceCodec, n_chunks_for
    from paper_1402_3392_b200.synth import synth_device

    n, C = 256 << 20, 65536
    k = n_chunks_for(n, C)
    d_msg = synth_device(n, 1.1, 77)
    d_out = torch.empty(n, dtype=torch.uint8, device=d_msg.device)
    codec = DeviceCodec(n, C, 32, sb)
    codec.reset_status()
    codec.histogram(d_msg, n)
    codec.build_table_from_counts()
    codec.encode(d_msg, n)
    codec.decode(d_out, n, final_states=True)
    codec.check_status()
    torch.cuda.synchronize()
    assert torch.equal(d_out, d_msg[:n])
    offs = codec.offsets[: k + 1].cpu().numpy().view(np.uint64)
    assert np.array_equal(codec.consumed[:k].cpu().numpy().view(np.uint64), np.diff(offs))
    assert (codec.final_states[: k * 32].cpu().numpy().view(np.uint32) == 1 << 16).all()
    msg = d_msg[:n].cpu().numpy()
    counts, alpha = oracle.histogram(msg)
    assert np.array_equal(codec.counts.cpu().numpy().view(np.uint64), counts)
    table = codec.read_table()
    assert table.freq == oracle.quantize(counts[:alpha], sb)
    payload = codec.payload[: int(offs[-1])].cpu().numpy().view(np.uint16)
    states = codec.states[: k * 32].cpu().numpy().view(np.uint32).reshape(k, 32)
    for j in (0, 1, 2047, k - 1):
        chunk = msg[j * C:(j + 1) * C]
        p, s = oracle.encode_interleaved_u16(chunk, table.freq_u32, table.cum_u32, sb, 32)
        assert np.array_equal(payload[int(offs[j]):int(offs[j + 1])], p)
        assert np.array_equal(states[j], s)


def test_chunked_edge_shapes():
    from paper_1402_3392_b200.chunked import ChunkedContainer, decode_chunked, encode_chunked

    rng = np.random.default_rng(4)
    for n, C, lanes in ((0, 1024, 32), (1, 16, 1), (17, 16, 3), (4096, 1024, 32),
                        (100_000, 1008, 7), (65536 * 3 + 5, 65536, 32)):
        t = random_table(rng)
        msg = random_message(rng, t, n)
        cc = encode_chunked(msg, t, lanes, C)
        ref_p, ref_o, ref_s = oracle.encode_chunks_u16(msg, C, t.freq_u32, t.cum_u32,
                                                       t.scale_bits, lanes)
        assert np.array_equal(cc.payload, ref_p) and np.array_equal(cc.states, ref_s)
        back = ChunkedContainer.from_bytes(cc.to_bytes())
        assert np.array_equal(decode_chunked(back), msg)


@pytest.mark.parametrize("C, lanes, sb", [(16, 1, 12), (512, 32, 12), (1024, 32, 14),
                                           (2048, 32, 13)])
def test_chunked_many_chunks_per_warp(C, lanes, sb):
    """More chunks than one wave of warps (the coders run one CTA per SM
    with at most 28 warps, so each warp walks several chunks): every chunk
    still matches the oracle's framing and decodes."""
    from paper_1402_3392_b200.chunked import decode_chunked, encode_chunked

    n = 148 * 28 * 3 * C + 11  # > 3 chunks per warp
    rng = np.random.default_rng(C + sb)
    counts = (rng.zipf(1.3, 256) % 1000 + 1).tolist()
    t = SymbolTable(oracle.quantize(counts, sb), sb)
    msg = random_message(rng, t, n)
    cc = encode_chunked(msg, t, lanes, C)
    ref_p, ref_o, ref_s = oracle.encode_chunks_u16(msg, C, t.freq_u32, t.cum_u32, sb, lanes)
    assert np.array_equal(cc.payload, ref_p) and np.array_equal(cc.states, ref_s)
    assert np.array_equal(decode_chunked(cc), msg)


@pytest.mark.parametrize("sb", [11, 12, 13])
def test_chunked_skewed_tables_both_lut_forms(sb):
    """The packed decode entry holds f in 12 bits: a single-symbol source at
    sb=12 (f = 4096) must take the two-lookup form, f = 4095 and sb = 11
    the packed one; all decode through the device-built model."""
    from paper_1402_3392_b200.chunked import decode_chunked, encode_chunked

    rng = np.random.default_rng(sb)
    single = np.full(70_000, 9, dtype=np.uint8)
    skew = np.zeros(70_000, dtype=np.uint8)
    skew[rng.integers(0, len(skew), 3)] = 1   # -> f = {m - 1, 1}
    for msg in (single, skew):
        cc = encode_chunked(msg, None, 32, 4096, sb)
        t = cc.table
        ref_p, _, ref_s = oracle.encode_chunks_u16(msg, 4096, t.freq_u32, t.cum_u32, sb, 32)
        assert np.array_equal(cc.payload, ref_p) and np.array_equal(cc.states, ref_s)
        assert np.array_equal(decode_chunked(cc), msg)
        c = ilb.encode_interleaved(msg, t, 32, WORD16)
        assert np.array_equal(ilb.decode_interleaved(c), msg)


@pytest.mark.parametrize("n, C, lanes, sb, zipf", [
    (3_000_017, 65536, 32, 12, 1.1),    # packed LUT, fast batches, partial last chunk
    (1_000_003, 16384, 7, 12, 1.4),     # generic per-group loop (N < 32)
    (700_001, 4096, 32, 14, 0.8),       # two-lookup LUT (sb > 12)
    (300, 1024, 32, 11, 1.1),           # one partial chunk: tail only
])
def test_decode_fused_adler32_matches_zlib(n, C, lanes, sb, zipf):
    """Decode fused with its consumer: the per-chunk Adler-32
    computed in registers by the decoder equals zlib.adler32 of each chunk
    of the original message, and the stream is consumed exactly."""
    import zlib

    import torch

    from paper_1402_3392_b200.chunked import DeviceCodec, n_chunks_for
    from paper_1402_3392_b200.synth import synth_host

    msg = synth_host(n, zipf, seed=n)
    dev = torch.device("cuda", 0)
    codec = DeviceCodec(n, C, lanes, sb, dev)
    d_msg = torch.from_numpy(msg).to(dev)
    codec.histogram(d_msg, n)
    codec.build_table_from_counts()
    codec.reset_status()
    codec.encode(d_msg, n)
    adler = codec.decode_adler32(n).cpu().numpy().view(np.uint32)
    codec.check_status()
    k = n_chunks_for(n, C)
    want = [zlib.adler32(msg[i * C:(i + 1) * C].tobytes()) for i in range(k)]
    assert adler.tolist() == want
    assert codec.adler32(d_msg, n).cpu().numpy().view(np.uint32).tolist() == want
    offs = codec.offsets[: k + 1].cpu().numpy()
    assert np.array_equal(codec.consumed[:k].cpu().numpy(), offs[1:] - offs[:-1])


def test_fuzz_random_shapes_against_oracle():
    """Randomized sweep over lane counts, chunk lengths, message lengths,
    table shapes and scale_bits: chunked encode/decode and the single-stream
    drop-ins agree with the oracle bit for bit."""
    from paper_1402_3392_b200.chunked import decode_chunked, encode_chunked

    import os

    rng = np.random.default_rng(int(os.environ.get("ILANS_FUZZ_SEED", "2026")))
    for it in range(int(os.environ.get("ILANS_FUZZ_ITERS", "60"))):
        sb = int(rng.integers(1, 17))
        n_sym = int(rng.integers(1, min(256, 1 << sb) + 1))
        counts = rng.integers(0, 50, size=n_sym) ** int(rng.integers(1, 4))
        counts[int(rng.integers(0, n_sym))] += 1
        t = SymbolTable(oracle.quantize(counts, sb), sb)
        n = int(rng.choice([0, 1, 31, 32, 33, 511, 512, 513, 4097, 70_001, 300_000]))
        lanes = int(rng.choice([1, 2, 3, 4, 7, 8, 16, 31, 32]))
        C = int(rng.choice([16, 512, 1024, 4096, 65536]))
        msg = random_message(rng, t, n)
        cc = encode_chunked(msg, t, lanes, C)
        ref_p, ref_o, ref_s = oracle.encode_chunks_u16(msg, C, t.freq_u32, t.cum_u32, sb, lanes)
        assert np.array_equal(cc.payload, ref_p), (it, sb, n, lanes, C)
        assert np.array_equal(cc.states, ref_s), (it, sb, n, lanes, C)
        assert np.array_equal(decode_chunked(cc), msg), (it, sb, n, lanes, C)
        if n <= 70_001:
            N = int(rng.choice([1, 2, 5, 8, 16, 32, 33, 100]))
            p, st = B.encode_interleaved_u16(msg, t.freq_u32, t.cum_u32, sb, N)
            rp, rs = oracle.encode_interleaved_u16(msg, t.freq_u32, t.cum_u32, sb, N)
            assert np.array_equal(p, rp) and np.array_equal(st, rs), (it, sb, n, N)
            out, used = B.decode_interleaved_u16(p, st, t.slot_u8, t.freq_u32, t.cum_u32, sb,
                                                 n, N)
            assert np.array_equal(out, msg) and used == len(p), (it, sb, n, N)


def test_decode_from_slot_layout_matches_packed_decode():
    """DeviceCodec.decode_slots (straight from the encode scratch, no
    packing pass) returns the message, consumes exactly each chunk's word
    count, and matches the packed-stream decode and its final states; the
    fused Adler-32 over the slot layout equals zlib per chunk."""
    import zlib

    import torch

    from paper_1402_3392_b200.chunked import DeviceCodec
    from paper_1402_3392_b200.synth import synth_host

    for n, C, N, sb in ((3_000_017, 65536, 32, 12), (1_000_000, 16384, 32, 14),
                        (700_001, 4096, 7, 11), (250_000, 1024, 16, 15)):
        msg = synth_host(n, 1.2, seed=n)
        d = torch.from_numpy(msg).cuda()
        codec = DeviceCodec(n, C, N, sb)
        codec.histogram(d, n)
        codec.build_table_from_counts()
        codec.reset_status()
        codec.encode(d, n, frame=False)
        offs = codec.directory(n).clone()
        k = len(offs) - 1
        out = torch.empty(n, dtype=torch.uint8, device="cuda")
        codec.decode_slots(out, n, final_states=True)
        codec.check_status()
        assert np.array_equal(out.cpu().numpy(), msg)
        words = codec.chunk_words[:k].to(torch.int64)
        assert torch.equal(codec.consumed[:k], words)
        assert torch.equal(offs[1:] - offs[:-1], words)
        fs_slots = codec.final_states[: k * N].clone()
        codec.frame_range(n, 0, k, codec.payload.data_ptr())
        out2 = torch.empty_like(out)
        codec.decode(out2, n, final_states=True)
        codec.check_status()
        assert torch.equal(out, out2) and torch.equal(codec.final_states[: k * N], fs_slots)
        ad = codec.decode_adler32(n, slots=True).cpu().numpy().view(np.uint32)
        ref = [zlib.adler32(msg[i * C:(i + 1) * C].tobytes()) for i in range(k)]
        assert ad.tolist() == ref


def test_chunked_covered_encode_equals_checked_encode_and_user_tables_still_check():
    """The covered entry (table quantized from this message's own histogram,
    no zero-frequency check) writes exactly what the checking entry writes;
    a user table (build_table_from_freq) keeps the check and reports the
    highest zero-frequency index like the reference."""
    import torch

    from paper_1402_3392_b200.chunked import DeviceCodec
    from paper_1402_3392_b200.synth import synth_host

    for sb in (12, 14):
        n, C = 2_000_003, 65536
        msg = synth_host(n, 1.1, seed=sb)
        d = torch.from_numpy(msg).cuda()
        codec = DeviceCodec(n, C, 32, sb)
        codec.histogram(d, n)
        codec.build_table_from_counts()
        assert codec._covers == (d.data_ptr(), n)
        codec.reset_status()
        codec.encode(d, n)  # covered entry
        codec.check_status()
        covered = codec.encoded_host(n, codec.read_table())
        k = covered.n_chunks
        codec.reset_status()
        codec.encode_range(d.data_ptr(), n, 0, k, covered=False)  # checking entry
        codec.frame_range(n, 0, k, codec.payload.data_ptr())
        codec.check_status()
        checked = codec.encoded_host(n, covered.table)
        assert covered.to_bytes() == checked.to_bytes()
        # a user table without symbol 200 while the message holds it
        freqs = list(covered.table.freq)
        msg2 = msg.copy()
        msg2[1_500_000] = 200
        msg2[10] = 200
        if 200 < len(freqs) and freqs[200]:
            moved = freqs[200]
            freqs[200] = 0
            freqs[0] += moved
        t = SymbolTable(freqs, sb)
        d2 = torch.from_numpy(msg2).cuda()
        codec.build_table_from_freq(t)
        assert codec._covers is None
        codec.reset_status()
        codec.encode(d2, n)
        want = int(np.nonzero(msg2 == 200)[0].max())  # the highest offending index
        with pytest.raises(UnencodableSymbolError, match=f"index {want}$"):
            codec.check_status()


@pytest.mark.parametrize("C, sb", [(1536, 12), (2560 + 96, 12), (1536, 14), (512 * 7, 13)])
def test_chunked_odd_block_counts_match_oracle(C, sb):
    """Chunks whose 512-byte block count is odd (with and without a tail):
    the encoder's pair-of-blocks loop hands the last block to the one-block
    loop; every chunk equals the oracle's."""
    from paper_1402_3392_b200.chunked import decode_chunked, encode_chunked
    from paper_1402_3392_b200.synth import synth_host

    msg = synth_host(C * 300 + 777, 1.15, seed=C + sb)
    cc = encode_chunked(msg, None, 32, C, sb)
    t = cc.table
    p, o, st = oracle.encode_chunks_u16(msg, C, t.freq_u32, t.cum_u32, sb, 32)
    assert np.array_equal(cc.payload, p) and np.array_equal(cc.word_offsets, o)
    assert np.array_equal(cc.states, st)
    assert np.array_equal(decode_chunked(cc), msg)
