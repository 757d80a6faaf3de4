"""Reference-suite behaviours on the B200 path that go beyond plain
encode/decode: lockstep step generators (acceptance criterion 2,
pkg/tests/test_acceptance.py:65-88), the stats= counters (criterion 3,
test_acceptance.py:91-110; test_interleave.py:128-142) and the
decoder-returns-to-L property (test_interleave.py:114-121). The expected
step traces come from the oracle's serial decoder run group by group."""

import numpy as np
import pytest

import oracle
import paper_1402_3392_b200 as ilb
from paper_1402_3392_b200 import _lib
from paper_1402_3392_b200.errors import TruncatedStreamError, UnsupportedVariantError
from paper_1402_3392_b200.interleave import Container, decode_interleaved_steps
from paper_1402_3392_b200.lanes import MAX_LANES, decode_lanes_steps
from paper_1402_3392_b200.rans import BYTE8, WORD16, RenormStats, SymbolTable

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if _lib.device_count() == 0:
        pytest.fail("no CUDA device: the -m gpu suite must run on a B200")


def random_table(rng, max_n=64, max_scale=14):
    n = int(rng.integers(2, max_n + 1))
    sb = int(rng.integers(max(1, (n - 1).bit_length()), max_scale + 1))
    counts = rng.integers(0, 900, size=n)
    counts[int(rng.integers(0, n))] += 1
    return SymbolTable(oracle.quantize(counts, sb), sb)


def random_message(rng, table, n):
    return rng.choice(table.alphabet_size, size=n, p=table.freq_u32 / table.total).astype(np.uint8)


def oracle_steps(c: Container):
    """Per-group (symbols, states, read_pos) from the oracle's serial decoder."""
    t, N, n = c.table, c.lane_count, c.message_length
    f, cum, slot = t.freq_u32, t.cum_u32, t.slot_u8
    states = np.asarray(c.final_states, dtype=np.uint32)
    out = []
    pos = 0
    for base in range(0, n, N):
        active = min(N, n - base)  # one group: symbols base .. base+active-1
        o, used, states = oracle._decode(oracle.lib().orc_decode_u16, c.payload[pos:], states,
                                         slot, f, cum, t.scale_bits, active, N)
        pos += used
        out.append((tuple(o.tolist()), tuple(int(x) for x in states), pos))
    return out


def test_lockstep_steps_match_serial_decoder():
    rng = np.random.default_rng(2026)
    for lanes in (1, 2, 4, 8, 16, 32, 40):
        for n in (0, 1, max(0, lanes - 1), lanes, lanes + 1, 2 * lanes + 1, 97, 1500):
            t = random_table(rng)
            msg = random_message(rng, t, n)
            c = ilb.encode_interleaved(msg, t, lanes, WORD16)
            want = oracle_steps(c)
            got = list(decode_interleaved_steps(c))
            assert got == want, (lanes, n)
            if lanes <= MAX_LANES:
                assert list(decode_lanes_steps(c)) == want
            if n:
                assert got[-1][1] == (WORD16.lower_bound,) * lanes  # back to L
                assert got[-1][2] == len(c.payload)
            collected = [s for syms, _, _ in got for s in syms]
            assert collected == msg.tolist()


def test_steps_raise_lazily_on_truncation():
    rng = np.random.default_rng(7)
    t = random_table(rng)
    msg = random_message(rng, t, 3000)
    c = ilb.encode_interleaved(msg, t, 4, WORD16)
    cut = Container(c.variant, 4, c.message_length, t, c.final_states, c.payload[: len(c.payload) // 2])
    gen = decode_interleaved_steps(cut)
    first = next(gen)  # groups before the failure are still produced
    assert first == oracle_steps(c)[0]
    with pytest.raises(TruncatedStreamError):
        for _ in gen:
            pass


def test_steps_reject_unsupported():
    t = SymbolTable([1, 3], 2)
    c8 = Container(BYTE8, 2, 3, t, (1 << 23, 1 << 23), np.zeros(0, np.uint8))
    with pytest.raises(UnsupportedVariantError):
        next(decode_lanes_steps(c8))
    c33 = ilb.encode_interleaved([0, 1] * 40, t, MAX_LANES + 1, WORD16)
    with pytest.raises(UnsupportedVariantError):
        next(decode_lanes_steps(c33))
    assert len(list(decode_interleaved_steps(c33))) == 3  # serial steps are fine


def test_host_codec_batched_pipeline_matches_oracle():
    """HostCodec (pinned host buffers, 3 streams, batches packed straight into
    host memory over PCIe) == the oracle's chunk framing, and round-trips."""
    import torch

    from paper_1402_3392_b200.chunked import HostCodec
    from paper_1402_3392_b200.synth import synth_host

    for n, C, batch in ((5_000_003, 65536, 1 << 20), (300_000, 16384, 64 << 10), (100, 1024, 4096)):
        msg = synth_host(n, 1.3, seed=n)
        hc = HostCodec(n, C, 32, 12, batch_bytes=batch)
        h_msg = torch.from_numpy(msg).pin_memory()
        pay, offs, states = hc.encode(h_msg, n)
        counts, alpha = oracle.histogram(msg)
        freqs = oracle.quantize(counts[:alpha], 12)
        f, cum, _ = oracle.table_views(freqs, 12)
        ref_p, ref_o, ref_s = oracle.encode_chunks_u16(msg, C, f, cum, 12, 32)
        assert np.array_equal(pay.numpy().view(np.uint16), ref_p)
        assert np.array_equal(offs.numpy().view(np.uint64), ref_o)
        assert np.array_equal(states.numpy().view(np.uint32).reshape(-1, 32), ref_s)
        h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        hc.decode(pay.clone(), offs.clone(), states.clone(), n, h_out)
        assert np.array_equal(h_out.numpy(), msg)


def test_host_codec_async_round_trips_overlap():
    """encode_async / decode_async with two slots and three different
    messages in flight the way bench.py pipelines them: every payload equals
    the oracle's chunk framing under that message's own model, every decode
    returns its own message, and slot reuse waits for the earlier round trip."""
    import torch

    from paper_1402_3392_b200.chunked import HostCodec
    from paper_1402_3392_b200.synth import synth_host

    n, C = 3_000_017, 65536
    hc = HostCodec(n, C, 32, 12, batch_bytes=1 << 20, slots=2)
    msgs = [synth_host(n - 7 * i, s, seed=i) for i, s in enumerate((1.1, 1.6, 0.7))]
    outs = [torch.zeros(n, dtype=torch.uint8, pin_memory=True) for _ in msgs]
    pins = [torch.from_numpy(m).pin_memory() for m in msgs]

    def check(i, ej):
        pay, offs, states = ej.wait()
        counts, alpha = oracle.histogram(msgs[i])
        f, cum, _ = oracle.table_views(oracle.quantize(counts[:alpha], 12), 12)
        ref_p, ref_o, ref_s = oracle.encode_chunks_u16(msgs[i], C, f, cum, 12, 32)
        assert np.array_equal(pay.numpy().view(np.uint16), ref_p)
        assert np.array_equal(offs.numpy().view(np.uint64), ref_o)
        assert np.array_equal(states.numpy().view(np.uint32).reshape(-1, 32), ref_s)

    jobs = []
    for i in range(2):
        ej = hc.encode_async(pins[i], len(msgs[i]))
        jobs.append((ej, hc.decode_async(ej, outs[i])))
    check(0, jobs[0][0])
    jobs[0][1].wait()
    ej = hc.encode_async(pins[2], len(msgs[2]))  # reuses slot 0
    jobs.append((ej, hc.decode_async(ej, outs[2])))
    check(1, jobs[1][0])
    check(2, jobs[2][0])
    for i, (_, dj) in enumerate(jobs):
        assert np.array_equal(dj.wait().numpy(), msgs[i])


def test_host_codec_decodes_a_container_with_its_own_table():
    """HostCodec.decode(..., table=) decodes a stored chunked stream with the
    model it carries, not with the model of whatever was encoded last."""
    import torch

    from paper_1402_3392_b200.chunked import ChunkedContainer, HostCodec, encode_chunked
    from paper_1402_3392_b200.synth import synth_host

    n, C = 1_000_003, 65536
    a = synth_host(n, 1.3, seed=5)
    cc = ChunkedContainer.from_bytes(encode_chunked(a, None, 32, C, 12).to_bytes())
    hc = HostCodec(n, C, 32, 12, batch_bytes=1 << 18)
    hc.encode(torch.from_numpy(synth_host(n, 0.6, seed=6)).pin_memory(), n)  # other model
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()  # noqa: E731
    offs = cc.word_offsets.astype(np.int64)
    h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    hc.decode(pin(cc.payload.view(np.int16)), pin(offs), pin(cc.states.reshape(-1).view(np.int32)),
              n, h_out, table=cc.table)
    assert np.array_equal(h_out.numpy(), a)


def test_host_codec_raw_decode_after_async_encode_keeps_both():
    """encode_async(A) then decode_async(raw payload of B, no table=): B is
    decoded with A's model in A's slot without corrupting A's pending
    payload downloads (the raw branch fences every slot stream)."""
    import torch

    from paper_1402_3392_b200.chunked import HostCodec, encode_chunked
    from paper_1402_3392_b200.synth import synth_host

    n, C = 2_500_009, 65536
    a = synth_host(n, 1.2, seed=11)
    b = synth_host(n, 1.25, seed=12)
    hc = HostCodec(n, C, 32, 12, batch_bytes=1 << 19, slots=2)
    ej = hc.encode_async(torch.from_numpy(a).pin_memory(), n)
    ta = encode_chunked(a, None, 32, C, 12)
    cb = encode_chunked(b, ta.table, 32, C, 12)  # B under A's model
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()  # noqa: E731
    h_out = torch.zeros(n, dtype=torch.uint8, pin_memory=True)
    dj = hc.decode_async(pin(cb.payload.view(np.int16)), h_out, n,
                         pin(cb.word_offsets.astype(np.int64)),
                         pin(cb.states.reshape(-1).view(np.int32)))
    assert np.array_equal(dj.wait().numpy(), b)
    pay, offs, states = ej.wait()
    assert np.array_equal(pay.numpy().view(np.uint16), ta.payload)
    assert np.array_equal(offs.numpy().view(np.uint64), ta.word_offsets)
    assert np.array_equal(states.numpy().view(np.uint32).reshape(-1, 32), ta.states)


def test_stats_counters_single_digit_property():
    rng = np.random.default_rng(3)
    stats = RenormStats()
    for _ in range(5):
        t = random_table(rng)
        msg = random_message(rng, t, 50_000)
        c = ilb.encode_interleaved(msg, t, 4, WORD16, stats=stats)
        assert c.to_bytes() == ilb.encode_interleaved(msg, t, 4, WORD16).to_bytes()
        assert np.array_equal(ilb.decode_interleaved(c, stats=stats), msg)
    assert stats.encode_symbols == stats.decode_symbols == 250_000
    assert stats.encode_digits == stats.decode_digits > 0
    assert stats.max_encode_digits == stats.max_decode_digits == 1


def test_stats_are_measured_by_the_kernel():
    """max_decode_digits comes from the kernel: a lane state of 0 (below L,
    handed in directly) pops to x' = 0, one refill leaves it below L, and the
    reference's refill loop (rans.py:305-309) would need a second digit --
    the kernel reports 2. Outputs still follow the compiled kernel
    (_core.pyx:107-112: one refill)."""
    import warnings

    t = SymbolTable([3, 1], 2)
    c = Container(WORD16, 1, 1, t, (0,), np.array([5, 7], dtype=np.uint16))
    stats = RenormStats()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        out = ilb.decode_interleaved(c, stats=stats)
    ref, used = oracle.decode_interleaved_u16(c.payload, np.array([0], np.uint32), t.slot_u8,
                                              t.freq_u32, t.cum_u32, 2, 1, 1)
    assert np.array_equal(out, ref) and used == 1
    assert stats.max_decode_digits == 2 and stats.decode_digits == 1
    # N > 32 and N = 32 go through the CTA / warp kernels' measuring loops too
    rng = np.random.default_rng(5)
    for lanes in (3, 32, 40, 100):
        tt = random_table(rng)
        msg = random_message(rng, tt, 20_000)
        st2 = RenormStats()
        cc = ilb.encode_interleaved(msg, tt, lanes, WORD16, stats=st2)
        assert cc.to_bytes() == ilb.encode_interleaved(msg, tt, lanes, WORD16).to_bytes()
        assert np.array_equal(ilb.decode_interleaved(cc, stats=st2), msg)
        assert st2.max_encode_digits == st2.max_decode_digits == 1
        assert st2.encode_digits == st2.decode_digits == len(cc.payload)


def test_drop_in_calls_from_many_threads():
    """The host-buffer drop-ins keep one context (stream, buffers, pinned
    staging, cached model) per host thread: concurrent calls from 8 threads
    with two alternating tables all return the oracle's bytes."""
    from concurrent.futures import ThreadPoolExecutor

    rng = np.random.default_rng(77)
    tables = [random_table(rng, max_scale=12), random_table(rng, max_scale=14)]
    jobs = []
    for i in range(64):
        t = tables[i % 2]
        jobs.append((t, random_message(rng, t, int(rng.integers(0, 70_000))), 1 + i % 32))

    def run(job):
        t, msg, lanes = job
        c = ilb.encode_interleaved(msg, t, lanes)
        ref_p, ref_s = oracle.encode_interleaved_u16(msg, t.freq_u32, t.cum_u32, t.scale_bits,
                                                     lanes)
        ok = np.array_equal(c.payload, ref_p) and c.final_states == tuple(ref_s.tolist())
        return ok and np.array_equal(ilb.decode_interleaved(c), msg)

    with ThreadPoolExecutor(8) as ex:
        assert all(ex.map(run, jobs))


def test_sharded_codec_gather_single_rank_matches_encode_chunked():
    """ShardedCodec (one rank, no process group): build_global_model +
    encode + gather gives the same ICH1 bytes as encode_chunked."""
    import torch

    from paper_1402_3392_b200.chunked import encode_chunked
    from paper_1402_3392_b200.dist import ShardedCodec
    from paper_1402_3392_b200.synth import synth_host

    n, C = 2_000_003, 65536
    msg = synth_host(n, 1.2, seed=9)
    sc = ShardedCodec(n, 0, 1, C, 32, 12)
    d = torch.from_numpy(msg).cuda()
    sc.build_global_model(d)
    sc.encode(d)
    assert sc.gather(n).to_bytes() == encode_chunked(msg, None, 32, C, 12).to_bytes()
