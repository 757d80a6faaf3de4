"""The N = 32 encoder's direct spill stores keep the stack top's byte address
as a 32-bit low word beside a fixed high word; an iteration that could
borrow across a 4 GiB boundary runs the 64-bit ("wide") body instead
(csrc/encode.cu, QUAD pair loop). Here the encode scratch is placed inside a
>4 GiB device buffer so that chunks' slots cross a 4 GiB boundary at several
positions -- inside the fast loop, at an iteration edge, in the per-group
tail -- and the framed stream must equal, byte for byte, the one encoded
with an ordinary scratch (contract: per chunk, reference
interleave.py:182-212 / _core.pyx:14-43)."""

import numpy as np
import pytest
import torch

from paper_1402_3392_b200 import _lib
from paper_1402_3392_b200.chunked import DeviceCodec, n_chunks_for
from paper_1402_3392_b200.synth import synth_device

pytestmark = pytest.mark.gpu

GIB4 = 1 << 32


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if _lib.device_count() == 0:
        pytest.fail("no CUDA device: the -m gpu suite must run on a B200")


def _framed(codec, d_msg, n):
    codec.reset_status()
    codec.histogram(d_msg, n)
    codec.build_table_from_counts()
    codec.encode(d_msg, n)  # encode + offset scan + compaction
    codec.check_status()
    k = n_chunks_for(n, codec.chunk_len)
    offs = codec.offsets[: k + 1].clone()
    words = int(offs[-1])
    return (codec.payload[:words].clone(), offs, codec.states[: k * codec.lane_count].clone(),
            codec.chunk_words[:k].clone())


@pytest.mark.parametrize("sb, zipf_s", [(12, 1.1), (14, 1.1), (12, 2.97)])
def test_encode_scratch_across_4gib_boundary(sb, zipf_s):
    """zipf_s = 2.97 (H ~ 1 bit) gives a symbol above m/2: the EncQuadX
    records (exact 33-bit magic) on the same paths."""
    dev = torch.device("cuda", 0)
    C, N, k = 65536, 32, 6
    n = C * k - 777  # a short last chunk (per-group tail + fast blocks)
    d_msg = synth_device(n, zipf_s, 99, device=dev)
    ref = _framed(DeviceCodec(n, C, N, sb, dev), d_msg, n)
    w = ref[3].cpu().numpy().astype(np.int64)  # words per chunk (right-aligned in the slot)

    big = torch.empty(GIB4 + (8 << 20), dtype=torch.uint8, device=dev)
    base = big.data_ptr()
    boundary = (base // GIB4 + 1) * GIB4  # the 4 GiB boundary inside `big`
    assert base < boundary < base + big.numel() - (4 << 20)
    codec = DeviceCodec(n, C, N, sb, dev)
    # chunk j's written words are scratch words [jC + len_j - w_j, jC + len_j);
    # put the boundary `back` words below chunk j's slot top
    cases = [(2, 1000), (2, 1024), (3, 5), (1, int(w[1]) - 3), (4, 4096 + 17)]
    for j, back in cases:
        len_j = min(C, n - j * C)
        top_word = j * C + len_j
        start = boundary - 2 * (top_word - back)
        start -= start % 16  # keep the scratch 16-byte aligned (shifts the crossing by < 8 words)
        off = start - base
        assert 0 <= off and off + 2 * (n + 8) <= big.numel()
        codec.scratch = big[off: off + 2 * (n + 8)].view(torch.int16)
        got = _framed(codec, d_msg, n)
        for a, b, name in zip(got, ref, ("payload", "offsets", "states", "chunk_words")):
            assert torch.equal(a, b), (sb, j, back, name)
        d_out = torch.empty(n, dtype=torch.uint8, device=dev)
        codec.reset_status()
        codec.decode(d_out, n)
        codec.check_status()
        assert torch.equal(d_out, d_msg[:n]), (sb, j, back)
    del big
    torch.cuda.empty_cache()
