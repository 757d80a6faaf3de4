"""Chunked byte8 throughput on one B200 (device-resident, CUDA events):
encode (one warp per chunk) + byte framing, and decode, at 256 MiB of the
config-2 Zipf source, for N = 2 (config 1's lane count) and N = 32.

    python tools/byte8_chunked_probe.py [mib] [lanes:chunk,...]
"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
from paper_1402_3392_b200 import _lib  # noqa: E402
from paper_1402_3392_b200.chunked import _Model, n_chunks_for  # noqa: E402
from paper_1402_3392_b200.synth import synth_device  # noqa: E402

mib = int(sys.argv[1]) if len(sys.argv) > 1 else 256
n = mib << 20
dev = torch.device("cuda", 0)
d_msg = synth_device(n, 1.1, 1234)
m = _Model(torch, dev)
table = m.from_message(d_msg, n, 12)
p = lambda t: int(t.data_ptr())  # noqa: E731
cases = ((2, 65536), (32, 65536), (32, 16384))
if len(sys.argv) > 2:
    cases = [tuple(int(v) for v in c.split(":")) for c in sys.argv[2].split(",")]
for lanes, C in cases:
    k = n_chunks_for(n, C)
    scratch = torch.empty(3 * n + 16, dtype=torch.uint8, device=dev)
    payload = torch.empty(3 * n + 16, dtype=torch.uint8, device=dev)
    nbytes = torch.zeros(k, dtype=torch.int32, device=dev)
    offs = torch.zeros(k + 1, dtype=torch.int64, device=dev)
    states = torch.empty(k * lanes, dtype=torch.int32, device=dev)
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    consumed = torch.zeros(k, dtype=torch.int64, device=dev)

    def enc():
        _lib.check_dev(_lib.lib.ilans_encode_chunks_u8_dev(
            p(d_msg), n, C, lanes, p(m.table), p(scratch), p(nbytes), p(states), p(m.status),
            m.s), "enc")
        _lib.check_dev(_lib.lib.ilans_frame_chunks_u8_dev(
            p(scratch), n, C, p(nbytes), p(offs), p(payload), m.s), "frame")

    def dec():
        _lib.check_dev(_lib.lib.ilans_decode_chunks_u8_dev(
            p(payload), p(offs), p(states), n, C, lanes, p(m.table), p(out), p(consumed),
            p(m.status), m.s), "dec")

    def timed(f, reps=5):
        f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            f()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    m.reset()
    te = timed(enc)
    td = timed(dec)
    m.check()
    assert torch.equal(out, d_msg[:n])
    total = int(offs[-1].item())
    print(f"byte8 chunked N={lanes} C={C}: encode+frame {n / te / 1e6:.1f} GB/s ({te:.3f} ms), "
          f"decode {n / td / 1e6:.1f} GB/s ({td:.3f} ms), {8 * total / n:.3f} bits/byte")
