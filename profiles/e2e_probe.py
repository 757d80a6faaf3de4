"""Timeline of the HostCodec end-to-end round trips (pipelined two deep, as
bench.py's e2e runs them): per step, device timestamps of the message
upload, the encode kernel, the payload download, the payload upload and the
decoded-bytes download, relative to the first step's start.

    python profiles/e2e_probe.py [batch_MiB]
"""

import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1402_3392_b200.chunked import HostCodec  # noqa: E402
from paper_1402_3392_b200.synth import synth_device  # noqa: E402


def main():
    n = 256 << 20
    batch = (int(sys.argv[1]) if len(sys.argv) > 1 else 32) << 20
    slots = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    depth = int(sys.argv[3]) if len(sys.argv) > 3 else 2  # decodes in flight
    dev = torch.device("cuda", 0)
    d = synth_device(n, 1.1, 1234, device=dev)
    h_msg = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_msg.copy_(d[:n])
    outs = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(4)]
    hc = HostCodec(n, 65536, 32, 12, dev, batch_bytes=batch, slots=slots)
    for i in range(3):
        hc.decode_async(hc.encode_async(h_msg, n), outs[i % 2]).wait()
    torch.cuda.synchronize()
    hc.trace = []
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    w0 = time.perf_counter()
    pend = []
    steps = 10
    ejs = [hc.encode_async(h_msg, n)]
    for i in range(steps):
        hc._mark(f"step{i}", torch.cuda.current_stream())
        if i + 1 < steps:
            ejs.append(hc.encode_async(h_msg, n))
        pend.append(hc.decode_async(ejs[i], outs[i % 4]))
        if len(pend) == depth:
            pend.pop(0).wait()
    for p in pend:
        p.wait()
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    rows = [(name, round(t0.elapsed_time(e), 3)) for name, e in hc.trace]
    print(json.dumps({"batch_MiB": batch >> 20, "slots": slots, "depth": depth, "GBps": n * steps / wall / 1e9,
                      "ms_per_step": 1e3 * wall / steps}))
    for name, t in rows:
        print(f"{t:9.3f}  {name}")


if __name__ == "__main__":
    main()
