"""Break down the HostCodec end-to-end round trip (encode / decode wall time
per call, batch sizes) to see where PCIe and the kernels overlap."""

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
    dev = torch.device("cuda", 0)
    d = synth_device(n, 1.1, 1234, device=dev)
    h_msg = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_msg.copy_(d[:n])
    h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    res = {}
    for batch in (8 << 20, 32 << 20, 64 << 20, 256 << 20):
        hc = HostCodec(n, 65536, 32, 12, dev, batch_bytes=batch)
        p, o, s = hc.encode(h_msg, n)
        hc.decode(p, o, s, n, h_out)
        assert torch.equal(h_out, h_msg)
        enc, dec = [], []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            p, o, s = hc.encode(h_msg, n)
            t1 = time.perf_counter()
            hc.decode(p, o, s, n, h_out)
            t2 = time.perf_counter()
            enc.append(t1 - t0)
            dec.append(t2 - t1)
        res[f"batch_{batch >> 20}MiB"] = {"encode_ms": 1e3 * min(enc), "decode_ms": 1e3 * min(dec),
                                          "round_trip_GBps": n / (min(enc) + min(dec)) / 1e9}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
