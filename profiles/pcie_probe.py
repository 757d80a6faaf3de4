"""Host<->device copy ceilings on this box (pinned memory), for the e2e
numbers: H2D, D2H, and both directions at once, 256 MiB, CUDA events."""

import json

import torch


def main():
    n = 256 << 20
    dev = torch.device("cuda", 0)
    h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d1 = torch.empty(n, dtype=torch.uint8, device=dev)
    d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(reps):
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best

    out["h2d_GBps"] = n / (timed(lambda: d1.copy_(h1, non_blocking=True)) * 1e-3) / 1e9
    out["d2h_GBps"] = n / (timed(lambda: h2.copy_(d2, non_blocking=True)) * 1e-3) / 1e9

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    out["bidir_GBps_each"] = n / (timed(both) * 1e-3) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
