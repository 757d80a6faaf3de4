"""e2e (HostCodec async round trips from pinned memory) at several step
counts: how much of the per-step time is pipeline fill / drain."""
import sys, os, types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1402_3392_b200.synth import synth_device

n = 256 << 20
dev = torch.device("cuda", 0)
d_msg = synth_device(n, 1.1, 1234, device=dev)
for steps in [int(s) for s in (sys.argv[1] if len(sys.argv) > 1 else "4,8,16,32").split(",")]:
    a = types.SimpleNamespace(steps=steps)
    r = bench.e2e(a, n, n // 65536, 65536, 32, 12, dev, d_msg, None, 1, n,
                  slots=int(os.environ.get("SLOTS", "3")))
    print(steps, round(r["value"], 2), "seq", round(r["sequential_GBps"], 2), r["steps"])
