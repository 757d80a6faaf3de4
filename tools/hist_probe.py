"""Histogram kernel alone at 256 MiB (config 2's message): CUDA-event time
per launch on the launching stream."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1402_3392_b200 import _lib
from paper_1402_3392_b200.synth import synth_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256 << 20
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
dev = torch.device("cuda", 0)
d = synth_device(n, 1.1, 1234, device=dev)
counts = torch.zeros(256, dtype=torch.int64, device=dev)
s = torch.cuda.current_stream().cuda_stream
for _ in range(5):
    _lib.lib.ilans_histogram_u8_dev(d.data_ptr(), n, counts.data_ptr(), s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    _lib.lib.ilans_histogram_u8_dev(d.data_ptr(), n, counts.data_ptr(), s)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"histogram n={n}: {ms*1e3:.1f} us/launch, {n/ms/1e6:.0f} GB/s")
