"""One chunked byte8 encode + frame + decode at N = 32 (for ncu captures)."""
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_1402_3392_b200 import _lib  # noqa: E402
from paper_1402_3392_b200.chunked import _Model, n_chunks_for  # noqa: E402
from paper_1402_3392_b200.synth import synth_device  # noqa: E402

n, C, lanes = (int(sys.argv[1]) if len(sys.argv) > 1 else 64) << 20, 65536, 32
dev = torch.device("cuda", 0)
d_msg = synth_device(n, 1.1, 1234)
m = _Model(torch, dev)
m.from_message(d_msg, n, 12)
p = lambda t: int(t.data_ptr())  # noqa: E731
k = n_chunks_for(n, C)
scratch = torch.empty(3 * n + 16, dtype=torch.uint8, device=dev)
payload = torch.empty(3 * n + 16, dtype=torch.uint8, device=dev)
nbytes = torch.zeros(k, dtype=torch.int32, device=dev)
offs = torch.zeros(k + 1, dtype=torch.int64, device=dev)
states = torch.empty(k * lanes, dtype=torch.int32, device=dev)
out = torch.empty(n, dtype=torch.uint8, device=dev)
consumed = torch.zeros(k, dtype=torch.int64, device=dev)
_lib.check_dev(_lib.lib.ilans_encode_chunks_u8_dev(p(d_msg), n, C, lanes, p(m.table), p(scratch),
                                                   p(nbytes), p(states), p(m.status), m.s), "e")
_lib.check_dev(_lib.lib.ilans_frame_chunks_u8_dev(p(scratch), n, C, p(nbytes), p(offs), p(payload),
                                                  m.s), "f")
_lib.check_dev(_lib.lib.ilans_decode_chunks_u8_dev(p(payload), p(offs), p(states), n, C, lanes,
                                                   p(m.table), p(out), p(consumed), p(m.status),
                                                   m.s), "d")
torch.cuda.synchronize()
assert torch.equal(out, d_msg[:n])
print("ok")
