"""One single-stream encode + decode at N lanes (default 33): the wide
one-warp kernels, for an ncu capture."""
import sys
import numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
import paper_1402_3392_b200 as ilb
from paper_1402_3392_b200.synth import synth_host

N = int(sys.argv[1]) if len(sys.argv) > 1 else 33
msg = synth_host(1 << 20, 1.1, seed=1)
t = ilb.SymbolTable.from_counts(np.bincount(msg, minlength=256).tolist(), 14)
c = ilb.encode_interleaved(msg, t, N)
assert bytes(ilb.decode_interleaved(c)) == bytes(msg)
print("ok", N, len(c.payload) if hasattr(c, "payload") else "")
