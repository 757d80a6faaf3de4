import sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1402_3392_b200 import mux as bm
from paper_1402_3392_b200.rans import SymbolTable
from paper_1402_3392_b200.synth import synth_host
K, N, F = 16, 65536, 4096
src = synth_host(K * N, 1.1, seed=7)
t = SymbolTable.from_counts(np.bincount(src, minlength=256).tolist(), 12)
coders = [bm.RansStreamCodec(t) if j % 4 != 3 else bm.RawStreamCodec(12) for j in range(K)]
rng = np.random.default_rng(3)
msgs = [src[j*N:(j+1)*N].astype(np.int64) if j % 4 != 3 else rng.integers(0, 4096, size=N) for j in range(K)]
sched = np.asarray(bm.round_robin_schedule([N] * K), dtype=np.int32)
cont, _ = bm.mux_with_flush(msgs, coders, sched, F)
out = bm.demux_decode(cont, coders, sched)
print("ok", sum(len(o) for o in out))
