import sys, time, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle/_ref')
import paper_1402_3392_b200 as ilb
from paper_1402_3392_b200.synth import synth_host
import ilans as ref
msg = synth_host(1 << 20, 1.1, seed=1)
counts = np.bincount(msg, minlength=256)
for N in [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else "1,2,4,8,16,32".split(","))]:
    t = ilb.SymbolTable.from_counts(counts.tolist(), 14)
    rt = ref.rans.SymbolTable.from_counts(counts.tolist(), 14)
    c = ilb.encode_interleaved(msg, t, N); ilb.decode_interleaved(c)
    rc = ref.interleave.encode_interleaved(msg, rt, N, ref.rans.WORD16, backend="ext")
    def tm(f, r=5):
        f(); t0 = time.perf_counter()
        for _ in range(r): f()
        return (time.perf_counter() - t0) / r
    e_g = tm(lambda: ilb.encode_interleaved(msg, t, N)); d_g = tm(lambda: ilb.decode_interleaved(c))
    e_r = tm(lambda: ref.interleave.encode_interleaved(msg, rt, N, ref.rans.WORD16, backend="ext"), 2)
    d_r = tm(lambda: ref.interleave.decode_interleaved(rc, backend="ext"), 2)
    mb = len(msg) / 1e6
    print(f"N={N}: b200 encode {mb/e_g:.0f} MB/s decode {mb/d_g:.0f} MB/s | reference encode {mb/e_r:.0f} decode {mb/d_r:.0f} MB/s")
