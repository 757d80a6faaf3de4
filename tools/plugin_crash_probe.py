# Plugin threads (8 / 16 / 32) through Backend("b200") under faulthandler:
# checks that the process exits cleanly after many per-thread contexts
# (ilans_process_exiting hook). 8 of 8 runs clean at the final tree.
import faulthandler, sys, threading
faulthandler.enable()
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_1402_3392_b200.rans import SymbolTable, WORD16
from paper_1402_3392_b200.interleave import encode_interleaved, decode_interleaved
from paper_1402_3392_b200.synth import synth_host
C = 65536
msg = synth_host(C * 256, 1.1, 7)
counts = np.bincount(msg, minlength=256)
t = SymbolTable.from_counts(counts[: int(np.nonzero(counts)[0][-1]) + 1].tolist(), 12)
def work(lo, hi):
    for k in range(lo, hi):
        c = encode_interleaved(msg[k*C:(k+1)*C], t, 32, WORD16, backend="b200")
        decode_interleaved(c, backend="b200")
for T in (8, 16, 32):
    ths = [threading.Thread(target=work, args=(i*256//T, (i+1)*256//T)) for i in range(T)]
    [x.start() for x in ths]; [x.join() for x in ths]
print("done")
