# Round-end evidence in one GPU session: tests, smoke, bench (+ reference
# arm), ncu of one step, compute-sanitizer on the newest kernels, probes.
# usage: bash tools/final_check.sh <tag>
set -x
tag=${1:-final}
bash tools/gpu_check.sh ${tag}
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_mux.py tests/test_gpu_byte8.py -q > gpurun_out/${tag}_memcheck_mux.log 2>&1
tail -n 3 gpurun_out/${tag}_memcheck_mux.log
timeout 600 python tools/single_stream_probe.py 1,2,3,4,5,7,8,12,16,31,32,33,64,128,256,1024,4096 > gpurun_out/${tag}_single_stream.log 2>&1
timeout 600 python tools/mux_probe.py 16 65536 4096 > gpurun_out/${tag}_mux.log 2>&1
timeout 600 python tools/mux_probe.py 256 8192 0 >> gpurun_out/${tag}_mux.log 2>&1
timeout 600 python tools/byte8_chunked_probe.py 256 > gpurun_out/${tag}_byte8.log 2>&1
python - <<'PY' > gpurun_out/${tag}_readme.log 2>&1
import numpy as np
import paper_1402_3392_b200 as ilans
msg = np.random.default_rng(0).integers(0, 16, 1 << 20).astype(np.uint8)
table = ilans.SymbolTable.from_counts(np.bincount(msg).tolist(), 12)
c = ilans.encode_interleaved(msg, table, 32)
assert (ilans.decode_interleaved(ilans.Container.from_bytes(c.to_bytes())) == msg).all()
from paper_1402_3392_b200.chunked import encode_chunked, decode_chunked
cc = encode_chunked(msg, None, 32, 65536, 12)
assert (decode_chunked(cc) == msg).all()
from paper_1402_3392_b200.rans import BYTE8
cb = encode_chunked(msg, None, 2, 65536, 12, variant=BYTE8)
assert (decode_chunked(cb) == msg).all()
from paper_1402_3392_b200 import mux
coders = [mux.RansStreamCodec(table), mux.RawStreamCodec(12)]
streams = [msg[:1000].tolist(), list(range(500))]
box, budget = mux.mux_with_flush(streams, coders, flush_interval=64)
assert mux.demux_decode(box.to_bytes(), coders) == streams
print("README snippet ok", budget)
PY
cat gpurun_out/${tag}_readme.log
ls -la gpurun_out | grep ${tag}
