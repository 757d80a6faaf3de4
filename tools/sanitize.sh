# compute-sanitizer over the GPU parity suite: memcheck (the -m gpu tests but
# the full-size / multi-process / subprocess ones), racecheck and synccheck
# (the warp-synchronous coders, word16 and byte8); logs in gpurun_out/
sel='not fullsize and not own_suite and not gpu_dist'
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests -m gpu -x -q \
    --ignore tests/test_gpu_fullsize.py --ignore tests/test_gpu_reference_own_suite.py \
    --ignore tests/test_gpu_dist.py > gpurun_out/memcheck.log 2>&1
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py \
    tests/test_gpu_byte8.py -x -q -k "fixtures or fast or adler or slot or chunk" > gpurun_out/racecheck.log 2>&1
timeout 600 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_byte8.py \
    -x -q -k "fixtures or fast or slot" > gpurun_out/synccheck.log 2>&1
tail -n 3 gpurun_out/memcheck.log gpurun_out/racecheck.log gpurun_out/synccheck.log
