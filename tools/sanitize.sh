# compute-sanitizer over the GPU parity suite: memcheck (all -m gpu tests),
# racecheck and synccheck (the warp-synchronous coders); logs in gpurun_out/
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests -m gpu -x -q > gpurun_out/memcheck.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "fixtures or fast or adler" > gpurun_out/racecheck.log 2>&1
timeout 600 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_parity.py -x -q -k "fixtures or fast" > gpurun_out/synccheck.log 2>&1
tail -n 3 gpurun_out/memcheck.log gpurun_out/racecheck.log gpurun_out/synccheck.log
