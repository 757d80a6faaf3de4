mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x --deselect tests/test_gpu_fullsize.py::test_config3_8gib_every_chunk_bit_exact 2>&1 | tail -2 > gpurun_out/r02w_gputest.txt
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_byte8.py -x -q -k "fixtures or fast or adler or slot or chunk" > gpurun_out/racecheck.log 2>&1
cat gpurun_out/r02w_gputest.txt; tail -3 gpurun_out/racecheck.log
