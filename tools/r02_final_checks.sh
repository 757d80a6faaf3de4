# Round-2 final checks: full -m gpu suite (incl. 8 GiB), sanitizers.
mkdir -p gpurun_out
python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/r02f_gputest.txt
bash tools/sanitize.sh > /dev/null 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_variants.py tests/test_gpu_byte8.py -q -x > gpurun_out/memcheck_new.log 2>&1
cat gpurun_out/r02f_gputest.txt
tail -n 3 gpurun_out/memcheck.log gpurun_out/racecheck.log gpurun_out/synccheck.log gpurun_out/memcheck_new.log
