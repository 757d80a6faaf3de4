# Round-2 late evidence after the direct-store encoder: sanitizers over the
# GPU suite, config 3 (8 GiB), config 4 sweep, config 5 stress, byte8 probe.
mkdir -p gpurun_out
bash tools/sanitize.sh > /dev/null 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu --no-plugin --no-e2e --stress > gpurun_out/r02z_stress.json 2> gpurun_out/r02z_stress.err
python bench.py --steps 5 --warmup 3 --no-cpu --no-plugin --global-mib 8192 > gpurun_out/r02z_cfg3.json 2> gpurun_out/r02z_cfg3.err
python bench.py --steps 10 --warmup 3 --no-cpu --no-plugin --no-e2e --sweep > gpurun_out/r02z_sweep.json 2> gpurun_out/r02z_sweep.err
python tools/byte8_chunked_probe.py > gpurun_out/r02z_byte8.txt 2>&1
tail -n 3 gpurun_out/memcheck.log gpurun_out/racecheck.log gpurun_out/synccheck.log
tail -n 2 gpurun_out/r02z_*.err
