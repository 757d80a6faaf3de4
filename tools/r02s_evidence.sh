mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02s_smi.txt
python bench.py --steps 20 --warmup 3 > gpurun_out/r02s_bench.json 2> gpurun_out/r02s_bench.err
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r02s_ref.json 2> gpurun_out/r02s_ref.err
python bench.py --steps 10 --warmup 3 --no-cpu --no-plugin --no-e2e --stress > gpurun_out/r02s_stress.json 2> gpurun_out/r02s_stress.err
python bench.py --steps 5 --warmup 3 --no-cpu --no-plugin --global-mib 8192 > gpurun_out/r02s_cfg3.json 2> gpurun_out/r02s_cfg3.err
python bench.py --steps 10 --warmup 3 --no-cpu --no-plugin --no-e2e --sweep > gpurun_out/r02s_sweep.json 2> gpurun_out/r02s_sweep.err
tail -2 gpurun_out/r02s_*.err
