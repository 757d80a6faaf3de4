# One evidence pass at the current tree: sanitizers over the GPU suite,
# config 3 (8 GiB), config 4 sweep, config 5 stress, byte8 probe, the bench
# line, the reference arm and the ncu capture of one step.
# usage: bash tools/evidence.sh <tag>
tag=${1:-ev}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; tail -n 1 gpurun_out/${tag}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" && echo smoke ok
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2>&1
bash tools/sanitize.sh > /dev/null 2>&1
for t in memcheck racecheck synccheck; do cp gpurun_out/$t.log gpurun_out/${tag}_$t.log; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-plugin --no-e2e --stress > gpurun_out/${tag}_stress.json 2> gpurun_out/${tag}_stress.err
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-plugin --global-mib 8192 > gpurun_out/${tag}_cfg3.json 2> gpurun_out/${tag}_cfg3.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-plugin --no-e2e --sweep > gpurun_out/${tag}_sweep.json 2> gpurun_out/${tag}_sweep.err
timeout 300 python tools/byte8_chunked_probe.py > gpurun_out/${tag}_byte8.txt 2>&1
bash tools/profile_round.sh ${tag} > /dev/null 2>&1
tail -n 2 gpurun_out/${tag}_memcheck.log gpurun_out/${tag}_racecheck.log gpurun_out/${tag}_synccheck.log
tail -n 2 gpurun_out/${tag}_*.err
ls -la gpurun_out | grep ${tag}
