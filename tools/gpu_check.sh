# One full GPU pass: parity tests, smoke, the bench line and the reference
# arm, then the ncu evidence for one step (tools/profile_round.sh).
# usage: bash tools/gpu_check.sh [tag]
set -x
tag=${1:-check}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; tail -n 3 gpurun_out/${tag}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2>&1
bash tools/profile_round.sh ${tag}
ls -la gpurun_out | grep ${tag}
