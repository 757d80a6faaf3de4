# ncu --set full capture of the encode + decode kernels of one bench step
tag=${1:-cap}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"encode_warp|decode_warp" -c 2 -f -o gpurun_out/$tag python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/$tag.log 2>&1
tail -2 gpurun_out/$tag.log
