# ncu evidence for one bench step: launch list (durations) + one --set full
# capture of every kernel of the step. Summarise here afterwards with
#   python profiles/summarize.py gpurun_out/<tag>.ncu-rep gpurun_out/<tag>_launches.csv <tag>
tag=${1:-prof}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/${tag}_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"histogram|build_table|encode_warp|compact|decode_warp|chunk_offsets" -c 8 -f \
    -o gpurun_out/${tag} python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/${tag}.log 2>&1
ls -la gpurun_out | grep $tag
