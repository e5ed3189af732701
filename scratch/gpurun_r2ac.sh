# round-2 final capture: default bench (C4), launch list, ncu --set full of one
# iteration's stream + post kernels (measurement aid)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2ac_bench.log 2>&1; echo "bench rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-fasterpam --no-dissimilarity --no-cpu-baseline --no-clara"
timeout 600 $CMD > gpurun_out/r2ac_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2ac_launches.csv $CMD > gpurun_out/r2ac_ncu1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_swap_stream_seg2|k_fp1_post" -s 12 -c 2 -o gpurun_out/r2ac_prof $CMD > gpurun_out/r2ac_ncu2.log 2>&1
echo "rc=$?"
