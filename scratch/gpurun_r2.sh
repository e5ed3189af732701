mkdir -p gpurun_out
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-fasterpam --no-dissimilarity --no-cpu-baseline --no-clara"
$CMD > gpurun_out/r2ab_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2ab_launches.csv $CMD > gpurun_out/r2ab_ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_swap_stream_seg2|k_fp1_post|k_swap_combine" -s 12 -c 3 -o gpurun_out/r2ab_prof $CMD > gpurun_out/r2ab_ncu2.log 2>&1
echo "rc=$?"
