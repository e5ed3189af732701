# final round-2 launch list (default bench minus FastCLARA's host threads, which ncu cannot follow) + ncu capture
mkdir -p gpurun_out
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-fasterpam --no-dissimilarity --no-cpu-baseline --no-clara"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2bb_launches.csv python bench.py --no-clara > gpurun_out/r2bb_ncu1.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_swap_stream_seg2|k_fp1_post" -s 12 -c 2 -o gpurun_out/r2bb_prof $CMD > gpurun_out/r2bb_ncu2.log 2>&1; echo "full rc=$?"
