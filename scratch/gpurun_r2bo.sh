# end-of-session round-2 measurements: default bench x2, sharded bench (graph), launch list of the whole default bench, ncu capture
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2bo_bench1.log 2>&1; echo "bench1 rc=$?"
timeout 900 python bench.py > gpurun_out/r2bo_bench2.log 2>&1; echo "bench2 rc=$?"
timeout 600 python bench.py --sharded --steps 30 --warmup 3 --no-fasterpam --no-dissimilarity --no-clara > gpurun_out/r2bo_sharded.log 2>&1; echo "sharded rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2bo_launches.csv python bench.py > gpurun_out/r2bo_ncu1.log 2>&1; echo "launches rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-fasterpam --no-dissimilarity --no-cpu-baseline --no-clara"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_swap_stream_seg2|k_fp1_post" -s 12 -c 2 -o gpurun_out/r2bo_prof $CMD > gpurun_out/r2bo_ncu2.log 2>&1; echo "full rc=$?"
