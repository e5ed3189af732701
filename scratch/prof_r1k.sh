#!/bin/bash
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity"
$B > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1k.csv $B > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
F="python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity"
$F > gpurun_out/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_swap_stream_seg2 -s 4 -c 1 -o gpurun_out/r1k_k1_seg2_c4 $F > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_fp1_post -s 4 -c 1 -o gpurun_out/r1k_post_c4 $F > gpurun_out/ncu_post.log 2>&1
echo "post rc=$?"
