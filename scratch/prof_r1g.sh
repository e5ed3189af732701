#!/bin/bash
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity"
$B > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1g.csv $B > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
$B > gpurun_out/plain_post.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fp1_post -s 5 -c 1 -o gpurun_out/r1g_post_c4 $B > gpurun_out/ncu_post.log 2>&1
echo "post rc=$?"
F="python scratch/fp3_perf.py 4 build"
$F > gpurun_out/plain_fp3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fp3_window -s 2 -c 1 -o gpurun_out/r1g_fp3_c4 $F > gpurun_out/ncu_fp3.log 2>&1
echo "fp3 rc=$?"
