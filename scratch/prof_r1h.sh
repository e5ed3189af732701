#!/bin/bash
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity"
$B > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1h.csv $B > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
F="python scratch/inc_perf.py 4 build"
$F > gpurun_out/plain_inc.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fp3_window -s 1 -c 1 -o gpurun_out/r1h_inc_c4 $F > gpurun_out/ncu_inc.log 2>&1
echo "inc rc=$?"
