#!/bin/bash
cd $GRAFT_REPO_ROOT
F="python bench.py --config 5 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity"
$F > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_swap_stream_seg2 -s 4 -c 1 -o gpurun_out/r1m_k1_seg2_c5 $F > gpurun_out/ncu_c5.log 2>&1
echo "c5 rc=$?"
F3="python bench.py --config 3 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity"
$F3 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_swap_stream_seg2 -s 4 -c 1 -o gpurun_out/r1m_k1_seg2_c3 $F3 > gpurun_out/ncu_c3.log 2>&1
echo "c3 rc=$?"
