#!/bin/bash
cd $GRAFT_REPO_ROOT
python scratch/dist_once.py 4 > gpurun_out/plain_dist.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_dist_l2_ws -s 1 -c 1 -o gpurun_out/r1j_dist_ws_c4 python scratch/dist_once.py 4 > gpurun_out/ncu_dist_j.log 2>&1
echo "l2 rc=$?"
python scratch/l1_once.py 100000 > gpurun_out/plain_l1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_dist_l1_u16x2 -c 1 -o gpurun_out/r1j_dist_l1_c5 python scratch/l1_once.py 100000 > gpurun_out/ncu_l1_j.log 2>&1
echo "l1 rc=$?"
