#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -3
timeout 300 python scratch/dist_perf.py 2>&1 | grep -E "C5|C1"
KM_DIST_L1=f32 timeout 300 python scratch/dist_perf.py 2>&1 | grep -E "C5"
