#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_fastpam1_inc.py tests/test_gpu_fasterpam.py -x -q 2>&1 | tail -1
KM_FASTER_PROF=1 timeout 300 python scratch/inc_perf.py 4 build 2>&1 | tail -3
timeout 300 python scratch/inc_perf.py 3 random 2>&1 | tail -2
timeout 300 python scratch/inc_perf.py 5 build 2>&1 | tail -2
