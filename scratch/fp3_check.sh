#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_fasterpam.py tests/test_gpu_fastpam1_inc.py -x -q 2>&1 | tail -1
for c in "4 build" "3 random"; do KM_FASTER_PROF=1 timeout 300 python scratch/fp3_perf.py $c 2>&1 | grep -E "fasterpam:|pass: swaps [1-9][0-9]" | tail -2; done
timeout 300 python scratch/inc_perf.py 4 build 2>&1 | tail -2
