#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_init.py tests/test_gpu_clara.py -x -q 2>&1 | tail -1
timeout 600 python scratch/init_perf.py 4 2>&1 | tail -8
timeout 600 python scratch/init_perf.py 5 2>&1 | tail -8
