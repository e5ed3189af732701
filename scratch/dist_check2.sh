#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -1
for st in 1 2; do KM_DIST_STAGES=$st timeout 300 python scratch/dist_perf.py 2>&1 | grep -E "C3|C4" | sed "s/^/stages=$st /"; done
