#!/bin/bash
cd $GRAFT_REPO_ROOT
for c in par par4; do KM_COMBINE=$c timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -1; done
for cfg in 4 3; do for c in seq par par4; do
KM_COMBINE=$c KM_STEP_PROF=1 python bench.py --config $cfg --steps 60 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>&1 | grep -E "step phases" | tail -1 | sed "s/^/cfg $cfg $c /"
done; done
