#!/bin/bash
cd $GRAFT_REPO_ROOT
for b in 1 2 4; do for cfg in 3 4; do
KM_POST_BPS=$b KM_STEP_PROF=1 timeout 200 python bench.py --config $cfg --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>&1 | grep "step phases" | tail -1 | sed "s/^/bps=$b cfg=$cfg /"
done; done
