#!/bin/bash
cd $GRAFT_REPO_ROOT
for t in 128 64 32; do for cfg in 4 3; do
KM_COMB_TPB=$t KM_STEP_PROF=1 timeout 200 python bench.py --config $cfg --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>&1 | grep "step phases" | tail -1 | sed "s/^/tpb=$t cfg=$cfg /"
done; done
KM_COMB_TPB=64 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
