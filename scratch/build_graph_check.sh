#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_clara.py tests/test_gpu_fullsize.py tests/test_gpu_init.py -x -q 2>&1 | tail -1
for g in 1 0; do
KM_BUILD_GRAPH=$g timeout 200 python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('graph=$g C4 build ms', d['init'])"
KM_BUILD_GRAPH=$g timeout 300 python scratch/clara_perf.py 2>&1 | tail -3
done
