#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -1
for i in 1 2 3; do timeout 200 python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4 build', d['init'])"; done
timeout 200 python bench.py --config 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2 build', d['init'])"
