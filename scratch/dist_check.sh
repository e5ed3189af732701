#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -2
timeout 300 python scratch/dist_perf.py
python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-fasterpam 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['dissimilarity'])"
