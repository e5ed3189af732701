#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1000 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in 5 3; do
timeout 240 python bench.py --config $cfg --variant fastpam2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg $cfg fp2', round(d['ms_per_step'],4), round(r['kernel_ms'],4), d['value'], d.get('timed_swaps'), d['td_after'])"
done
timeout 300 python bench.py --sharded --steps 30 --warmup 3 --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sharded x1', round(d['ms_per_step'],4), d['init'])"
KM_FASTER_PROF=1 timeout 300 python scratch/fp3_perf.py 4 build 2>&1 | grep "fasterpam:" | tail -1
