#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q -k "fp2 or fastpam2 or shard or parity" 2>&1 | tail -15
for cfg in 5 3; do
timeout 240 python bench.py --config $cfg --variant fastpam2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg $cfg fp2', round(d['ms_per_step'],4), round(r['kernel_ms'],4), d['value'], d.get('timed_swaps'), d['td_after'])"
done
