#!/bin/bash
cd $GRAFT_REPO_ROOT
for v in seg2 seg6 seg5; do for cfg in 4 3 5; do
KM_STREAM=$v timeout 200 python bench.py --config $cfg --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v cfg $cfg', round(d['ms_per_step'],4), round(r['kernel_ms'],4), flush=True)"
done; done
