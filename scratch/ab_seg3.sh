#!/bin/bash
cd $GRAFT_REPO_ROOT
for i in 1 2 3; do for v in seg2 seg3; do
KM_STREAM=$v timeout 200 python bench.py --config 4 --steps 60 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', round(d['ms_per_step'],4), round(r['kernel_ms'],4), flush=True)"
done; done
for v in seg2 seg3; do KM_STREAM=$v timeout 200 python bench.py --config 5 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('C5 $v', round(d['ms_per_step'],4), round(r['kernel_ms'],4), flush=True)"; done
