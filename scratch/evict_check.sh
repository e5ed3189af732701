#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -1
for cfg in 4 3 5; do
KM_STEP_PROF=1 timeout 200 python bench.py --config $cfg --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>&1 | grep "step phases" | tail -1 | sed "s/^/cfg=$cfg /"
timeout 200 python bench.py --config $cfg --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg $cfg', round(d['ms_per_step'],4), round(r['kernel_ms'],4))"
done
