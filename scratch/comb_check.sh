#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fasterpam.py -x -q 2>&1 | tail -1
for cfg in 4 3 5; do
KM_STEP_PROF=1 python bench.py --config $cfg --steps 60 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>&1 | grep -E "step phases" | tail -1
python bench.py --config $cfg --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg $cfg', round(d['ms_per_step'],4), round(r['kernel_ms'],4), d['value'])"
done
