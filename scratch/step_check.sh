#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_step.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/pytest_step.log
for cfg in 4 3; do
KM_STEP_PROF=1 python bench.py --config $cfg --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>&1 | grep -E "phases" | tail -2
python bench.py --config $cfg --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg $cfg', round(d['ms_per_step'],4), round(r['kernel_ms'],4), d['value'])"
done
