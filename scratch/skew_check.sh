#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_skew15.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/pytest_skew15.log
for sk in 0 15; do for cfg in 4 5; do
KM_PART_SKEW=$sk python bench.py --config $cfg --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-dissimilarity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; f=d['fasterpam']; print('cfg $cfg skew=$sk', round(d['ms_per_step'],4), round(r['kernel_ms'],4), 'build', round(d['init']['ms'],2), 'fp3', round(f['s_to_converge'],4), 'inc', round(f['fastpam1_incremental_s_to_converge'],4), flush=True)"
done; done
