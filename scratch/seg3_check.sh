#!/bin/bash
cd $GRAFT_REPO_ROOT
KM_STREAM=seg3 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -1
for v in seg3 seg2; do for cfg in 4 5 3; do
KM_STREAM=$v timeout 200 python bench.py --config $cfg --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v cfg $cfg', round(d['ms_per_step'],4), round(r['kernel_ms'],4), round(r['frac_of_read_only_peak'],4), flush=True)"
done; done
