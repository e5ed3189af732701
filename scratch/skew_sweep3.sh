#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tilt" 2>&1 | tail -1
KM_PART_SKEW=32 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -1
run() { # cfg P skew
  export KM_PART_SKEW=$3; if [ $2 = 0 ]; then unset KM_PARTS; else export KM_PARTS=$2; fi
  timeout 200 python bench.py --config $1 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg $1 P=$2 skew=$3', round(d['ms_per_step'],4), round(r['kernel_ms'],4), round(r['frac_of_read_only_peak'],4), flush=True)"
}
for sk in 15 16 24 32 48; do run 4 0 $sk; done
for sk in 15 24 32 48; do run 3 0 $sk; done
for sk in 15 32; do run 5 0 $sk; done
for sk in 32 48; do run 4 63 $sk; run 3 100 $sk; done
