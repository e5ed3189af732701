#!/bin/bash
cd $GRAFT_REPO_ROOT
run() { # cfg P
  if [ $2 = 0 ]; then unset KM_PARTS; else export KM_PARTS=$2; fi
  timeout 200 python bench.py --config $1 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg $1 P=$2', round(d['ms_per_step'],4), round(r['kernel_ms'],4), flush=True)"
}
for P in 0 30 40 46; do run 3 $P; done
for P in 0 30 40; do run 4 $P; done
