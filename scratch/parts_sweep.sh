#!/bin/bash
# stream kernel time vs row parts P (C4 and C3), FastPAM1 bench lines
cd $GRAFT_REPO_ROOT
for cfg in 4 3; do
for P in 0 7 15 16 23 24 31 39 47; do
  if [ $P = 0 ]; then unset KM_PARTS; else export KM_PARTS=$P; fi
  python bench.py --config $cfg --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $cfg P=$P', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
done; done
