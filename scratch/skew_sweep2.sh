#!/bin/bash
cd $GRAFT_REPO_ROOT
run() { # cfg P skew
  export KM_PART_SKEW=$3; if [ $2 = 0 ]; then unset KM_PARTS; else export KM_PARTS=$2; fi
  python bench.py --config $1 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg $1 P=$2 skew=$3', round(d['ms_per_step'],4), round(r['kernel_ms'],4), round(r['frac'],4), round(r['frac_of_read_only_peak'],4), d['clocks']['sm_mhz'], round(d['init']['ms'],2), flush=True)"
}
for P in 0 39 63 80; do run 4 $P 15; done
run 4 0 0
for P in 0 100 160; do run 3 $P 15; done
for P in 0 24 40; do run 5 $P 15; done
for P in 0 8 12; do run 2 $P 15; done
