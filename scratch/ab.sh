#!/bin/bash
# usage: scratch/ab.sh "<kinds>" <config> <reps>
for r in $(seq 1 $3); do for k in $1; do KM_STREAM=$k timeout 300 python bench.py --config $2 --steps 60 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab.log 2>&1; python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().splitlines()[-1]);print('C$2', '$k', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done; done
