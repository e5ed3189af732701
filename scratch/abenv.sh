#!/bin/bash
# usage: scratch/abenv.sh "<env1>|<env2>|..." <config> <reps> [extra bench args]
# each env is a space-separated list of VAR=value (or "-" for none); prints
# step ms, stream kernel ms and roofline fraction per run (measurement aid)
mkdir -p gpurun_out
IFS='|' read -ra ENVS <<< "$1"
for r in $(seq 1 $3); do for e in "${ENVS[@]}"; do
  ee="$e"; [ "$ee" = "-" ] && ee=""
  env $ee timeout 300 python bench.py --config $2 --steps 60 --warmup 3 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity --no-clara ${@:4} > gpurun_out/abenv.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/abenv.log').read().splitlines()[-1]);print('C$2', '[$e]', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['ms_per_step']-d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -5 gpurun_out/abenv.log
done; done
