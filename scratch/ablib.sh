#!/bin/bash
# usage: scratch/ablib.sh "<configs>" <reps>: the saved baseline library
# (scratch/old/libkmedoids.so) against the current build, alternating,
# step ms / stream ms / overhead per run (measurement aid)
mkdir -p gpurun_out
cp paper_2008_05171_b200/libkmedoids.so /tmp/km_new.so
for r in $(seq 1 $2); do for c in $1; do for lib in old new; do
  if [ $lib = old ]; then cp scratch/old/libkmedoids.so paper_2008_05171_b200/libkmedoids.so; else cp /tmp/km_new.so paper_2008_05171_b200/libkmedoids.so; fi
  timeout 300 python bench.py --config $c --steps 60 --warmup 3 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity --no-clara > gpurun_out/ablib.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ablib.log').read().splitlines()[-1]);print('C$c', '$lib', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['ms_per_step']-d['roofline']['kernel_ms'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/ablib.log
done; done; done
cp /tmp/km_new.so paper_2008_05171_b200/libkmedoids.so
