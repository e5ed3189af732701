#!/bin/bash
cd $GRAFT_REPO_ROOT
for cfg in "4 build" "3 random"; do
for WL in "7168 4096" "7168 2048" "7168 1024" "7168 512" "3584 1024" "14336 2048"; do
  set -- $WL
  KM_FASTER_COOP_W=$1 KM_FASTER_L=$2 timeout 300 python scratch/fp3_perf.py $cfg 2>&1 | grep "fasterpam:" | tail -1 | sed "s/^/W=$1 L=$2 /"
done; done
