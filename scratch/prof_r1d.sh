#!/bin/bash
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-fasterpam"
for ch in 0 256 512 1024; do for c in 4 3; do
  if [ $ch = 0 ]; then unset KM_SORT_CHUNKS; else export KM_SORT_CHUNKS=$ch; fi
  python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $c chunks $ch', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],4), flush=True)"
done; done
unset KM_SORT_CHUNKS
$B > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1d.csv $B > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
F="python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --no-fasterpam"
$F > gpurun_out/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_swap_stream_seg2 -s 4 -c 1 -o gpurun_out/r1d_k1_seg2_c4 $F > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
