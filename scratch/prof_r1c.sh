#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1c.csv $B > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
F="python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline"
$F > gpurun_out/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_swap_stream_seg -s 4 -c 1 -o gpurun_out/r1c_k1_seg_c4 $F > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
G="python bench.py --config 5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$G > gpurun_out/plain_full5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_swap_stream_seg -s 4 -c 1 -o gpurun_out/r1c_k1_seg_c5 $G > gpurun_out/ncu_full5.log 2>&1
echo "full5 rc=$?"
