#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1000 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests.log
F="python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity"
$F > gpurun_out/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_swap_stream_seg3 -s 4 -c 1 -o gpurun_out/r1l_k1_seg3_c4 $F > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 400 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?
