#!/bin/bash
# round-1 re-entry check: build, gpu tests, smoke, default bench
set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench_c4.log | cut -c1-600
