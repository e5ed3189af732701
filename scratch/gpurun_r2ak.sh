mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2ak_gputest.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py > gpurun_out/r2ak_bench.log 2>&1; echo "bench rc=$?"
KM_GRAPH_EVENTS=1 timeout 900 python bench.py --no-e2e --no-fasterpam --no-dissimilarity --no-clara --no-cpu-baseline > gpurun_out/r2ak_bench_ev1.log 2>&1; echo "bench rc=$?"
