mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/r2bn_tests.log 2>&1; echo "sharded tests rc=$?"; tail -3 gpurun_out/r2bn_tests.log
timeout 600 python bench.py --sharded --steps 30 --warmup 3 --no-fasterpam --no-dissimilarity --no-clara > gpurun_out/r2bn_bench_graph.log 2>&1; echo "bench graph rc=$?"; tail -1 gpurun_out/r2bn_bench_graph.log | cut -c1-600
timeout 600 python bench.py --sharded --no-graph --steps 30 --warmup 3 --no-fasterpam --no-dissimilarity --no-clara --no-e2e --no-cpu-baseline > gpurun_out/r2bn_bench_direct.log 2>&1; echo "bench direct rc=$?"; tail -1 gpurun_out/r2bn_bench_direct.log | cut -c1-400
