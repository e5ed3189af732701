mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fastpam2_queued.py tests/test_gpu_parity.py tests/test_gpu_goldens.py tests/test_gpu_sharded.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r2bt_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2bt_tests.log
KM_STEP_PROF=1 timeout 300 python scratch/fp2prof.py 5 10 2>&1 | grep phases | tail -1
for c in 5 3; do timeout 900 python bench.py --config $c --variant fastpam2 --steps 10 --warmup 3 --no-e2e --no-fasterpam --no-dissimilarity --no-clara --no-cpu-baseline > gpurun_out/r2bt_bench_c$c.log 2>&1; echo "bench C$c rc=$?"; tail -1 gpurun_out/r2bt_bench_c$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['ms_per_step'])"; done
