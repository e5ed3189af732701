mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_clara.py tests/test_gpu_clara_points.py tests/test_gpu_parity.py -x -q > gpurun_out/r2bg_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2bg_tests.log
timeout 300 python scratch/clara_perf.py 4; timeout 300 python scratch/clara_perf.py 3
timeout 300 python scratch/clara_repro.py 2 5 2>&1 | tail -5
timeout 300 python scratch/clara_repro.py 1 1 2>&1 | tail -3
