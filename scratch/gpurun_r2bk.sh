mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_build_small.py tests/test_gpu_parity.py tests/test_gpu_clara.py tests/test_gpu_clara_points.py tests/test_gpu_goldens.py -x -q > gpurun_out/r2bk_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r2bk_tests.log
timeout 300 python scratch/clara_perf.py 4; timeout 300 python scratch/clara_perf.py 3
timeout 300 python scratch/clara_repro.py 2 5 2>&1 | tail -5
timeout 300 python scratch/clara_repro.py 1 1 2>&1 | tail -3
KM_BUILD_SMALL=0 timeout 300 python scratch/clara_repro.py 1 1 2>&1 | tail -3
