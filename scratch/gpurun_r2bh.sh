mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_clara.py tests/test_gpu_clara_points.py -x -q > gpurun_out/r2bh_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2bh_tests.log
timeout 300 python scratch/clara_perf.py 4; timeout 300 python scratch/clara_perf.py 3
timeout 300 python scratch/clara_repro.py 2 5 2>&1 | tail -5
timeout 300 python scratch/clara_repro.py 1 1 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2bh_clara_launches.csv python scratch/clara_repro.py 1 5 > gpurun_out/r2bh_ncu.log 2>&1; echo "ncu clara rc=$?"
