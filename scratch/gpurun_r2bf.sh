# single-thread FastCLARA driver: clara tests, clara timing, ncu launch list of the clara repro
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_clara.py tests/test_gpu_clara_points.py -x -q > gpurun_out/r2bf_tests.log 2>&1; echo "clara tests rc=$?"; tail -3 gpurun_out/r2bf_tests.log
timeout 300 python scratch/clara_perf.py > gpurun_out/r2bf_perf.log 2>&1; echo "perf rc=$?"; tail -20 gpurun_out/r2bf_perf.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2bf_clara_launches.csv python scratch/clara_repro.py 1 5 > gpurun_out/r2bf_ncu.log 2>&1; echo "ncu clara rc=$?"; tail -3 gpurun_out/r2bf_ncu.log
