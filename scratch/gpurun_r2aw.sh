mkdir -p gpurun_out
for c in 1 0 1; do KM_DIST_CENTER=$c timeout 300 python scratch/dist_c4.py 2>&1 | grep -v Warn; done > gpurun_out/r2aw_dist.log
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_clara_points.py -x -q > gpurun_out/r2aw_tests.log 2>&1; echo "tests rc=$?"
