mkdir -p gpurun_out
python -m pytest tests/test_gpu_dist.py -x -q -p no:cacheprovider > gpurun_out/r2o_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2o_pytest.log
python scratch/dist_accuracy.py > gpurun_out/r2o_acc.log 2>&1
python bench.py --no-e2e --no-fasterpam --no-cpu-baseline --no-clara --steps 10 --warmup 3 > gpurun_out/r2o_bench.log 2>&1
