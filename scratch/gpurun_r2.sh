mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_goldens.py -x -q -p no:cacheprovider -k "symmetric or fastpam2 or c5" > gpurun_out/r2s_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2s_pytest.log
python bench.py --config 5 --variant fastpam2 --warmup 3 --steps 10 --no-e2e --no-fasterpam --no-dissimilarity --no-cpu-baseline --no-clara > gpurun_out/r2s_c5fp2.log 2>&1
python bench.py --config 3 --variant fastpam2 --warmup 3 --steps 10 --no-e2e --no-fasterpam --no-dissimilarity --no-cpu-baseline --no-clara > gpurun_out/r2s_c3fp2.log 2>&1
