mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_goldens.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "not c4_build and not c4_fastpam1_full" > gpurun_out/r2p_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2p_pytest.log
timeout 400 python scratch/stress.py 7 300 > gpurun_out/r2p_stress.log 2>&1; echo rc=$? >> gpurun_out/r2p_stress.log
