mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_goldens.py -x -q -p no:cacheprovider -k "chunk_loop or c3_fasterpam" > gpurun_out/r2t_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2t_pytest.log
