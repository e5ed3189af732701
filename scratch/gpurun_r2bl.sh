mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2bl_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2bl_gputests.log
timeout 600 python scratch/clara_perf.py 5
timeout 600 python scratch/clara_big.py
