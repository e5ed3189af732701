# re-entry check: gpu tests, smoke, default bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2bc_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2bc_gputests.log 2>&1; echo "gpu tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2bc_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r2bc_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r2bc_bench.log
