mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2bs_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2bs_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2bs_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2bs_smoke.log
