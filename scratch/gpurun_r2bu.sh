# final HEAD validation: every GPU test, smoke, default bench
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2bu_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/r2bu_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2bu_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2bu_smoke.log
timeout 900 python bench.py > gpurun_out/r2bu_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2bu_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['seconds'], d['clocks'])"
