mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "part_counts or random_int or fastpam2_int or per_candidate" > gpurun_out/r2r_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2r_pytest.log
for qu in 8 4 16 8 16; do KM_COMB_QU=$qu python bench.py --no-e2e --no-fasterpam --no-dissimilarity --no-cpu-baseline --no-clara --steps 40 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C4 qu=$qu', round(d['ms_per_step']*1e3,1), round(d['roofline']['kernel_ms']*1e3,1), round(d['ms_per_step']*1e3-d['roofline']['kernel_ms']*1e3,1))" >> gpurun_out/r2r_qu.log; done
for qu in 8 16; do KM_COMB_QU=$qu python bench.py --config 3 --no-e2e --no-fasterpam --no-dissimilarity --no-cpu-baseline --no-clara --steps 40 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C3 qu=$qu', round(d['ms_per_step']*1e3,1), round(d['roofline']['kernel_ms']*1e3,1), round(d['ms_per_step']*1e3-d['roofline']['kernel_ms']*1e3,1))" >> gpurun_out/r2r_qu.log; done
python bench.py --config 1 --warmup 2 --steps 1 --no-e2e --no-fasterpam --no-dissimilarity --no-cpu-baseline --no-clara 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C1', d['ms_per_step'])" >> gpurun_out/r2r_qu.log
