mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/r2v_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2v_pytest.log
for c in 4 3 4; do python bench.py --config $c --no-e2e --no-fasterpam --no-dissimilarity --no-cpu-baseline --no-clara --steps 40 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('C$c', round(d['ms_per_step']*1e3,1), round(r['kernel_ms']*1e3,1), round(r['frac'],4), round(r['frac_of_read_only_peak'],4))" >> gpurun_out/r2v_bench.log; done
python bench.py --config 5 --no-e2e --no-fasterpam --no-dissimilarity --no-cpu-baseline --no-clara --steps 15 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('C5', round(d['ms_per_step']*1e3,1), round(r['kernel_ms']*1e3,1), round(r['frac'],4), round(r['frac_of_read_only_peak'],4))" >> gpurun_out/r2v_bench.log
