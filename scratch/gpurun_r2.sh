mkdir -p gpurun_out
for rep in 1 2; do for v in 1 2; do KM_STREAM_STAGED=$v python bench.py --config 5 --no-e2e --no-fasterpam --no-dissimilarity --no-cpu-baseline --no-clara --steps 15 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('C5 staged=$v', round(d['ms_per_step']*1e3,1), round(r['kernel_ms']*1e3,1), round(r['frac_of_read_only_peak'],4))" >> gpurun_out/r2aa_bench.log; done; done
KM_STREAM_STAGED=2 python -m pytest tests/test_gpu_parity.py tests/test_gpu_goldens.py -x -q -p no:cacheprovider -k "int or c5 or c1 or fastpam2" > gpurun_out/r2aa_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2aa_pytest.log
