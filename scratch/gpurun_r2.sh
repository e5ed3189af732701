mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_goldens.py tests/test_gpu_sharded.py tests/test_gpu_fasterpam.py -x -q -p no:cacheprovider -k "not c4_build and not c4_fastpam1_full" > gpurun_out/r2g_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2g_pytest.log
python bench.py --no-e2e --no-fasterpam --no-dissimilarity --no-cpu-baseline --steps 40 --warmup 5 > gpurun_out/r2g_bench_c4.log 2>&1
python bench.py --config 3 --no-e2e --no-fasterpam --no-dissimilarity --no-cpu-baseline --steps 40 --warmup 5 > gpurun_out/r2g_bench_c3.log 2>&1
KM_STEP_PROF=1 python -c "
import torch, kmsynth, numpy as np
from paper_2008_05171_b200 import KMedoids
cfg=kmsynth.CONFIGS[4]; X=kmsynth.make_points(cfg); Dt=kmsynth.dist_cuda(X,cfg.metric)
km=KMedoids(Dt,cfg.n,cfg.k); km.init_build()
for _ in range(60): km.swap_iter()
" > gpurun_out/r2g_stepprof.log 2>&1
python bench.py --no-fasterpam --no-dissimilarity --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r2g_bench_e2e.log 2>&1
