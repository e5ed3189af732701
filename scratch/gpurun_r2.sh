mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "run_host or swap_iters" > gpurun_out/r2m_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2m_pytest.log
KM_E2E_PROF=1 python - > gpurun_out/r2m_e2e.log 2>&1 <<'PY'
import time, numpy as np, torch, kmsynth
from paper_2008_05171_b200 import kmedoids_run_host
from paper_2008_05171_b200.kmedoids import pinned_empty
cfg = kmsynth.CONFIGS[4]
X = kmsynth.make_points(cfg)
Dt = kmsynth.dist_cuda(X, cfg.metric)
Dh, Dh_t = pinned_empty(tuple(Dt.shape), cfg.dtype)
Dh_t.copy_(Dt)
del Dt
torch.cuda.synchronize(); torch.cuda.empty_cache()
for i in range(8):
    t = time.perf_counter()
    r = kmedoids_run_host(Dh, cfg.k, use_build=True)
    print("job", i, time.perf_counter() - t, r.n_iter, flush=True)
PY
