mkdir -p gpurun_out
python -m pytest tests/test_gpu_clara_points.py -x -q -p no:cacheprovider > gpurun_out/r2i_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2i_pytest.log
python - > gpurun_out/r2i_clara_time.log 2>&1 <<'PY'
import time, numpy as np, torch, kmsynth
from paper_2008_05171_b200 import kmedoids_clara_points
for cid in (4, 5):
    cfg = kmsynth.CONFIGS[cid]
    X = kmsynth.make_points(cfg)
    metric = "l2" if cfg.metric == kmsynth.L2_F32 else "l1"
    Xt = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32 if metric == "l2" else np.int32)).cuda()
    rng = np.random.default_rng(5)
    s = 80 + 4 * cfg.k
    samples = np.stack([rng.choice(cfg.n, size=s, replace=False) for _ in range(5)])
    for v in ("fastpam1", "fasterpam"):
        kmedoids_clara_points(Xt, metric, cfg.k, samples, v)
        torch.cuda.synchronize(); t = time.perf_counter()
        M, td, b, _ = kmedoids_clara_points(Xt, metric, cfg.k, samples, v)
        print(cfg.name, v, "s", s, "time_ms", (time.perf_counter() - t) * 1e3, "td", td, "best", b, flush=True)
rng = np.random.default_rng(6)
n, d, k = 1_000_000, 32, 200
X = (8.0 * rng.standard_normal((200, d)))[rng.integers(0, 200, size=n)] + rng.standard_normal((n, d))
Xt = torch.from_numpy(X.astype(np.float32)).cuda()
samples = np.stack([rng.choice(n, size=80 + 4 * k, replace=False) for _ in range(5)])
kmedoids_clara_points(Xt, "l2", k, samples)
torch.cuda.synchronize(); t = time.perf_counter()
M, td, b, _ = kmedoids_clara_points(Xt, "l2", k, samples)
print("n=1e6 d=32 k=200 fastpam1 s", 80 + 4 * k, "time_ms", (time.perf_counter() - t) * 1e3, "td", td, flush=True)
PY
