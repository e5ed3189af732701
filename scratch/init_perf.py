"""Init + SWAP pipelines on a config: BUILD / distance-weighted / LAB, then FastPAM1 / FasterPAM."""
import sys, os, time, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import kmsynth
from paper_2008_05171_b200 import KMedoids
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = kmsynth.CONFIGS[cid]; n, k = cfg.n, cfg.k
torch.cuda.set_device(0)
X = kmsynth.make_points(cfg); Dt = kmsynth.dist_cuda(X, cfg.metric)
st = torch.cuda.current_stream()
import math
s = 10 + math.ceil(math.sqrt(n))
rng = np.random.Generator(np.random.PCG64(cfg.seed + 3000))
u = rng.random(k)
rows = np.stack([rng.choice(n, size=min(n, s + k), replace=False) for _ in range(k)]).astype(np.int32)
def timed(fn):
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); r = fn(); e1.record(st); torch.cuda.synchronize(); return r, e0.elapsed_time(e1)
for init in ["build", "weighted", "lab"]:
    km = KMedoids(Dt, n, k, stream=st)
    km.init_weighted(u) if init == "weighted" else (km.init_lab(s, rows) if init == "lab" else None)   # warm-up
    if init == "build": (M, td0), ms = timed(km.init_build)
    elif init == "weighted": (M, td0), ms = timed(lambda: km.init_weighted(u))
    else: (M, td0), ms = timed(lambda: km.init_lab(s, rows))
    for variant in ["fastpam1", "fasterpam"]:
        km.set_medoids(M)
        km.run(use_build=False, variant=variant) if variant == "fasterpam" else None   # warm-up allocations
        km.set_medoids(M)
        r, ms2 = timed(lambda: km.run(use_build=False, variant=variant))
        print(f"C{cid} {init:9s} init {ms:8.2f} ms (TD {td0:.6g}) + {variant:9s} {ms2:8.2f} ms: {r.n_iter} iters, "
              f"{r.n_swaps} swaps, TD {r.td:.10g}", flush=True)
    km.close()
