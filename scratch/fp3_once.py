"""One FasterPAM run (random init) for launch-list profiling."""
import sys, os, time, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import kmsynth
from paper_2008_05171_b200 import KMedoids
cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = kmsynth.CONFIGS[cfgi]; n, k = cfg.n, cfg.k
torch.cuda.set_device(0)
X = kmsynth.make_points(cfg); Dt = kmsynth.dist_cuda(X, cfg.metric)
km = KMedoids(Dt, n, k)
km.set_medoids(kmsynth.random_medoids(cfg))
torch.cuda.synchronize(); t0 = time.perf_counter()
r = km.run(use_build=False, variant="fasterpam")
print(f"{cfg.name} fasterpam random init: passes {r.n_iter} swaps {r.n_swaps} td {r.td} wall {1e3*(time.perf_counter()-t0):.1f} ms")
