"""Per-phase FastPAM1 step profile (measurement aid): single swap_iter calls
with KM_STEP_PROF=1 (launch -> stream, stream, combine, post; post phases).
usage: KM_STEP_PROF=1 python scratch/stepprof.py <config> [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kmsynth  # noqa: E402
from paper_2008_05171_b200 import KMedoids  # noqa: E402

cid = int(sys.argv[1])
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
cfg = kmsynth.CONFIGS[cid]
X = kmsynth.make_points(cfg)
Dt = kmsynth.dist_cuda(X, cfg.metric)
km = KMedoids(Dt, cfg.n, cfg.k, stream=torch.cuda.current_stream())
km.set_symmetric(True)
if cfg.init == "build":
    M0, _ = km.init_build()
else:
    M0 = kmsynth.random_medoids(cfg)
    km.set_medoids(M0)
for _ in range(5):
    km.swap_iter("fastpam1")
done = restarts = 0
while done < iters:
    conv, sw, td = km.swap_iter("fastpam1")
    if conv:                      # converged: restart from the initial medoids (small configs)
        km.set_medoids(M0)
        restarts += 1
        continue
    done += 1
print(f"C{cid}: {done} single iterations, {restarts} restarts", flush=True)
