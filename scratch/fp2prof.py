"""Per-phase FastPAM2 iteration profile (measurement aid): KM_STEP_PROF=1
python scratch/fp2prof.py <config> [iters] (restarts from the initial medoids
on convergence)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kmsynth  # noqa: E402
from paper_2008_05171_b200 import KMedoids  # noqa: E402

cid = int(sys.argv[1])
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = kmsynth.CONFIGS[cid]
X = kmsynth.make_points(cfg)
Dt = kmsynth.dist_cuda(X, cfg.metric)
km = KMedoids(Dt, cfg.n, cfg.k, stream=torch.cuda.current_stream())
km.set_symmetric(True)
M0 = kmsynth.random_medoids(cfg)
km.set_medoids(M0)
done = 0
sw = []
while done < iters:
    conv, s, td = km.swap_iter("fastpam2")
    if conv:
        km.set_medoids(M0)
        continue
    sw.append(s)
    done += 1
print(f"C{cid}: {done} FastPAM2 iterations, swaps per iteration {sw}", flush=True)
