"""Repro aid: kmedoids_clara_points at C4 (5 samples, s = 880), FastPAM1 and
FasterPAM, three calls each (as bench.py), repeated R times."""
import os
import sys

import time

import numpy as np
import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import kmsynth  # noqa: E402
from paper_2008_05171_b200 import kmedoids_clara_points  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 1
NS = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = kmsynth.CONFIGS[4]
X = kmsynth.make_points(cfg)
Xt = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).cuda()
n, k = cfg.n, cfg.k
s_cl = min(n, 80 + 4 * k)
crng = np.random.default_rng(cfg.seed + 2000)
samples = np.stack([crng.choice(n, size=s_cl, replace=False) for _ in range(NS)])
for r in range(R):
    for v in ("fastpam1", "fasterpam"):
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            M, td, b, _ = kmedoids_clara_points(Xt, "l2", k, samples, v)
            ms = (time.perf_counter() - t0) * 1e3
        print("rep", r, v, "td", td, "best", b, f"third call {ms:.2f} ms", flush=True)
print("clara repro ok", flush=True)
