"""Measurement aid: FastCLARA from points at n = 1e6, d = 32, k = 200 (a 4 TB
matrix if materialised), 5 samples of s = 80 + 4k and of s = sqrt(n) + 4k
(P:1122-1126); wall clock of the third identical call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2008_05171_b200 import kmedoids_clara_points  # noqa: E402

rng = np.random.default_rng(3)
n, d, k = 1_000_000, 32, 200
X = ((8 * rng.standard_normal((400, d)))[rng.integers(0, 400, size=n)] + rng.standard_normal((n, d))).astype(np.float32)
Xt = torch.from_numpy(X).cuda()
for s in (80 + 4 * k, int(np.sqrt(n)) + 4 * k):
    samples = np.stack([rng.choice(n, size=s, replace=False) for _ in range(5)])
    for v in ("fastpam1", "fasterpam"):
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            M, td, b, _ = kmedoids_clara_points(Xt, "l2", k, samples, v)
            ms = (time.perf_counter() - t0) * 1e3
        print(f"n=1e6 d=32 k=200 5 x s={s} {v}: {ms:.1f} ms TD {td:.6g} best {b}", flush=True)
