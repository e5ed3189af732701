"""Relative error of the tensor-core L2 dissimilarities on the config recipes
(prefix of n points), by distance quantile, with and without centring."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kmsynth, oracle
from paper_2008_05171_b200 import kmedoids_dissimilarity
for cid, n in ((3, 6000), (4, 6000), (2, 5000)):
    cfg = kmsynth.CONFIGS[cid]
    X = kmsynth.make_points(cfg, n=n).astype(np.float32)
    Dx = oracle.dist_l2(X)
    off = ~np.eye(n, dtype=bool)
    q = np.quantile(Dx[off], [0.01, 0.1])
    for env in ("0", "1"):
        os.environ["KM_DIST_CENTER"] = env
        Dg = kmedoids_dissimilarity(torch.from_numpy(X).cuda(), "l2")[:, :n].double().cpu().numpy()
        r = np.abs(Dg - Dx)[off] / Dx[off]
        d = Dx[off]
        print(f"C{cid} n={n} center={env}: max rel all {r.max():.2e}, max rel d<=q10 {r[d <= q[1]].max():.2e}, "
              f"max rel d<=q1 {r[d <= q[0]].max():.2e}, max abs {np.abs(Dg - Dx)[off].max():.2e}", flush=True)
