"""Relative error of the tensor-core L2 dissimilarities on the config recipes
(prefix of n points) against the oracle's definition, by distance quantile,
with the exact recomputation of cancelling pairs off (KM_DIST_TAU=0) and on
(default), and the C4 full-size kernel time of both (measurement aid)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kmsynth, oracle
from paper_2008_05171_b200 import kmedoids_dissimilarity
for cid, n in ((4, 6000), (3, 6000), (2, 5000)):
    cfg = kmsynth.CONFIGS[cid]
    X = kmsynth.make_points(cfg, n=n).astype(np.float32)
    Dx = oracle.dist_l2(X).astype(np.float32).astype(np.float64)    # the definition, rounded to f32
    off = ~np.eye(n, dtype=bool)
    q = np.quantile(Dx[off], [0.01, 0.1])
    for tau in ("0", "0.0625"):
        os.environ["KM_DIST_TAU"] = tau
        Dg = kmedoids_dissimilarity(torch.from_numpy(X).cuda(), "l2")[:, :n].double().cpu().numpy()
        r = np.abs(Dg - Dx)[off] / Dx[off]
        d = Dx[off]
        print(f"C{cid} n={n} tau={tau}: max rel all {r.max():.2e}, d<=q10 {r[d <= q[1]].max():.2e}, "
              f"d<=q1 {r[d <= q[0]].max():.2e}, bit-equal {np.mean(Dg[off] == Dx[off]):.4f}", flush=True)
cfg = kmsynth.CONFIGS[4]
Xt = torch.from_numpy(kmsynth.make_points(cfg).astype(np.float32)).cuda()
D = torch.empty((cfg.n, cfg.n), dtype=torch.float32, device="cuda")
for tau in (sys.argv[1].split(",") if len(sys.argv) > 1 else ("0", "0.0625", "0", "0.0625")):
    os.environ["KM_DIST_TAU"] = tau
    kmedoids_dissimilarity(Xt, "l2", D=D)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        kmedoids_dissimilarity(Xt, "l2", D=D)
    b.record()
    b.synchronize()
    print(f"C4 full n={cfg.n} tau={tau}: {a.elapsed_time(b) / 5:.3f} ms per call", flush=True)
