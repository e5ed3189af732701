import os, sys, numpy as np, torch
sys.path.insert(0, '.')
import kmsynth
from paper_2008_05171_b200 import KMedoids
rng = np.random.default_rng(8)
for n, k, dim in [(1500, 17, 5), (300, 5, 3), (100, 3, 2)]:
    X = rng.normal(size=(n, dim))
    D = kmsynth.dist_numpy(X, kmsynth.L2_F32)
    Dt = torch.from_numpy(D).cuda()
    M0 = rng.choice(n, size=k, replace=False)
    res = {}
    for kind in ("tma", "seg"):
        os.environ["KM_STREAM"] = kind
        km = KMedoids(Dt, n, k)
        km.set_medoids(M0)
        res[kind] = km.eval_candidates()
    v1, s1 = res["tma"]; v2, s2 = res["seg"]
    bad = np.where((np.abs(v1 - v2) > 1e-6 * np.abs(v1).max()) | (s1 != s2))[0]
    print(n, k, "bad", len(bad), bad[:10], v1[bad[:5]], v2[bad[:5]], s1[bad[:5]], s2[bad[:5]])
