import os, sys, numpy as np, torch
sys.path.insert(0, '.')
import kmsynth
from paper_2008_05171_b200 import KMedoids
cfg = kmsynth.CONFIGS[2]
n = 2000
X = kmsynth.make_points(cfg, n=n)
Dt = kmsynth.dist_cuda(X, cfg.metric)
res = {}
for kind in ("tma", "seg"):
    os.environ["KM_STREAM"] = kind
    km = KMedoids(Dt, n, cfg.k)
    M, td = km.init_build()
    res[kind] = km.eval_candidates()
    print(kind, M[:5], td)
v1, s1 = res["tma"]; v2, s2 = res["seg"]
bad = np.where((np.abs(v1 - v2) > 1e-6 * np.abs(v1[s1>=0]).max()) | (s1 != s2))[0]
print(n, "bad", len(bad), bad[:10], v1[bad[:5]], v2[bad[:5]], s1[bad[:5]], s2[bad[:5]])
# same with set_medoids
for kind in ("tma", "seg"):
    os.environ["KM_STREAM"] = kind
    km = KMedoids(Dt, n, cfg.k)
    km.set_medoids(M)
    res[kind] = km.eval_candidates()
v1, s1 = res["tma"]; v2, s2 = res["seg"]
bad = np.where((np.abs(v1 - v2) > 1e-6 * np.abs(v1[s1>=0]).max()) | (s1 != s2))[0]
print(n, "bad(set)", len(bad), bad[:10], v1[bad[:5]], v2[bad[:5]], s1[bad[:5]], s2[bad[:5]])
