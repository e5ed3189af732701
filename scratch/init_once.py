import sys, os, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import kmsynth
from paper_2008_05171_b200 import KMedoids
cid = int(sys.argv[1]); which = sys.argv[2]
cfg = kmsynth.CONFIGS[cid]; n, k = cfg.n, cfg.k
X = kmsynth.make_points(cfg); Dt = kmsynth.dist_cuda(X, cfg.metric)
km = KMedoids(Dt, n, k)
u = np.random.default_rng(1).random(k)
import math
s = 10 + math.ceil(math.sqrt(n))
rows = np.stack([np.random.default_rng(i).choice(n, size=s + k, replace=False) for i in range(k)]).astype(np.int32)
for _ in range(2):
    M, td = km.init_weighted(u) if which == "w" else km.init_lab(s, rows)
print("ok", td)
