import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import kmsynth
from paper_2008_05171_b200 import KMedoids
cid = int(sys.argv[1]); variant = sys.argv[2]
cfg = kmsynth.CONFIGS[cid]
X = kmsynth.make_points(cfg)
Dt = kmsynth.dist_cuda(X, cfg.metric)
km = KMedoids(Dt, cfg.n, cfg.k)
km.set_medoids(kmsynth.random_medoids(cfg))
km.set_profiling(True)
torch.cuda.synchronize()
t0 = time.perf_counter()
its = []
while True:
    t1 = time.perf_counter()
    conv, sw, td = km.swap_iter(variant)
    its.append((time.perf_counter() - t1, sw))
    if conv or len(its) > 3000:
        break
tot = time.perf_counter() - t0
ms, cnt = km.stream_time()
print(f"C{cid} {variant}: iters={len(its)} swaps={sum(s for _, s in its)} total={tot:.3f}s stream_total={ms/1e3:.3f}s td={td}")
print("first iters (s, swaps):", [(round(a*1e3,2), b) for a, b in its[:8]], "last:", [(round(a*1e3,2), b) for a, b in its[-3:]])
