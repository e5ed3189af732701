"""BUILD (Alg.1) timing on the device: the first call (direct launches) and
replays (CUDA graph), CUDA events on the library's stream (measurement aid).
usage: python scratch/build_perf.py <config> [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kmsynth  # noqa: E402
from paper_2008_05171_b200 import KMedoids  # noqa: E402

cid = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = kmsynth.CONFIGS[cid]
X = kmsynth.make_points(cfg)
Dt = kmsynth.dist_cuda(X, cfg.metric)
st = torch.cuda.current_stream()
km = KMedoids(Dt, cfg.n, cfg.k, stream=st)
ts = []
for r in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    M, td = km.init_build()
    b.record(st)
    b.synchronize()
    ts.append(a.elapsed_time(b))
print(f"C{cid} BUILD ms per call: {[round(t, 3) for t in ts]} td {td} medoids[:5] {list(M[:5])}", flush=True)
