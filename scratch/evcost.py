"""Measurement aid: FastPAM1 step time over K queued iterations (one event pair
around the whole batch), e.g. KM_GRAPH_EVENTS=0 vs 1.
usage: python scratch/evcost.py <config> [K]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kmsynth  # noqa: E402
from paper_2008_05171_b200 import KMedoids  # noqa: E402

cid = int(sys.argv[1])
K = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cfg = kmsynth.CONFIGS[cid]
X = kmsynth.make_points(cfg)
Dt = kmsynth.dist_cuda(X, cfg.metric)
st = torch.cuda.current_stream()
km = KMedoids(Dt, cfg.n, cfg.k, stream=st)
km.set_symmetric(True)
if cfg.init == "build":
    M0, _ = km.init_build()
else:
    M0 = kmsynth.random_medoids(cfg)
    km.set_medoids(M0)
for _ in range(3):
    km.swap_iter("fastpam1")
M1 = km.get_state().medoids
res = []
kern = []
for rep in range(5):
    km.set_medoids(M1)
    km.swap_iters(2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    km.set_profiling(True)
    km.stream_time(reset=True)
    torch.cuda.synchronize()
    e0.record(st)
    conv, done, sw, td = km.swap_iters(K)
    e1.record(st)
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / done)
    ms, cnt = km.stream_time()
    kern.append(ms / max(cnt, 1))
print(f"C{cid} KM_GRAPH_EVENTS={os.environ.get('KM_GRAPH_EVENTS', '1')}: ms/step", " ".join(f"{x:.4f}" for x in res),
      "| stream", " ".join(f"{x:.4f}" for x in kern), f"done={done} conv={conv}", flush=True)
