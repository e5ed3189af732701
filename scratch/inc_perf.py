"""Streaming FastPAM1 vs incremental FastPAM1 (same swaps) to convergence."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import kmsynth
from paper_2008_05171_b200 import KMedoids
cid = int(sys.argv[1]); init = sys.argv[2]
cfg = kmsynth.CONFIGS[cid]; n, k = cfg.n, cfg.k
torch.cuda.set_device(0)
X = kmsynth.make_points(cfg); Dt = kmsynth.dist_cuda(X, cfg.metric)
st = torch.cuda.current_stream()
km = KMedoids(Dt, n, k, stream=st)
M0 = km.init_build()[0] if init == "build" else kmsynth.random_medoids(cfg)
for variant in ["fastpam1_inc", "fastpam1", "fastpam1_inc"]:
    km.set_medoids(M0)
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); r = km.run(use_build=False, variant=variant); e1.record(st); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"C{cid} {init} {variant:13s}: {ms:9.2f} ms, {r.n_iter} iters ({ms / r.n_iter * 1e3:.0f} us/iter), "
          f"{r.n_swaps} swaps, TD {r.td:.10g}", flush=True)
