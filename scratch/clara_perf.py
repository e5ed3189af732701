"""FastCLARA (5 samples of 80 + 4k) at a config vs the full-matrix runs."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import kmsynth
from paper_2008_05171_b200 import KMedoids
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = kmsynth.CONFIGS[cid]; n, k = cfg.n, cfg.k
torch.cuda.set_device(0)
X = kmsynth.make_points(cfg); Dt = kmsynth.dist_cuda(X, cfg.metric)
st = torch.cuda.current_stream()
s = min(n, 80 + 4 * k)
rng = np.random.Generator(np.random.PCG64(cfg.seed + 5000))
S = np.stack([rng.choice(n, size=s, replace=False) for _ in range(5)]).astype(np.int32)
km = KMedoids(Dt, n, k, stream=st)
km.clara(S, "fastpam1"); km.clara(S, "fasterpam")          # warm-up (nested handles, scratch, graphs)
for variant in ["fastpam1", "fasterpam"]:
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); M, td, j = km.clara(S, variant); e1.record(st); torch.cuda.synchronize()
    print(f"C{cid} FastCLARA 5 x s={s} {variant}: {e0.elapsed_time(e1):.1f} ms, TD {td:.10g} (best sample {j})", flush=True)
