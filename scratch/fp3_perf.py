"""FasterPAM vs FastPAM1 time to convergence on a config (GPU)."""
import sys, os, time, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import kmsynth
from paper_2008_05171_b200 import KMedoids
cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 4
init = sys.argv[2] if len(sys.argv) > 2 else "build"
cfg = kmsynth.CONFIGS[cfgi]; n, k = cfg.n, cfg.k
torch.cuda.set_device(0)
X = kmsynth.make_points(cfg); Dt = kmsynth.dist_cuda(X, cfg.metric)
st = torch.cuda.current_stream()
if init == "build":
    km = KMedoids(Dt, n, k); M0, td0 = km.init_build(); km.close()
else:
    M0 = kmsynth.random_medoids(cfg)
for variant in ("fasterpam", "fastpam1", "fasterpam"):
    km = KMedoids(Dt, n, k, stream=st)
    km.set_medoids(M0)
    td0 = km.get_state().td
    km.set_profiling(True); km.stream_time(reset=True)
    l0 = km.launch_count()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    passes = 0; swaps = 0; per = []
    while True:
        t1 = time.perf_counter()
        conv, sw, td = km.swap_iter(variant)
        per.append((sw, time.perf_counter() - t1))
        passes += 1; swaps += sw
        if conv or passes > 3000: break
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    ms, nl = km.stream_time(reset=True)
    print(f"{cfg.name} {variant}: init td {td0:.6g} -> {td:.10g}; passes {passes} swaps {swaps}; wall {dt*1e3:.1f} ms; "
          f"stream {ms:.1f} ms in {nl} launches; kernels {km.launch_count()-l0}")
    if variant == "fasterpam":
        print("   per pass (swaps, ms):", [(a, round(b * 1e3, 2)) for a, b in per[:8]])
    km.close()
