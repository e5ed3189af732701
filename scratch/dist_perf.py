"""Time kmedoids_dissimilarity (tensor-core L2 / CUDA-core L1) at config sizes."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import kmsynth
from paper_2008_05171_b200 import kmedoids_dissimilarity
torch.cuda.set_device(0)
for cid in [2, 3, 4, 5, 1]:
    cfg = kmsynth.CONFIGS[cid]
    X = kmsynth.make_points(cfg)
    metric = "l2" if cfg.metric == kmsynth.L2_F32 else "l1"
    Xt = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32 if metric == "l2" else np.int32)).cuda()
    n, d = Xt.shape
    D = kmedoids_dissimilarity(Xt, metric)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        kmedoids_dissimilarity(Xt, metric, D=D)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    gb = D.numel() * 4 / 1e9
    # generator (kmsynth, exact fp64) for comparison
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(); Dg = kmsynth.dist_cuda(X, cfg.metric); g1.record(); torch.cuda.synchronize()
    if metric == "l1":
        same = bool((D[:, :n] == Dg[:, :n]).all().item())
    else:
        same = float((D[:, :n].double() - Dg[:, :n].double()).abs().max().item())
    dpad = (d + 7) // 8 * 8
    tf = 3 * 2 * n * n * dpad / (ms / 1e3) / 1e12 if metric == "l2" else None
    print(f"C{cid} n={n} d={d} {metric}: {ms:.3f} ms, {gb:.2f} GB written -> {gb / (ms / 1e3):.0f} GB/s"
          f"{'' if tf is None else f', {tf:.1f} TFLOP/s tf32'}; kmsynth fp64 generator {g0.elapsed_time(g1):.2f} ms; "
          f"{'identical' if same is True else f'max |diff| vs generator {same}'}", flush=True)
    del D, Dg, Xt
    torch.cuda.empty_cache()
