"""Find nondeterminism in eval_candidates along the C4 trajectory."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import kmsynth
from paper_2008_05171_b200 import KMedoids
cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 4
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 80
cfg = kmsynth.CONFIGS[cfgi]; n, k = cfg.n, cfg.k
torch.cuda.set_device(0)
X = kmsynth.make_points(cfg); Dt = kmsynth.dist_cuda(X, cfg.metric)
def exact(M, cands):
    idx = torch.as_tensor(np.asarray(M, np.int64), device=Dt.device)
    Dm = Dt[:n, idx].double()
    v2, j2 = torch.topk(Dm, 2, dim=1, largest=False)
    # nearest with smallest slot on ties: topk tie order not guaranteed; only values matter for dTD
    dn, ds = v2[:, 0], v2[:, 1]
    near = j2[:, 0]
    td = dn.sum()
    out = []
    for c in cands:
        col = Dt[:n, c].double()
        a = torch.minimum(col, dn)
        b = torch.minimum(col, ds) - a
        per = torch.zeros(k, dtype=torch.float64, device=Dt.device).index_add_(0, near, b)
        d = (a.sum() + per - td).cpu().numpy()
        out.append(d)
    return out
km = KMedoids(Dt, n, k)
M, td0 = km.init_build()
if cfg.init != "build" and len(sys.argv) > 3:
    M = kmsynth.random_medoids(cfg); km.set_medoids(M)
nd = 0
for it in range(maxit):
    M = km.get_state().medoids
    v1, s1 = km.eval_candidates()
    v2, s2 = km.eval_candidates()
    diff = np.nonzero((v1 != v2) | (s1 != s2))[0]
    if len(diff):
        nd += 1
        print(f"iter {it}: {len(diff)} candidates differ between two evals; first {diff[:8].tolist()}")
        ex = exact(M, diff[:4])
        for c, e in zip(diff[:4], ex):
            print(f"  c={c} run1=({v1[c]:.6f},{s1[c]}) run2=({v2[c]:.6f},{s2[c]}) exact min={e.min():.6f} argmin={int(np.argmin(e))}")
        np.save(os.path.join("gpurun_out", f"race_M_it{it}.npy"), M)
        if nd >= 3: break
    conv, sw, td = km.swap_iter()
    if conv: print("converged at", it); break
print("done, nondeterministic iterations:", nd)
