"""Determinism / trajectory check at C4: handle loop vs run() vs run_host()."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import kmsynth
from paper_2008_05171_b200 import KMedoids, kmedoids_run_host
from paper_2008_05171_b200.kmedoids import pinned_empty
cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = kmsynth.CONFIGS[cfgi]; n, k = cfg.n, cfg.k
torch.cuda.set_device(0)
X = kmsynth.make_points(cfg); Dt = kmsynth.dist_cuda(X, cfg.metric)
def td_of(M):
    idx = torch.as_tensor(np.asarray(M, np.int64), device=Dt.device)
    return Dt[:, idx][:n].double().min(dim=1).values.sum().item()
def loop(prof):
    km = KMedoids(Dt, n, k)
    M, td0 = km.init_build()
    tr = []
    if prof: km.set_profiling(True)
    for it in range(300):
        conv, sw, td = km.swap_iter()
        if conv: break
        (i, c, d), = km.last_swaps()
        tr.append((i, c, d, td))
    st = km.get_state(); km.close()
    return M, td0, tr, st
M1, t1, tr1, s1 = loop(False)
print("loop1 build td", t1, "iters", len(tr1), "final", s1.td, "recomp", td_of(s1.medoids))
M2, t2, tr2, s2 = loop(True)
print("loop2 build td", t2, "iters", len(tr2), "final", s2.td, "recomp", td_of(s2.medoids))
print("build same", (M1 == M2).all(), "trace same", tr1 == tr2)
for j, (a, b) in enumerate(zip(tr1, tr2)):
    if a != b:
        print("first diff at", j, a, b); break
km = KMedoids(Dt, n, k); r = km.run(use_build=True); km.close()
print("run(): iters", r.n_iter, "swaps", r.n_swaps, "td", r.td, "recomp", td_of(r.medoids), "same medoids as loop1", (r.medoids == s1.medoids).all())
Dh, Dh_t = pinned_empty(tuple(Dt.shape), cfg.dtype); Dh_t.copy_(Dt); torch.cuda.synchronize()
r2 = kmedoids_run_host(Dh, k, use_build=True)
print("run_host: iters", r2.n_iter, "swaps", r2.n_swaps, "td", r2.td, "recomp", td_of(r2.medoids), "same medoids as loop1", (r2.medoids == s1.medoids).all())
# verify some trace steps: td after swap recomputed
M = M1.copy()
bad = 0
for j, (i, c, d, td) in enumerate(tr1):
    M[i] = c
    if j % 10 == 0 or j == len(tr1) - 1:
        rt = td_of(M)
        if abs(rt - td) > 1e-9 * abs(rt): bad += 1; print("td mismatch at", j, td, rt)
print("trace td checks bad =", bad)
