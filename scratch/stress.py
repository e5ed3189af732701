"""Randomised stress: FastPAM1 / FastPAM2 / FasterPAM / incremental FastPAM1 on
random integer instances (ties, sizes across tiles and parts) vs the oracle."""
import sys, os, time, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import oracle
from paper_2008_05171_b200 import KMedoids
torch.cuda.set_device(0)

def rand_int(rng, n, hi, symmetric=True):
    A = rng.integers(0, hi, size=(n, n)).astype(np.uint32)
    if symmetric:
        A = np.triu(A, 1); A = A + A.T
    np.fill_diagonal(A, 0)
    return A

def to_dev(D):
    n = D.shape[0]
    ld = (n + 3) // 4 * 4
    t = torch.zeros((n, ld), dtype=torch.int32, device="cuda")
    t[:, :n] = torch.from_numpy(D.view(np.int32))
    return t

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
t0 = time.time(); fails = 0; runs = 0
while time.time() - t0 < float(sys.argv[2]) if len(sys.argv) > 2 else 240:
    n = int(rng.choice([5, 17, 64, 129, 300, 777, 1500, 2600]))
    kmax = int(os.environ.get("STRESS_KMAX", "40"))
    k = int(rng.integers(2, min(kmax, n - 1) + 1))
    hi = int(rng.choice([2, 7, 1000, 10**6]))
    D = rand_int(rng, n, hi, symmetric=bool(rng.integers(0, 4)))
    M0 = rng.choice(n, size=k, replace=False).astype(np.int32)
    Dt = to_dev(D)
    for variant, ov in [("fastpam1", oracle.FASTPAM1), ("fastpam2", oracle.FASTPAM2), ("fasterpam", None),
                        ("fastpam1_inc", oracle.FASTPAM1)]:
        ref = oracle.fasterpam_run(D, M0) if ov is None else oracle.swap_run(D, M0, ov)
        km = KMedoids(Dt, n, k)
        km.set_medoids(M0)
        r = km.run(use_build=False, variant=variant)
        km.close()
        runs += 1
        ok = r.medoids.tolist() == ref.medoids.tolist() and r.td == ref.td
        if variant != "fasterpam":
            ok = ok and r.n_iter == ref.n_iter
        if not ok:
            fails += 1
            print("FAIL", variant, n, k, hi, r.td, ref.td, r.n_iter, ref.n_iter, flush=True)
print(f"stress: {runs} runs, {fails} failures, {time.time() - t0:.0f} s", flush=True)
