import sys, numpy as np, torch
sys.path.insert(0, '.')
import kmsynth
from paper_2008_05171_b200 import KMedoids
cid = int(sys.argv[1])
cfg = kmsynth.CONFIGS[cid]
X = kmsynth.make_points(cfg)
Dt = kmsynth.dist_cuda(X, cfg.metric)
n, k = cfg.n, cfg.k
km = KMedoids(Dt, n, k)
if cfg.init == 'build':
    km.init_build()
else:
    km.set_medoids(kmsynth.random_medoids(cfg))
near, sec, dn, ds = km.get_cache()
D = Dt.view(torch.float32) if cfg.metric == 1 else Dt
dsT = torch.from_numpy(ds.astype(np.float64)).cuda()
dnT = torch.from_numpy(dn.astype(np.float64)).cuda()
tot_hit = 0; tot_i = 0; any32 = 0; cnt32 = 0; anyrow = 0; cntrow = 0
for a in range(0, n, 2000):
    blk = D[a:a+2000, :n].double() if cfg.metric == 1 else D[a:a+2000, :n].to(torch.int64).double()
    h = blk < dsT[a:a+2000, None]
    hi = blk < dnT[a:a+2000, None]
    tot_hit += h.sum().item(); tot_i += hi.sum().item()
    m = n // 128 * 128
    hh = h[:, :m].reshape(h.shape[0], -1, 32, 4)   # rows x warps x lanes x elems
    e_any = hh.any(dim=2)                            # rows x warps x elems
    any32 += e_any.sum().item(); cnt32 += e_any.numel()
    r_any = hh.any(dim=3).any(dim=2)
    anyrow += r_any.sum().item(); cntrow += r_any.numel()
print(f"C{cid}: hit(d<ds) frac={tot_hit/n/n:.5f} case_i frac={tot_i/n/n:.5f} elem-any={any32/cnt32:.4f} row-any={anyrow/cntrow:.4f}")
