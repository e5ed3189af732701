"""One C5-size L1 dissimilarity call (for ncu)."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import kmsynth
from paper_2008_05171_b200 import kmedoids_dissimilarity
torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
X = kmsynth.make_points(kmsynth.CONFIGS[5], n=n) if n <= 100000 else None
Xt = torch.from_numpy(np.ascontiguousarray(X, dtype=np.int32)).cuda()
D = kmedoids_dissimilarity(Xt, "l1")
torch.cuda.synchronize()
print("ok", D.shape)
