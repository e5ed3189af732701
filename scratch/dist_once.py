import sys, os, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import kmsynth
from paper_2008_05171_b200 import kmedoids_dissimilarity
cfg = kmsynth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
X = torch.from_numpy(np.ascontiguousarray(kmsynth.make_points(cfg), dtype=np.float32)).cuda()
D = kmedoids_dissimilarity(X, "l2"); torch.cuda.synchronize()
D = kmedoids_dissimilarity(X, "l2", D=D); torch.cuda.synchronize()
print("ok", D.shape)
