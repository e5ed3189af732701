"""Measurement aid: kmedoids_dissimilarity (L2) at C3/C4 sizes, ms per call."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import kmsynth  # noqa: E402
from paper_2008_05171_b200 import kmedoids_dissimilarity  # noqa: E402

for cid in [3, 4]:
    cfg = kmsynth.CONFIGS[cid]
    X = kmsynth.make_points(cfg)
    Xt = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).cuda()
    D = kmedoids_dissimilarity(Xt, "l2")
    torch.cuda.synchronize()
    res = []
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            kmedoids_dissimilarity(Xt, "l2", D=D)
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / 5)
    print(f"C{cid} center={os.environ.get('KM_DIST_CENTER', '1')}: ms", " ".join(f"{x:.3f}" for x in res), flush=True)
    del D
    torch.cuda.empty_cache()
