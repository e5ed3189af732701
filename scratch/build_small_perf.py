"""Measurement aid: BUILD time of small problems (CUDA events around
init_build, third call = graph replay), small cooperative kernel vs
KM_BUILD_SMALL=0.  usage: python scratch/build_small_perf.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import kmsynth  # noqa: E402
from paper_2008_05171_b200 import KMedoids, kmedoids_dissimilarity  # noqa: E402

rng = np.random.default_rng(1)
st = torch.cuda.current_stream()
for n, k in [(480, 100), (880, 200), (880, 20), (2080, 500), (4000, 200)]:
    X = (6 * rng.standard_normal((40, 32)))[rng.integers(0, 40, size=n)] + rng.standard_normal((n, 32))
    Xt = torch.from_numpy(X.astype(np.float32)).cuda()
    Dt = kmedoids_dissimilarity(Xt, "l2")
    torch.cuda.synchronize()
    out = []
    for mode in ["1", "0"]:
        os.environ["KM_BUILD_SMALL"] = mode
        km = KMedoids(Dt, n, k, stream=st)
        ts = []
        for _ in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            M, td = km.init_build()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out.append((mode, ts[-1], td, M[:5].tolist()))
        km.close()
    print(f"n={n} k={k}: small {out[0][1]:.3f} ms ({1e3 * out[0][1] / k:.1f} us/step) | incremental {out[1][1]:.3f} ms "
          f"({1e3 * out[1][1] / k:.1f} us/step) | same medoids {out[0][3] == out[1][3]} td {out[0][2]:.6f} {out[1][2]:.6f}",
          flush=True)
