"""Sharded FastPAM2 on virtual ranks (one GPU, LocalComm): per-rank phase
times of one iteration in the owner-side ("owner") and the column-gather
("gather") forms, for the G-rank projection in DESIGN section 7 (measurement
aid).  usage: python scratch/fp2_owner_perf.py <config> <world> [iters]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import kmsynth  # noqa: E402
from paper_2008_05171_b200 import parallel  # noqa: E402

cid, world = int(sys.argv[1]), int(sys.argv[2])
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = kmsynth.CONFIGS[cid]
n, k = cfg.n, cfg.k
X = kmsynth.make_points(cfg)
Dt = kmsynth.dist_cuda(X, cfg.metric)
M0 = kmsynth.random_medoids(cfg)
cb = parallel.column_bounds(n, world)


def timed(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, 1e3 * (time.perf_counter() - t)


for mode in ("owner", "gather"):
    hs = [parallel.CudaShard(Dt[:, int(cb[r]):], n, k, r, cb) for r in range(world)]
    comm = parallel.LocalComm(world)
    parallel.set_medoids(hs, comm, cb, M0, n)
    for it in range(iters):
        ph = {"eval": [], "plan": [], "round_eval": [], "round_apply": [], "apply": []}
        for h in hs:
            h.fp2_exchange_tensors(world)
            _, t = timed(h.fp2_shard_eval)
            ph["eval"].append(t)
        comm.allgather_fp2_records(hs)
        plans = []
        for h in hs:
            p, t = timed(lambda: h.fp2_shard_plan(cb))
            plans.append(p)
            ph["plan"].append(t)
        m, maxcnt = plans[0]
        rounds = 0
        gbytes = 0
        if m > 0 and mode == "owner":
            while True:
                re = []
                for h in hs:
                    _, t = timed(h.fp2_round_eval)
                    re.append(t)
                ph["round_eval"].append(max(re))
                comm.allgather_fp2_round(hs)
                gbytes += world * hs[0].fp2_round_tensors(world)[2]
                ra = []
                res = []
                for h in hs:
                    r, t = timed(h.fp2_round_apply)
                    ra.append(t)
                    res.append(r)
                ph["round_apply"].append(max(ra))
                rounds += 1
                more, swaps, _ = res[0]
                if not more:
                    break
        elif m > 0:
            for h in hs:
                h.fp2_exchange_tensors(world, need=maxcnt)
            comm.allgather_fp2_columns(hs, maxcnt)
            gbytes = world * maxcnt * 4 * n
            res = []
            for h in hs:
                r, t = timed(h.fp2_shard_apply)
                ph["apply"].append(t)
                res.append(r)
            swaps = res[0][1]
        else:
            swaps = 0
        print(f"C{cid} G={world} {mode} iter {it}: m={m} maxcnt={maxcnt} swaps={swaps} rounds={rounds} "
              f"eval max {max(ph['eval']):.3f} ms, plan max {max(ph['plan']):.3f} ms, "
              f"round_eval sum-of-max {sum(ph['round_eval']):.3f} ms ({[round(x, 3) for x in ph['round_eval']]}), "
              f"round_apply sum-of-max {sum(ph['round_apply']):.3f} ms, "
              f"gather-mode apply max {max(ph['apply']) if ph['apply'] else 0:.3f} ms, "
              f"received per rank {gbytes / 1e6:.1f} MB", flush=True)
    st = hs[0].km.get_state()
    print(f"  {mode}: td {st.td} n_swaps {st.n_swaps}", flush=True)
    for h in hs:
        h.km.close()
