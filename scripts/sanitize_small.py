#!/usr/bin/env python3
"""Small run of every kernel family of libkmedoids.so, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck, one tool per run):

  BUILD + FastPAM1 (single iterations and the queued path), FastPAM2,
  FasterPAM, incremental FastPAM1, distance-weighted and LAB seeding,
  dissimilarities from points (L2 tensor cores, L1), FastCLARA (matrix and
  from points), and the column-sharded phases with two virtual ranks.

Sizes are tiny (n <= 1200) but span several column tiles, row parts and
ragged tails.  Results are checked against the oracle so a run under the
tool is also a parity run.  Exit code 0 = every check passed.

usage: compute-sanitizer --tool memcheck python scripts/sanitize_small.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import kmsynth  # noqa: E402
import oracle  # noqa: E402
from paper_2008_05171_b200 import (KMedoids, kmedoids_clara_points, kmedoids_dissimilarity,  # noqa: E402
                                   parallel)


def to_dev(D):
    n = D.shape[0]
    ld = kmsynth.round_ld(n)
    buf = np.zeros((n, ld), D.dtype)
    buf[:, :n] = D
    return torch.from_numpy(buf.view(np.int32) if D.dtype == np.uint32 else buf).cuda()


def rand_int(rng, n, hi):
    A = rng.integers(0, hi, size=(n, n)).astype(np.uint32)
    A = np.triu(A, 1)
    A = A + A.T
    np.fill_diagonal(A, 0)
    return A


def check(cond, what):
    if not cond:
        raise SystemExit(f"FAILED: {what}")
    print("ok", what, flush=True)


def main():
    torch.cuda.set_device(0)
    rng = np.random.default_rng(2024)
    n, k = 1100, 7
    D = rand_int(rng, n, 500)
    Dt = to_dev(D)
    M0 = rng.choice(n, size=k, replace=False).astype(np.int32)

    # BUILD + FastPAM1, single iterations then the queued path
    Mb, _, _ = oracle.build_init(D, k)
    ref = oracle.swap_run(D, Mb, oracle.FASTPAM1)
    km = KMedoids(Dt, n, k)
    M, td = km.init_build()
    check(M.tolist() == Mb.tolist(), "BUILD")
    for _ in range(2):
        km.swap_iter()
    km.swap_iters(2000)
    st = km.get_state()
    check(st.medoids.tolist() == ref.medoids.tolist() and st.td == ref.td, "FastPAM1")
    km.eval_candidates()
    # FastPAM2
    km.set_medoids(M0)
    r2 = oracle.swap_run(D, M0, oracle.FASTPAM2)
    while not km.swap_iter("fastpam2")[0]:
        pass
    check(km.get_state().medoids.tolist() == r2.medoids.tolist(), "FastPAM2")
    # FasterPAM and incremental FastPAM1
    km.set_medoids(M0)
    rf = km.run(use_build=False, variant="fasterpam")
    check(rf.medoids.tolist() == oracle.fasterpam_run(D, M0).medoids.tolist(), "FasterPAM")
    km.set_medoids(M0)
    ri = km.run(use_build=False, variant="fastpam1_inc")
    check(ri.medoids.tolist() == oracle.swap_run(D, M0, oracle.FASTPAM1).medoids.tolist(), "incremental FastPAM1")
    # seeding
    u = rng.random(k)
    Mw, _ = km.init_weighted(u)
    check(Mw.tolist() == oracle.init_weighted(D, k, u).tolist(), "distance-weighted seeding")
    s, rows = oracle.lab_sample_rows(n, k, 9)
    Ml, _ = km.init_lab(s, rows)
    check(Ml.tolist() == oracle.init_lab(D, k, s, rows).tolist(), "LAB")
    # CLARA on the matrix
    samples = np.stack([rng.choice(n, size=80 + 4 * k, replace=False) for _ in range(3)])
    Mc, tdc, bc = km.clara(samples)
    tc, jc, Mco = oracle.clara(D, k, samples)
    check((Mc.tolist(), tdc, bc) == (Mco.tolist(), tc, jc), "CLARA (matrix)")
    km.close()

    # dissimilarities from points
    cfg = kmsynth.CONFIGS[4]
    X = kmsynth.make_points(cfg, n=700).astype(np.float32)
    D2 = kmedoids_dissimilarity(torch.from_numpy(X).cuda(), "l2")[:, :700].double().cpu().numpy()
    check(np.abs(D2 - oracle.dist_l2(X)).max() < 1e-2, "L2 dissimilarity (tensor cores)")
    Xq = kmsynth.make_points(kmsynth.CONFIGS[5], n=600)
    D1 = kmedoids_dissimilarity(torch.from_numpy(np.ascontiguousarray(Xq)).cuda(), "l1")[:, :600].cpu().numpy()
    check((D1.view(np.uint32).astype(np.int64) == oracle.dist_l1(Xq)).all(), "L1 dissimilarity")

    # CLARA from points
    samples = np.stack([rng.choice(600, size=60, replace=False) for _ in range(3)])
    Mp, tdp, bp, _ = kmedoids_clara_points(torch.from_numpy(np.ascontiguousarray(Xq)).cuda(), "l1", 4, samples)
    tp, jp, Mpo, _ = oracle.clara_points(Xq, "l1", 4, samples)
    check((Mp.tolist(), tdp, bp) == (Mpo.tolist(), tp, jp), "CLARA from points")

    # column-sharded phases, two virtual ranks
    cb = parallel.column_bounds(n, 2)
    hs = [parallel.CudaShard(Dt[:, int(cb[r]):], n, k, r, cb) for r in range(2)]
    comm = parallel.LocalComm(2)
    Ms = parallel.build_async(hs, comm, cb, k)
    check(Ms == Mb.tolist(), "sharded BUILD")
    trace, iters, conv = parallel.run(hs, comm, cb)
    check([(a, b) for a, b, _ in trace] == [(a, b) for a, b, _ in ref.trace], "sharded FastPAM1")
    parallel.set_medoids(hs, comm, cb, M0, n)
    while not parallel.fp2_iter(hs, comm, cb)[0]:
        pass
    check(hs[0].km.get_state().medoids.tolist() == r2.medoids.tolist(), "sharded FastPAM2")
    torch.cuda.synchronize()
    print("all checks passed", flush=True)


if __name__ == "__main__":
    main()
