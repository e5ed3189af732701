#!/usr/bin/env python3
"""Full-size oracle goldens for the BASELINE.json workloads (SURVEY 8(c)
"trust chain").

Calls ONLY oracle/ (the plain single-threaded C restatement of the paper)
and kmsynth/ (the seeded input generator, no method arithmetic): nothing here
touches the CUDA path.  Each job writes one JSON file under tests/golden/full/
that the GPU parity tests (tests/test_gpu_goldens.py) compare the library's
whole trajectory with:

  c2_fastpam1   C2 n=5000  k=20  f32: BUILD (Alg.1) + FastPAM1 (Alg.3) to convergence
  c3_fastpam1   C3 n=20000 k=100 f32: random init + FastPAM1 to convergence
  c3_fastpam2   C3: random init + FastPAM2 (reading R6) to convergence, with
                the per-slot plan (v_i, c_i) of the first 3 iterations
  c4_build      C4 n=50000 k=200 f32: BUILD medoids, per-step gains, TD
  c4_fastpam1   C4: FastPAM1 from the BUILD medoids of c4_build, to convergence
  c5_fastpam2   C5 n=100000 k=500 u32: random init + 3 FastPAM2 iterations,
                with the per-slot plan of each iteration
  c3_fasterpam  C3: random init + FasterPAM (Alg.4, readings F1-F5) to convergence
  c4_fasterpam  C4: FasterPAM from the c4_build medoids to convergence

D is materialised on the CPU by kmsynth.dist_cpu, which is bit-identical to
kmsynth.dist_numpy and to the CUDA materialiser the GPU tests use (tests:
test_synth_*); its SHA-256 is recorded so a test can refuse a different D.

Usage: python scripts/make_goldens.py JOB [JOB ...]   (C4 takes ~2 h of one
core; C5 needs a 40 GB host buffer.)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import kmsynth  # noqa: E402
import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "full")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8)).hexdigest()


def num(v):
    return int(v) if isinstance(v, (int, np.integer)) else float(v)


def make_D(cid: int):
    cfg = kmsynth.CONFIGS[cid]
    X = kmsynth.make_points(cfg)
    t = time.time()
    D = kmsynth.dist_cpu(X, cfg.metric)
    assert D.shape == (cfg.n, cfg.n), "goldens assume ld == n"
    print(f"[C{cid}] D materialised in {time.time() - t:.1f} s", flush=True)
    return cfg, D


def header(cfg, D, job, what):
    return {"job": job, "config": cfg.name, "n": cfg.n, "k": cfg.k, "dtype": str(D.dtype),
            "D_sha256": sha(D), "generated_by": "scripts/make_goldens.py (oracle/ + kmsynth/ only)",
            "what": what}


def final_block(D, r):
    counts = np.bincount(r.assignment, minlength=len(r.medoids))
    return {"medoids": r.medoids.tolist(), "td": num(r.td), "n_iter": r.n_iter, "n_swaps": r.n_swaps,
            "converged": bool(r.converged), "assignment_sha256": sha(r.assignment.astype(np.int32)),
            "assignment_counts": counts.tolist()}


def slot_plan(D, M, td):
    """Reading R6 steps 2-5 at the state M: per-slot (v_i, c_i) and the
    improving slots in ascending (v_i, i)."""
    c = oracle.assign(D, M)
    R = oracle.removal_loss(c, len(M))
    sv, sc = oracle.fastpam2_slot_best(D, M, c, R)
    if D.dtype == np.uint32:
        imp = [i for i in range(len(M)) if sc[i] >= 0 and sv[i] < 0]
    else:
        imp = [i for i in range(len(M)) if sc[i] >= 0 and sv[i] < -oracle.EPS_REL * abs(td)]
    order = sorted(imp, key=lambda i: (sv[i], i))
    return {"v": [num(x) for x in sv], "c": sc.tolist(), "order": order}


def write(name, obj):
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, name + ".json")
    with open(path + ".tmp", "w") as f:
        json.dump(obj, f, separators=(",", ":"))
    os.replace(path + ".tmp", path)
    print(f"wrote {path} ({os.path.getsize(path)} B)", flush=True)


def job_build_fp1(cid, name, with_swap=True):
    cfg, D = make_D(cid)
    t = time.time()
    Mb, tdb, gains = oracle.build_init(D, cfg.k)
    tb = time.time() - t
    print(f"[{name}] BUILD {tb:.0f} s", flush=True)
    g = header(cfg, D, name, "BUILD (Alg.1, readings R3/R4)" + (" + FastPAM1 (Alg.3) to convergence" if with_swap else ""))
    g["build"] = {"medoids": Mb.tolist(), "td": num(tdb), "gains": [num(x) for x in gains], "oracle_s": round(tb, 1)}
    if with_swap:
        t = time.time()
        r = oracle.swap_run(D, Mb, oracle.FASTPAM1)
        g["fastpam1"] = {"init": Mb.tolist(), "trace": [[a, b, num(v)] for a, b, v in r.trace],
                         "final": final_block(D, r), "oracle_s": round(time.time() - t, 1)}
    write(name, g)
    return g


def job_c4_fastpam1():
    path = os.path.join(OUT, "c4_build.json")
    with open(path) as f:
        Mb = json.load(f)["build"]["medoids"]
    cfg, D = make_D(4)
    t = time.time()
    r = oracle.swap_run(D, Mb, oracle.FASTPAM1)
    g = header(cfg, D, "c4_fastpam1", "FastPAM1 (Alg.3) to convergence from the c4_build medoids")
    g["fastpam1"] = {"init": list(Mb), "trace": [[a, b, num(v)] for a, b, v in r.trace],
                     "final": final_block(D, r), "oracle_s": round(time.time() - t, 1)}
    write("c4_fastpam1", g)


def job_random(cid, name, variant, plan_iters=0, max_iter=2000):
    cfg, D = make_D(cid)
    M0 = kmsynth.random_medoids(cfg)
    g = header(cfg, D, name, f"random init (seed+1000) + {'FastPAM1' if variant == oracle.FASTPAM1 else 'FastPAM2 (R6)'}"
               + (f", {max_iter} iterations" if max_iter < 2000 else " to convergence"))
    t = time.time()
    r = oracle.swap_run(D, M0, variant, max_iter=max_iter)
    g["run"] = {"init": M0.tolist(), "trace": [[a, b, num(v)] for a, b, v in r.trace], "final": final_block(D, r)}
    print(f"[{name}] run: {r.n_iter} iterations, {r.n_swaps} swaps, {time.time() - t:.0f} s", flush=True)
    if plan_iters:
        # the first iterations one by one, with the per-slot plan at the start
        # of each: the oracle's FastPAM2 iteration depends only on M (its
        # cache is recomputed from scratch), so max_iter=1 calls chained from
        # the returned medoids retrace the run (checked against its trace)
        M = M0.copy()
        iters, pos = [], 0
        for it in range(min(plan_iters, r.n_iter)):
            td = oracle.td(D, M)
            plan = slot_plan(D, M, td)
            ri = oracle.swap_run(D, M, variant, max_iter=1)
            sw = [[a, b, num(v)] for a, b, v in ri.trace]
            assert [x[:2] for x in sw] == [x[:2] for x in g["run"]["trace"][pos:pos + len(sw)]]
            pos += len(sw)
            iters.append({"td_before": num(td), "plan": plan, "swaps": sw})
            M = ri.medoids.copy()
            print(f"[{name}] plan of iteration {it + 1}: {len(plan['order'])} improving slots, {len(sw)} swaps",
                  flush=True)
        g["run"]["iterations"] = iters
    g["run"]["oracle_s"] = round(time.time() - t, 1)
    write(name, g)


def job_fasterpam(cid, name, from_build=None):
    cfg, D = make_D(cid)
    if from_build:
        with open(os.path.join(OUT, from_build + ".json")) as f:
            M0 = np.asarray(json.load(f)["build"]["medoids"], np.int32)
        what = f"FasterPAM (Alg.4, F1-F5) to convergence from the {from_build} medoids"
    else:
        M0 = kmsynth.random_medoids(cfg)
        what = "random init (seed+1000) + FasterPAM (Alg.4, F1-F5) to convergence"
    t = time.time()
    r = oracle.fasterpam_run(D, M0)
    g = header(cfg, D, name, what)
    g["run"] = {"init": M0.tolist(), "trace": [[a, b, num(v), int(p)] for a, b, v, p in r.trace],
                "final": final_block(D, r), "oracle_s": round(time.time() - t, 1)}
    write(name, g)


JOBS = {
    "c2_fastpam1": lambda: job_build_fp1(2, "c2_fastpam1"),
    "c3_fastpam1": lambda: job_random(3, "c3_fastpam1", oracle.FASTPAM1),
    "c3_fastpam2": lambda: job_random(3, "c3_fastpam2", oracle.FASTPAM2, plan_iters=3),
    "c4_build": lambda: job_build_fp1(4, "c4_build", with_swap=False),
    "c4_fastpam1": job_c4_fastpam1,
    "c5_fastpam2": lambda: job_random(5, "c5_fastpam2", oracle.FASTPAM2, plan_iters=3, max_iter=3),
    "c3_fasterpam": lambda: job_fasterpam(3, "c3_fasterpam"),
    "c4_fasterpam": lambda: job_fasterpam(4, "c4_fasterpam", from_build="c4_build"),
}

if __name__ == "__main__":
    for j in sys.argv[1:] or list(JOBS):
        JOBS[j]()
