#!/usr/bin/env python
"""FastPAM1 SWAP throughput on B200 (BASELINE.json metric).

One *step* is one SWAP iteration of the whole hot path (SURVEY 8(a) a2-a5:
sort + removal loss, the SWAP-delta stream, the argmin reduction, the swap
and the nearest/second update) over the config's dissimilarity matrix, which
is resident in HBM before the timed region starts.  BUILD (a7) and the
initial cache (a1) run once before it and are reported separately.

  metric: SWAP candidate-pair evals/s = k(n-k) per iteration / s per iteration
  default workload: C4 (n=50,000, k=200, float32 Euclidean, BUILD + FastPAM1)

Multi-GPU (torchrun, one rank per GPU): the column-sharded path of
paper_2008_05171_b200.parallel; the candidate pairs of all ranks count, time
is the max over ranks (strong scaling: n is fixed).

--impl reference times the CPU oracle (oracle/, single thread) on bounded
samples of the same workload (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def host_info():
    cores = len(os.sched_getaffinity(0))
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return cores, model


# ------------------------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg and --impl reference): Alg.3's inner loop for a sample
# of candidates.  D is exactly symmetric (kmsynth), so column c is materialised as row c.
# ------------------------------------------------------------------------------------------
def oracle_pairs_per_s(cfg, medoids, n_cand, min_seconds, rng, D_rows=None):
    import kmsynth
    import oracle
    X = kmsynth.make_points(cfg)
    n, k = cfg.n, cfg.k
    if D_rows is None:
        def rows(idx):
            return np.stack([kmsynth.dist_numpy(X, cfg.metric, int(c), int(c) + 1)[:, 0] for c in idx])
    else:
        rows = D_rows
    cols = rows(medoids)                                      # d(x_o, m_j) = d(m_j, x_o)
    cache = oracle.assign_cols(cols)
    R = oracle.removal_loss(cache, k)
    pool = np.setdiff1d(np.arange(n), medoids)
    cand = rng.choice(pool, size=n_cand, replace=False)
    C = rows(cand)
    done, t_used = 0, 0.0
    while True:
        for j in range(n_cand):
            t0 = time.perf_counter()
            oracle.fastpam1_candidate_col(C[j], cache, R)
            t_used += time.perf_counter() - t0
            done += 1
        if t_used >= min_seconds:
            break
    return done * k / t_used, done, t_used


def run_reference(args):
    import kmsynth
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = kmsynth.CONFIGS[args.config]
    cores, model = host_info()
    rng = np.random.default_rng(12345)
    M = kmsynth.random_medoids(cfg)
    X = kmsynth.make_points(cfg)

    def rows(idx):
        return np.stack([kmsynth.dist_numpy(X, cfg.metric, int(c), int(c) + 1)[:, 0] for c in idx])

    import oracle
    cols = rows(M)
    cache = oracle.assign_cols(cols)
    R = oracle.removal_loss(cache, cfg.k)
    pool = np.setdiff1d(np.arange(cfg.n), M)
    per_step = args.ref_candidates
    cand = rng.choice(pool, size=per_step, replace=False)
    C = rows(cand)
    times = []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        for j in range(per_step):
            oracle.fastpam1_candidate_col(C[j], cache, R)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = per_step * cfg.k * len(times) / tot
    sample = (f"{per_step} candidate columns x all n={cfg.n} objects per step (Alg.3 inner loop, oracle "
              f"fastpam1_candidate_col), random-init medoids, single thread")
    line = {
        "impl": "reference", "metric": "swap_pair_evals_per_s", "value": value, "unit": "pair-evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * tot / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64" if cfg.metric == kmsynth.L2_F32 else "int64", "data": "synthetic",
        "config": {"workload": f"{cfg.name} n={cfg.n} k={cfg.k} ({'f32 Euclidean' if cfg.metric else 'u32 L1'})",
                   "variant": "fastpam1"},
        "cpu_baseline": {"value": value, "unit": "pair-evals/s", "cores": 1, "kind": "oracle", "sample": sample,
                         "host_cores": cores, "cpu_model": model},
        "e2e": {"value": value, "unit": "pair-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "s_per_iteration_extrapolated": (cfg.n - cfg.k) / (value / cfg.k),
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import kmsynth
    from paper_2008_05171_b200 import KMedoids, kmedoids_run_host

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        from paper_2008_05171_b200 import parallel
        return parallel.bench_main(args)

    torch.cuda.set_device(0)
    cfg = kmsynth.CONFIGS[args.config]
    n, k = cfg.n, cfg.k
    peak, peak_kind = measured_peaks()
    t0 = time.perf_counter()
    X = kmsynth.make_points(cfg)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    km = KMedoids(Dt, n, k, stream=stream)

    # one-time initialisation (a1 / a7), timed separately
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(stream)
    if cfg.init == "build":
        M0, td0 = km.init_build()
    else:
        M0 = kmsynth.random_medoids(cfg)
        km.set_medoids(M0)
        td0 = km.get_state().td
    ev[1].record(stream)
    torch.cuda.synchronize()
    init_ms = ev[0].elapsed_time(ev[1])

    for _ in range(args.warmup):
        km.swap_iter(args.variant)
    km.set_profiling(True)
    km.stream_time(reset=True)
    st0 = km.get_state()
    launches0 = km.launch_count()
    swaps = 0
    torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        ev[2].record(stream)
        for _ in range(args.steps):
            conv, sw, td = km.swap_iter(args.variant)
            swaps += sw
        ev[3].record(stream)
        torch.cuda.synchronize()
        if (args.steps * 0.0) == 0 and clk.rows == []:
            time.sleep(0.3)
    total_ms = ev[2].elapsed_time(ev[3])
    k1_ms, k1_launches = km.stream_time(reset=True)
    launches = km.launch_count() - launches0
    st1 = km.get_state()
    ms_step = total_ms / args.steps
    pairs = k * (n - k)
    value = pairs / (ms_step / 1e3)
    alg_bytes = 4.0 * n * (n - k)
    k1_avg = k1_ms / max(1, k1_launches)
    achieved = alg_bytes / (k1_avg / 1e3) / 1e9
    clocks = clk.summary()

    # whole run to convergence from the same init (reported, not the headline)
    conv_iters = st1.n_iter

    # e2e: the public host-buffer call (H2D of D, init, SWAP to convergence, D2H of the result)
    e2e = None
    if not args.no_e2e:
        from paper_2008_05171_b200.kmedoids import pinned_empty
        Dh, Dh_t = pinned_empty(tuple(Dt.shape), cfg.dtype)
        Dh_t.copy_(Dt.cpu() if False else Dt, non_blocking=False)
        del km
        torch.cuda.empty_cache()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        r = kmedoids_run_host(Dh, k, use_build=(cfg.init == "build"),
                              medoids=None if cfg.init == "build" else kmsynth.random_medoids(cfg),
                              variant=args.variant)
        e2e_s = time.perf_counter() - t1
        e2e = {"value": r.n_iter * pairs / e2e_s, "unit": "pair-evals/s",
               "h2d_bytes_per_step": int(Dh.nbytes), "d2h_bytes_per_step": int(4 * (k + n) + 8),
               "job": f"kmedoids_run_host: H2D of D + {'BUILD' if cfg.init == 'build' else 'init'} + "
                      f"{r.n_iter} SWAP iterations to convergence + D2H of medoids/assignment/TD",
               "seconds": e2e_s, "n_iter": r.n_iter, "td": r.td}
        del Dh, Dh_t

    cpu = None
    if not args.no_cpu_baseline:
        rng = np.random.default_rng(7)
        Dc = Dt

        def rows(idx):
            t = Dc[torch.as_tensor(np.asarray(idx, np.int64), device=Dc.device)][:, :n].cpu().numpy()
            return t.view(np.uint32) if t.dtype == np.int32 else t
        pps, done, used = oracle_pairs_per_s(cfg, st0.medoids, args.cpu_candidates, args.cpu_seconds, rng,
                                             D_rows=rows)
        cores, model = host_info()
        cpu = {"value": pps, "unit": "pair-evals/s", "cores": 1, "kind": "oracle",
               "sample": f"{done} oracle candidate evaluations (Alg.3 inner loop over all n={n} objects, "
                         f"k={k}) on the state of the first timed iteration, single thread, {used:.1f} s",
               "host_cores": cores, "cpu_model": model}

    line = {
        "metric": "swap_pair_evals_per_s", "value": value, "unit": "pair-evals/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32->f64" if cfg.metric == kmsynth.L2_F32 else "u32->int64", "data": "synthetic",
        "config": {"workload": f"{cfg.name} n={n} k={k} ({'f32 Euclidean' if cfg.metric else 'u32 L1'}, "
                               f"{cfg.init} init, {args.variant})",
                   "n": n, "k": k, "variant": args.variant, "parallelism": "1 GPU",
                   "l2": f"inputs larger than L2 ({4 * n * n / 1e9:.1f} GB D vs 126 MB L2), no flush needed"},
        "s_per_iteration": ms_step / 1e3,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "kernel": "k_swap_stream", "kernel_ms": k1_avg,
                     "alg_bytes_per_launch": alg_bytes, "peak_kind": peak_kind},
        "stream_share": k1_ms / total_ms,
        "gpu_launches": launches,
        "clocks": clocks,
        "init": {"kind": cfg.init, "ms": init_ms, "td": td0},
        "timed_swaps": swaps, "iterations_seen": conv_iters,
        "datagen_s": gen_s,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--variant", default="fastpam1", choices=["fastpam1", "fastpam2"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--cpu-candidates", type=int, default=2000)
    ap.add_argument("--ref-candidates", type=int, default=400)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
