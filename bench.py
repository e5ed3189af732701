#!/usr/bin/env python
"""FastPAM SWAP throughput on B200 (BASELINE.json metric).

A *step* is one SWAP iteration of the whole hot path (SURVEY 8(a) a2-a5:
slot sort + removal loss, the SWAP-delta stream, the argmin reduction, the
swap and the nearest/second update; a6 for FastPAM2) over the config's
dissimilarity matrix, resident in HBM before the timed region starts.  BUILD
(a7) and the initial cache (a1) run once before and are reported separately.

  metric: SWAP candidate-pair evaluations per second = k(n-k) / s per iteration
  default workload: C4 (n=50,000, k=200, float32 Euclidean, BUILD + FastPAM1),
  the config BASELINE.json quotes at 1/2/4/8 GPUs that fits one GPU.

N > 1 (torchrun, one rank per GPU, NCCL): the column-sharded path of
paper_2008_05171_b200.parallel; candidate pairs of all ranks count, the time
is the max over ranks (strong scaling: n is fixed).

--impl reference times the CPU oracle (oracle/, one thread) on bounded
samples of the same workload (this tier's reference arm).
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
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region
    (NVML every 20 ms; nvidia-smi -lms as a fallback)."""
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu_index=0, period=0.02):
        self.gpu, self.period = gpu_index, period
        self.sm, self.max_sm, self.reasons = [], None, set()
        self._stop = threading.Event()
        self._t = None
        self._proc = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nvml = None

    def _run(self):
        p = self._nvml
        while not self._stop.is_set():
            try:
                self.sm.append(p.nvmlDeviceGetClockInfo(self._h, p.NVML_CLOCK_SM))
                mask = p.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self._nvml is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        else:
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            try:
                self._proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                               "--format=csv,noheader,nounits", "-lms", "50"],
                                              stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            except Exception:
                self._proc = None
        return self

    def __exit__(self, *a):
        if self._t is not None:
            self._stop.set()
            self._t.join(timeout=5)
        if self._proc is not None:
            self._proc.terminate()
            out, _ = self._proc.communicate(timeout=10)
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for line in out.splitlines():
                f = [x.strip() for x in line.split(",")]
                if len(f) < 6:
                    continue
                try:
                    self.sm.append(float(f[0]))
                    self.max_sm = float(f[1])
                except ValueError:
                    continue
                for i, nm in enumerate(names):
                    if f[2 + i] == "Active":
                        self.reasons.add(nm)

    def summary(self):
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None,
                "sm_max_mhz": self.max_sm, "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def committed_traffic(tag):
    """dram__bytes_read+write per launch of the stream kernel from the committed
    `ncu --set full` capture (profiles/r*_traffic.json), if one matches the workload."""
    import glob
    best = None
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json"))):
        try:
            d = json.load(open(p))
        except Exception:
            continue
        if tag in d:
            best = d[tag]
    return best


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


def workload_name(cfg, variant):
    metric = "f32 Euclidean" if cfg.metric else "u32 L1 x100"
    return f"{cfg.name} n={cfg.n} k={cfg.k} ({metric}, {cfg.init} init, {variant})"


# ------------------------------------------------------------------------------------------
# CPU oracle timing: Alg.3's inner loop (oracle.fastpam1_candidate_col) for a sample of
# candidates.  D is exactly symmetric (kmsynth), so column c is materialised as row c.
# ------------------------------------------------------------------------------------------
def oracle_rate(rows, medoids, pool, n_cand, min_seconds, rng, k):
    import oracle
    cache = oracle.assign_cols(rows(medoids))
    R = oracle.removal_loss(cache, k)
    cand = rng.choice(pool, size=min(n_cand, len(pool)), replace=False)
    C = rows(cand)
    done, used = 0, 0.0
    while True:
        for j in range(len(cand)):
            t0 = time.perf_counter()
            oracle.fastpam1_candidate_col(C[j], cache, R)
            used += time.perf_counter() - t0
            done += 1
        if used >= min_seconds:
            break
    return done * k / used, done, used


def run_reference(args):
    """The tier's reference arm: the CPU oracle as it stands, one host core."""
    import kmsynth
    import oracle
    if int(os.environ.get("RANK", "0")) != 0:
        return
    cfg = kmsynth.CONFIGS[args.config]
    cores, model = host_info()
    rng = np.random.default_rng(12345)
    M = kmsynth.random_medoids(cfg)
    X = kmsynth.make_points(cfg)

    def rows(idx):
        return np.stack([kmsynth.dist_numpy(X, cfg.metric, int(c), int(c) + 1)[:, 0] for c in idx])

    cache = oracle.assign_cols(rows(M))
    R = oracle.removal_loss(cache, cfg.k)
    pool = np.setdiff1d(np.arange(cfg.n), M)
    per_step = args.ref_candidates
    C = rows(rng.choice(pool, size=per_step, replace=False))
    times = []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        for j in range(per_step):
            oracle.fastpam1_candidate_col(C[j], cache, R)
        if s >= args.warmup:
            times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = per_step * cfg.k * len(times) / tot
    sample = (f"per step {per_step} candidates x all n={cfg.n} objects x k={cfg.k} slots (oracle "
              f"fastpam1_candidate_col = Alg.3 lines P:879-891), random-init medoids, 1 thread")
    line = {
        "impl": "reference", "metric": "swap_pair_evals_per_s", "value": value, "unit": "pair-evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * tot / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64" if cfg.metric == kmsynth.L2_F32 else "int64", "data": "synthetic",
        "config": {"workload": workload_name(cfg, args.variant), "n": cfg.n, "k": cfg.k},
        "cpu_baseline": {"value": value, "unit": "pair-evals/s", "cores": 1, "kind": "oracle", "sample": sample,
                         "host_cores": cores, "cpu_model": model},
        "e2e": {"value": value, "unit": "pair-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "s_per_iteration_extrapolated": cfg.k * (cfg.n - cfg.k) / value,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
def run_ours(args):
    import torch

    import kmsynth
    from paper_2008_05171_b200 import KMedoids, kmedoids_run_host

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1 or args.sharded:
        return run_sharded(args)

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
    km.set_symmetric(True)          # the config's D is exactly symmetric (verified on the device)

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
    init_ms_first = ev[0].elapsed_time(ev[1])     # first call: lazy module loading, allocations
    init_ms = init_ms_first
    if cfg.init == "build":
        # steady-state BUILD: the second call captures the step graph, the
        # third replays it (what every later BUILD of a handle costs); same medoids
        init_ms = []
        for _ in range(2):
            ev[0].record(stream)
            M1, _ = km.init_build()
            ev[1].record(stream)
            torch.cuda.synchronize()
            init_ms.append(ev[0].elapsed_time(ev[1]))
            if M1.tolist() != M0.tolist():
                raise SystemExit("BUILD is not deterministic across calls")
        init_ms = init_ms[-1]

    for _ in range(args.warmup):
        km.swap_iter(args.variant)
    stream_kernel = km.stream_kernel()
    st0 = km.get_state()
    km.set_profiling(True)
    km.stream_time(reset=True)
    launches0 = km.launch_count()
    swaps = 0
    torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        ev[2].record(stream)
        # K iterations queued back to back (kmedoids_swap_iters[_variant]: the
        # product's run path; each is a full pass, the host reads each outcome)
        conv, done, swaps, td = km.swap_iters(args.steps, args.variant)
        if done != args.steps:
            raise SystemExit(f"converged after {done} of {args.steps} timed steps; use fewer --steps")
        ev[3].record(stream)
        torch.cuda.synchronize()
    total_ms = ev[2].elapsed_time(ev[3])
    k1_ms, k1_launches = km.stream_time(reset=True)
    km.set_profiling(False)
    launches = km.launch_count() - launches0
    st1 = km.get_state()
    ms_step = total_ms / args.steps
    pairs = k * (n - k)
    value = pairs / (ms_step / 1e3)
    alg_bytes = 4.0 * n * (n - k)
    k1_avg = k1_ms / max(1, k1_launches)
    achieved = alg_bytes / (k1_avg / 1e3) / 1e9
    # per-iteration distribution (median, mean, count): a separate
    # pass after the timed region with events around every iteration
    # (only improving passes count: when the run converges it restarts from the
    # medoids the timed region started from)
    it_ms = []
    restarts = 0
    while len(it_ms) < min(args.steps, 30) and restarts < 30:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        conv, sw, _ = km.swap_iter(args.variant)
        b.record(stream)
        b.synchronize()
        if conv:
            km.set_medoids(st0.medoids)
            restarts += 1
            continue
        it_ms.append(a.elapsed_time(b))
    iteration_ms = {"median": float(np.median(it_ms)), "mean": float(np.mean(it_ms)), "min": float(np.min(it_ms)),
                    "max": float(np.max(it_ms)), "n": len(it_ms), "restarts": restarts,
                    "note": "events around each improving swap_iter call in a pass after the timed region "
                            "(restarted from the timed region's initial medoids on convergence)"}
    # a read-only stream over the same D in the same job (a second denominator)
    # the best of a plain 128-bit load stream and a TMA bulk-copy stream
    read_peak_ldg = kmsynth.read_peak_gbs(Dt, reps=5, stream=stream)
    read_peak_bulk = kmsynth.read_peak_bulk_gbs(Dt, reps=5, stream=stream)
    read_peak = max(read_peak_ldg, read_peak_bulk)

    # CPU oracle baseline on the state of the first timed iteration (rank 0, N=1 only)
    cpu = None
    if not args.no_cpu_baseline:
        def rows(idx):
            t = Dt[torch.as_tensor(np.asarray(idx, np.int64), device=Dt.device)][:, :n].cpu().numpy()
            return t.view(np.uint32) if t.dtype == np.int32 else t
        pool = np.setdiff1d(np.arange(n), st0.medoids)
        pps, done, used = oracle_rate(rows, st0.medoids, pool, args.cpu_candidates, args.cpu_seconds,
                                      np.random.default_rng(7), k)
        cores, model = host_info()
        cpu = {"value": pps, "unit": "pair-evals/s", "cores": 1, "kind": "oracle",
               "sample": f"{done} oracle candidate evaluations (Alg.3 P:879-891 over all n={n} objects and "
                         f"k={k} slots) on the state before the timed region, 1 thread, {used:.1f} s",
               "host_cores": cores, "cpu_model": model}

    # NEXT-1: FasterPAM (Alg.4, eager swaps) vs FastPAM1 to convergence from the
    # same initial medoids, D resident in HBM, CUDA events on the library's stream.
    fpm = None
    if not args.no_fasterpam:
        def to_converge(variant):
            km.set_medoids(M0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = km.run(use_build=False, variant=variant)
            e1.record(stream)
            torch.cuda.synchronize()
            return r, e0.elapsed_time(e1) / 1e3
        to_converge("fasterpam")                     # warm-up (allocations, first launches)
        to_converge("fastpam1_inc")
        rf, sf = to_converge("fasterpam")
        ri, si = to_converge("fastpam1_inc")
        r1, s1 = to_converge("fastpam1")
        fpm = {"variant": "fasterpam (Alg.4 P:988-1027, exact eager scan)", "s_to_converge": sf,
               "passes": rf.n_iter, "swaps": rf.n_swaps, "td": rf.td,
               "fastpam1_s_to_converge": s1, "fastpam1_iterations": r1.n_iter, "fastpam1_td": r1.td,
               "speedup_vs_fastpam1": s1 / sf,
               "fastpam1_incremental_s_to_converge": si, "fastpam1_incremental_iterations": ri.n_iter,
               "fastpam1_incremental_td": ri.td, "fastpam1_incremental_same_medoids":
                   bool(ri.medoids.tolist() == r1.medoids.tolist()),
               "start": "the initial medoids of the timed run (after " + cfg.init + ")"}

    # NEXT-2: the dissimilarity matrix of the config materialised by the product
    # (kmedoids_dissimilarity: tensor-core L2 / exact integer L1), written into
    # a second buffer of the same shape, CUDA events on the current stream.
    dis = None
    if not args.no_dissimilarity:
        from paper_2008_05171_b200 import kmedoids_dissimilarity
        metric = "l2" if cfg.metric == kmsynth.L2_F32 else "l1"
        Xt = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32 if metric == "l2" else np.int32)).cuda()
        D2 = torch.empty_like(Dt)
        kmedoids_dissimilarity(Xt, metric, D=D2)
        torch.cuda.synchronize()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        d0.record(stream)
        for _ in range(reps):
            kmedoids_dissimilarity(Xt, metric, D=D2)
        d1.record(stream)
        torch.cuda.synchronize()
        dms = d0.elapsed_time(d1) / reps
        wb = n * D2.stride(0) * 4
        diff = (float((D2[:, :n].double() - Dt[:, :n].double()).abs().max().item()) if metric == "l2"
                else int((D2[:, :n] != Dt[:, :n]).sum().item()))
        # write-only stream over the same bytes, same job (overwrites D2, checked above)
        wpeak = kmsynth.write_peak_gbs(D2, reps=3, stream=stream)
        dpad = (Xt.shape[1] + 7) // 8 * 8
        wgbs = wb / (dms / 1e3) / 1e9
        dis = {"metric": metric, "engine": "tcgen05 kind::tf32 (hi/lo split)" if metric == "l2" else "CUDA cores",
               "ms": dms, "bytes_written": wb, "write_GBps": wgbs,
               "frac_of_hbm_peak": wgbs / peak,
               "write_only_peak_same_job": wpeak, "frac_of_write_only_peak": wgbs / wpeak,
               "tensor_TFLOPs": (3 * 2 * n * n * dpad / (dms / 1e3) / 1e12) if metric == "l2" else None,
               "max_abs_diff_vs_generator" if metric == "l2" else "mismatches_vs_generator": diff}
        del D2, Xt
        torch.cuda.empty_cache()

    # NEXT-3: FastCLARA from the config's points (no n x n matrix): 5 samples of
    # s = 80 + 4k, BUILD + SWAP per sample, TD over all n from points
    clara = None
    if not args.no_clara:
        from paper_2008_05171_b200 import kmedoids_clara_points
        metric = "l2" if cfg.metric == kmsynth.L2_F32 else "l1"
        Xt = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32 if metric == "l2" else np.int32)).cuda()
        s_cl = min(n, 80 + 4 * k)
        crng = np.random.default_rng(cfg.seed + 2000)
        samples = np.stack([crng.choice(n, size=s_cl, replace=False) for _ in range(5)])
        clara = {"samples": 5, "s": s_cl, "input": "the config's points; no n x n matrix is formed",
                 "timing": "wall clock of the third identical call (host threads, one stream per sample)"}
        for v in ("fastpam1", "fasterpam"):
            for _ in range(2):
                kmedoids_clara_points(Xt, metric, k, samples, v)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            Mc, tdc, bc, _ = kmedoids_clara_points(Xt, metric, k, samples, v)
            clara[v] = {"ms": (time.perf_counter() - t1) * 1e3, "td": tdc, "best_sample": bc}
        if fpm:
            clara["td_of_pam_on_all_of_D"] = fpm["fastpam1_td"]
        del Xt

    # e2e: the public host-buffer call kmedoids_run_host (H2D of D, init, SWAP to
    # convergence, D2H of medoids/assignment/TD) -- one whole job per e2e step.
    e2e = None
    if not args.no_e2e:
        from paper_2008_05171_b200.kmedoids import pinned_empty
        Dh, Dh_t = pinned_empty(tuple(Dt.shape), cfg.dtype)
        Dh_t.copy_(Dt)
        init_M = None if cfg.init == "build" else kmsynth.random_medoids(cfg)
        km.close()
        del km
        torch.cuda.synchronize()
        torch.cuda.empty_cache()                 # the job allocates its own device memory
        # one untimed warm-up job (the first call allocates the device copy of
        # D and captures the iteration graphs: +50-60 ms, once per process),
        # then the whole job five times; the median job is reported
        kmedoids_run_host(Dh, k, use_build=(cfg.init == "build"), medoids=init_M, variant=args.variant)
        jobs = []
        for _ in range(5):
            t1 = time.perf_counter()
            r = kmedoids_run_host(Dh, k, use_build=(cfg.init == "build"), medoids=init_M, variant=args.variant)
            jobs.append(time.perf_counter() - t1)
        e2e_s = float(np.median(jobs))
        e2e = {"value": r.n_iter * pairs / e2e_s, "unit": "pair-evals/s", "jobs_s": jobs, "warmup_jobs": 1,
               "h2d_bytes_per_step": int(Dh.nbytes), "d2h_bytes_per_step": int(4 * (k + n) + 8),
               "job": f"kmedoids_run_host: H2D of D ({Dh.nbytes / 1e9:.1f} GB pinned) + "
                      f"{'BUILD' if cfg.init == 'build' else 'set medoids'} + {r.n_iter} SWAP iterations to "
                      f"convergence + D2H of medoids/assignment/TD", "seconds": e2e_s,
               "n_iter": r.n_iter, "n_swaps": r.n_swaps, "td": r.td}
        del Dh, Dh_t

    line = {
        "metric": "swap_pair_evals_per_s", "value": value, "unit": "pair-evals/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32->f64" if cfg.metric == kmsynth.L2_F32 else "u32->int64", "data": "synthetic",
        "config": {"workload": workload_name(cfg, args.variant), "n": n, "k": k, "variant": args.variant,
                   "parallelism": "1 GPU",
                   "l2": f"inputs larger than L2 ({4 * n * n / 1e9:.1f} GB D vs 126 MB L2), no flush needed"},
        "s_per_iteration": ms_step / 1e3,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": (committed_traffic(cfg.name) or {}).get("traffic_bytes"),
                     "traffic_source": (committed_traffic(cfg.name) or {}).get("source"),
                     "kernel": stream_kernel, "kernel_ms": k1_avg,
                     "alg_bytes_per_launch": alg_bytes, "peak_kind": peak_kind,
                     "read_only_peak_same_job": read_peak, "frac_of_read_only_peak": achieved / read_peak,
                     "read_only_peak_ldg": read_peak_ldg, "read_only_peak_bulk": read_peak_bulk,
                     "frac_of_nominal_7700": achieved / 7700.0},
        "iteration_ms": iteration_ms,
        "stream_share_of_step": k1_ms / total_ms,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "init": {"kind": cfg.init, "ms": init_ms, "ms_first_call": init_ms_first, "td": td0},
        "timed_swaps": swaps, "iterations_total": st1.n_iter, "td_after": st1.td,
        "datagen_s": gen_s,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "fasterpam": fpm,
        "dissimilarity": dis, "clara_points": clara,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# N > 1: column-sharded path (paper_2008_05171_b200.parallel), one rank per GPU over NCCL
# ------------------------------------------------------------------------------------------
def run_sharded(args):
    import torch
    import torch.distributed as dist

    import kmsynth
    from paper_2008_05171_b200 import parallel
    from paper_2008_05171_b200.kmedoids import pinned_empty

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    os.environ.setdefault("RANK", "0")
    os.environ.setdefault("WORLD_SIZE", "1")
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = parallel.TorchComm()
    cfg = kmsynth.CONFIGS[args.config]
    n, k = cfg.n, cfg.k
    cb = parallel.column_bounds(n, world)
    X = kmsynth.make_points(cfg)
    Dt = kmsynth.dist_cuda(X, cfg.metric, int(cb[rank]), int(cb[rank + 1]))
    fp2 = args.variant == "fastpam2"
    use_graph = not fp2 and not args.no_graph
    # the iteration graph is captured on the handle's stream, which must not be
    # the legacy default stream
    stream = torch.cuda.Stream() if use_graph else torch.cuda.current_stream()

    def job(D_slab):
        h = parallel.CudaShard(D_slab, n, k, rank, cb, stream=stream)
        if cfg.init == "build":
            parallel.build_async([h], comm, cb, k)
        else:
            parallel.set_medoids([h], comm, cb, kmsynth.random_medoids(cfg), n)
        return h

    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    h = job(Dt)
    torch.cuda.synchronize()
    init_s = comm.max_over_ranks(time.perf_counter() - t0)

    def step(hh):
        # FastPAM1: the device-decided iteration (no host round trip; the timed
        # region ends with a device synchronisation)
        if fp2:
            return parallel.fp2_iter([hh], comm, cb)
        parallel.swap_iter_async([hh], comm)
        return None

    for _ in range(args.warmup):
        step(h)
    graph, graph_err = None, None
    if use_graph:
        # FastPAM1: the whole device-decided iteration (eval, all-gather,
        # decide, all-reduce, apply) captured once with its NCCL calls and
        # replayed per step (parallel.IterationGraph); a capture the runtime
        # refuses falls back to the enqueued iteration (reported in the line)
        try:
            graph = parallel.IterationGraph([h], comm)
        except Exception as e:              # noqa: BLE001
            graph_err = f"{type(e).__name__}: {e}"[:300]
            print(f"[bench] iteration graph unavailable, enqueuing iterations: {graph_err}", file=sys.stderr)
            torch.cuda.synchronize()
    if graph is None:
        h.km.set_profiling(True)
        h.km.stream_time(reset=True)
    l0 = h.km.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    dist.barrier()
    with ClockSampler(local) as clk:
        e0.record(stream)
        if graph is not None:
            graph.replay(args.steps)
        else:
            for _ in range(args.steps):
                step(h)
        e1.record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    ms = comm.max_over_ranks(e0.elapsed_time(e1))
    if graph is not None:
        graph.resync()
        launches = args.steps * graph.kernels_per_iter[0]
        # the stream kernel's time: CUDA events around it over a few directly
        # enqueued iterations right after the timed replays (same state)
        h.km.set_profiling(True)
        h.km.stream_time(reset=True)
        for _ in range(3):
            step(h)
        torch.cuda.synchronize()
    else:
        launches = h.km.launch_count() - l0
    k1_ms, k1_n = h.km.stream_time(reset=True)
    k1_ms = comm.max_over_ranks(k1_ms)
    h.km.set_profiling(False)
    ms_step = ms / args.steps
    pairs = k * (n - k)
    value = pairs / (ms_step / 1e3)

    # e2e: every rank copies its slab from pinned host memory, then the whole
    # sharded job (init + SWAP to convergence) and the D2H of the result
    e2e = None
    if not args.no_e2e:
        Dh, Dh_t = pinned_empty(tuple(Dt.shape), cfg.dtype)
        Dh_t.copy_(Dt)
        h.km.close()
        del h
        torch.cuda.synchronize()
        dist.barrier()
        t1 = time.perf_counter()
        with torch.cuda.stream(stream):          # the handle's stream: the copy is ordered before its kernels
            Dd = Dh_t.to(Dt.device, non_blocking=True)
        h2 = job(Dd)
        if fp2:
            it = 0
            while it < 2000:
                it += 1
                if step(h2)[0]:
                    break
        else:
            _, it, _ = parallel.run([h2], comm, cb)
        st = h2.km.get_state()
        torch.cuda.synchronize()
        e2e_s = comm.max_over_ranks(time.perf_counter() - t1)
        e2e = {"value": it * pairs / e2e_s, "unit": "pair-evals/s", "h2d_bytes_per_step": int(Dh.nbytes) * world,
               "d2h_bytes_per_step": int(4 * (k + n) + 8),
               "job": f"every rank: H2D of its {Dh.nbytes / 1e9:.2f} GB slab (pinned) + {cfg.init} init + {it} SWAP "
                      f"iterations to convergence + D2H of medoids/assignment/TD; max over ranks",
               "seconds": e2e_s, "n_iter": it, "td": st.td}
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        # the oracle on this host, one core, on a bounded sample of the same
        # workload's candidates (columns of rank 0's slab, state after the run)
        st0 = h.km.get_state() if e2e is None else st
        own = np.arange(int(cb[0]), int(cb[1]))

        def rows(idx):
            loc = torch.as_tensor(np.asarray(idx, np.int64) - int(cb[0]), device=Dt.device)
            t = Dt[:, loc].T.contiguous().cpu().numpy()
            return t.view(np.uint32) if t.dtype == np.int32 else t
        medoid_rows = kmsynth.dist_numpy(X, cfg.metric, 0, n)[st0.medoids] if n <= 20000 else None
        if medoid_rows is None:
            medoid_rows = np.stack([kmsynth.dist_numpy(X, cfg.metric, int(m), int(m) + 1)[:, 0] for m in st0.medoids])
        import oracle
        cache = oracle.assign_cols(np.ascontiguousarray(medoid_rows))
        R = oracle.removal_loss(cache, k)
        pool = np.setdiff1d(own, st0.medoids)
        cand = np.random.default_rng(7).choice(pool, size=min(200, len(pool)), replace=False)
        C = rows(cand)
        t0 = time.perf_counter()
        for j in range(len(cand)):
            oracle.fastpam1_candidate_col(C[j], cache, R)
        used = time.perf_counter() - t0
        cores, model = host_info()
        cpu = {"value": len(cand) * k / used, "unit": "pair-evals/s", "cores": 1, "kind": "oracle",
               "sample": f"{len(cand)} oracle candidate evaluations (Alg.3 P:879-891 over all n={n} objects and "
                         f"k={k} slots) on rank 0 after the run, 1 thread, {used:.1f} s",
               "host_cores": cores, "cpu_model": model}
    if rank == 0:
        peak, peak_kind = measured_peaks()
        slab_bytes = 4.0 * n * (int(cb[1]) - int(cb[0]))
        ct = committed_traffic(cfg.name) or {}
        traffic = None
        if ct.get("traffic_bytes"):
            traffic = ct["traffic_bytes"] / (4.0 * n * (n - k)) * slab_bytes
        k1_avg = k1_ms / max(1, k1_n)
        ach = slab_bytes / (k1_avg / 1e3) / 1e9
        line = {"metric": "swap_pair_evals_per_s", "value": value, "unit": "pair-evals/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None,
                "dtype": "f32->f64" if cfg.metric == kmsynth.L2_F32 else "u32->int64", "data": "synthetic",
                "config": {"workload": workload_name(cfg, args.variant) + f", column-sharded over {world} GPUs",
                           "n": n, "k": k, "variant": args.variant, "parallelism": f"column-shard x{world}",
                           "l2": "inputs larger than L2, no flush needed"},
                "s_per_iteration": ms_step / 1e3,
                "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                             "traffic": traffic,
                             "traffic_source": (f"{ct.get('source')} (1-GPU launch) scaled to the rank-0 slab"
                                                if traffic else None),
                             "kernel": "k_swap_stream_seg2 (rank 0 slab)", "kernel_ms": k1_avg,
                             "alg_bytes_per_launch": slab_bytes, "peak_kind": peak_kind},
                "gpu_launches": launches, "iteration_graph": graph is not None, "iteration_graph_error": graph_err,
                "clocks": clk.summary(), "init": {"kind": cfg.init, "s": init_s},
                "e2e": e2e, "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def relaunch(n: int):
    """`bench.py --gpus N` started without torchrun: run the same command as N
    ranks (one per GPU) through torch.distributed.run on 127.0.0.1, with NCCL's
    INFO log (communicator / rank lines) on, and exit with its status."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    sys.stdout.flush()
    r = subprocess.run(cmd, env=env)
    sys.exit(r.returncode)


def launcher_selftest(args):
    """The N-rank launch path without GPUs: every rank joins a gloo group and
    contributes 1 to an all-reduce; rank 0 prints what it saw."""
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    t = torch.ones(1)
    dist.all_reduce(t)
    if dist.get_rank() == 0:
        print(json.dumps({"launcher_selftest": True, "n_gpus": args.gpus, "world_size": dist.get_world_size(),
                          "ranks_seen": int(t.item()), "nccl_debug": os.environ.get("NCCL_DEBUG")}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--variant", default="fastpam1", choices=["fastpam1", "fastpam2"])
    ap.add_argument("--sharded", action="store_true", help="use the column-sharded path even on 1 GPU")
    ap.add_argument("--no-graph", action="store_true",
                    help="sharded FastPAM1: enqueue every iteration instead of replaying its CUDA graph")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fasterpam", action="store_true")
    ap.add_argument("--no-dissimilarity", action="store_true")
    ap.add_argument("--no-clara", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--cpu-candidates", type=int, default=2000)
    ap.add_argument("--ref-candidates", type=int, default=400)
    ap.add_argument("--launcher-selftest", action="store_true",
                    help="only check the N-rank launch (gloo, CPU): rank 0 prints the world it saw")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch(args.gpus)                      # does not return
    if args.launcher_selftest:
        launcher_selftest(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
