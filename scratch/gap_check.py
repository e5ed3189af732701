"""Measurement aid: the stream kernel's per-launch time (CUDA events on a side
branch of the iteration graph) back to back vs with idle gaps between
iterations -- is the ncu (isolated, cold) vs bench (sustained) gap thermal /
power?  usage: python scratch/gap_check.py [config]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kmsynth  # noqa: E402
from paper_2008_05171_b200 import KMedoids  # noqa: E402

try:
    import pynvml as nv
    nv.nvmlInit()
    hnd = nv.nvmlDeviceGetHandleByIndex(0)
except Exception:
    nv = None


def nvstat():
    if nv is None:
        return ""
    t = nv.nvmlDeviceGetTemperature(hnd, 0)
    p = nv.nvmlDeviceGetPowerUsage(hnd) / 1000
    c = nv.nvmlDeviceGetClockInfo(hnd, 1)
    m = nv.nvmlDeviceGetClockInfo(hnd, 2)
    try:
        mt = nv.nvmlDeviceGetFieldValues(hnd, [140])[0].value.uiVal   # NVML_FI_DEV_MEMORY_TEMP
    except Exception:
        mt = -1
    return f"gpuT={t}C memT={mt}C P={p:.0f}W sm={c} mem={m}"


cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = kmsynth.CONFIGS[cid]
X = kmsynth.make_points(cfg)
Dt = kmsynth.dist_cuda(X, cfg.metric)
st = torch.cuda.current_stream()
km = KMedoids(Dt, cfg.n, cfg.k, stream=st)
km.set_symmetric(True)
M0, _ = km.init_build()
for _ in range(3):
    km.swap_iter("fastpam1")
M1 = km.get_state().medoids


def run(mode, K=20):
    km.set_medoids(M1)
    km.swap_iters(2)
    km.set_profiling(True)
    km.stream_time(reset=True)
    torch.cuda.synchronize()
    s0 = nvstat()
    per = []
    if mode == "queued":
        km.swap_iters(K)
    else:
        for _ in range(K):
            if mode > 0:
                time.sleep(mode)
            km.stream_time(reset=True)
            km.swap_iter("fastpam1")
            ms, cnt = km.stream_time()
            per.append(ms / max(cnt, 1))
    torch.cuda.synchronize()
    ms, cnt = km.stream_time()
    km.set_profiling(False)
    if mode == "queued":
        avg = ms / max(cnt, 1)
        print(f"mode=queued K={K}: stream {avg:.4f} ms/launch | {s0} -> {nvstat()}", flush=True)
    else:
        per.sort()
        print(f"mode=sleep{mode} K={K}: stream median {per[len(per)//2]:.4f} min {per[0]:.4f} max {per[-1]:.4f} "
              f"| {s0} -> {nvstat()}", flush=True)


for mode in ["queued", 0, 0.002, 0.02, 0.2, "queued", 0.2, "queued"]:
    run(mode)
# long sustained run
run("queued", K=60)
run(0.5, K=10)
