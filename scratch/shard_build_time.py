"""Sharded BUILD timing on one rank (NCCL), device- vs host-decided protocol."""
import os, sys, time, torch, torch.distributed as dist
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import kmsynth
from paper_2008_05171_b200 import parallel
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
comm = parallel.TorchComm()
cfg = kmsynth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
n, k = cfg.n, cfg.k
cb = parallel.column_bounds(n, 1)
Dt = kmsynth.dist_cuda(kmsynth.make_points(cfg), cfg.metric, 0, n)
h = parallel.CudaShard(Dt, n, k, 0, cb, stream=torch.cuda.current_stream())
for name, fn in [("async", lambda: parallel.build_async([h], comm, cb, k)),
                 ("async", lambda: parallel.build_async([h], comm, cb, k)),
                 ("sync", lambda: [c for c, _ in parallel.build([h], comm, cb, k)])]:
    torch.cuda.synchronize(); t0 = time.perf_counter()
    M = fn()
    torch.cuda.synchronize()
    print(name, f"{(time.perf_counter() - t0) * 1e3:.1f} ms", M[:5], flush=True)
t0 = time.perf_counter()
for _ in range(200):
    comm.allgather_records([h])
torch.cuda.synchronize(); print("200 allgathers", f"{(time.perf_counter() - t0) * 1e3:.1f} ms")
t0 = time.perf_counter()
for _ in range(200):
    comm.allreduce_column([h])
torch.cuda.synchronize(); print("200 allreduces", f"{(time.perf_counter() - t0) * 1e3:.1f} ms")
dist.destroy_process_group()
