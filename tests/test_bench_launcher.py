"""bench.py --gpus N without torchrun relaunches itself as N ranks (one per
GPU) through torch.distributed.run on 127.0.0.1 with NCCL_DEBUG=INFO.  The
launch path is checked here on the CPU: --launcher-selftest makes every rank
join a gloo group and rank 0 report the world it saw."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_relaunches_n_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launcher-selftest"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["world_size"] == 2 and d["ranks_seen"] == 2 and d["n_gpus"] == 2
    assert d["nccl_debug"] == "INFO"
