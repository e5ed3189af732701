"""Host logic of the column-sharded path (paper_2008_05171_b200.parallel) on
the CPU: world_size-2 torch.distributed over gloo, with a mock shard whose
per-rank arithmetic comes from the oracle.  The real collectives, the
protocol order, the 16-byte record format and the column broadcast are the
product code; the result must equal the single-process oracle run exactly."""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from paper_2008_05171_b200 import parallel  # noqa: E402


def rand_int(rng, n, hi):
    A = rng.integers(0, hi, size=(n, n)).astype(np.uint32)
    A = np.triu(A, 1)
    A = A + A.T
    np.fill_diagonal(A, 0)
    return A


class MockShard:
    """Mirrors the CudaShard phase API on the CPU (int64 records)."""

    def __init__(self, D, rank, cb, k):
        self.D, self.rank, self.cb, self.k = D, rank, cb, k
        self.n = D.shape[0]
        self.c0, self.c1 = int(cb[rank]), int(cb[rank + 1])
        self._x = None
        self.exchange_tensors(len(cb) - 1)
        self.M = None
        self.td = 0

    def exchange_tensors(self, world):
        if self._x is None:
            self._x = (torch.zeros(16, dtype=torch.uint8), torch.zeros(16 * world, dtype=torch.uint8),
                       torch.zeros(4 * self.n, dtype=torch.uint8))
        return self._x

    def _write(self, v, slot, c):
        rec = np.zeros(16, np.uint8)
        rec[0:8] = np.array([v], np.int64).view(np.uint8)
        rec[8:12] = np.array([slot], np.int32).view(np.uint8)
        rec[12:16] = np.array([c], np.int32).view(np.uint8)
        self._x[0].copy_(torch.from_numpy(rec))

    def _recs(self):
        return parallel.decode_records(self._x[1].numpy(), np.int64)

    def _col(self):
        return self._x[2].numpy().view(np.uint32)

    # --- SWAP ---
    def shard_set_medoids(self, M, cols):
        self.M = [int(m) for m in M]
        self.MC = cols.numpy().view(np.uint32).reshape(self.k, self.n).copy()
        self.cache = oracle.assign_cols(self.MC)
        self.td = int(self.cache.dn.sum())
        self._status_reset()

    def shard_pack_column(self, c):
        assert self.c0 <= c < self.c1
        self._col()[:] = self.D[:, c]

    def shard_eval(self):
        R = oracle.removal_loss(self.cache, self.k)
        best = (np.iinfo(np.int64).max, 2**31 - 1, 2**31 - 1)
        for c in range(self.c0, self.c1):
            if c in self.M:
                continue
            vec, plus = oracle.fastpam1_candidate_col(self.D[:, c], self.cache, R)
            i = int(np.argmin(vec))
            best = min(best, (int(vec[i] + plus), i, c))
        self._write(*best)

    def shard_select(self, cb):
        v, slot, c = parallel.lexmin_records(self._recs())
        found = slot != 2**31 - 1 and v < 0
        owner = int(np.searchsorted(cb, c, side="right") - 1) if found else -1
        if found:
            self.M[slot] = c
            self.td += v
            self._pending = slot
        return found, slot, c, owner, v

    def shard_apply(self):
        self.MC[self._pending] = self._col()
        self.cache = oracle.assign_cols(self.MC)

    # --- device-decided iteration (sticky after convergence) ---
    column_dtype = "u32"

    def _status_reset(self):
        self._st = {"conv": False, "iters": 0, "swaps": 0, "trace": [], "apply": False}

    def shard_decide(self):
        st = self._st
        st["apply"] = False
        if not st["conv"]:
            v, slot, c = parallel.lexmin_records(self._recs())
            st["iters"] += 1
            if slot != 2**31 - 1 and v < 0:
                self.M[slot] = c
                self.td += v
                self._pending = slot
                st["apply"] = True
                st["swaps"] += 1
                st["trace"].append((slot, c, v))
            else:
                st["conv"] = True
        col = self._col()
        if st["apply"] and self.c0 <= self.M[self._pending] < self.c1:
            col[:] = self.D[:, self.M[self._pending]]
        else:
            col[:] = 0

    def shard_apply_async(self):
        if self._st["apply"]:
            self.shard_apply()

    def shard_status(self, wait=1):
        return self._st["conv"], self._st["iters"], self._st["swaps"], self.td

    def shard_trace(self):
        return list(self._st["trace"])

    # --- BUILD ---
    def build_eval(self, step):
        if step == 0:
            self.M = []
            self.dnear = None
        best = (np.iinfo(np.int64).max, 0, 2**31 - 1)
        for c in range(self.c0, self.c1):
            if c in self.M:
                continue
            col = self.D[:, c].astype(np.int64)
            if step == 0:
                g = int(col.sum() - col[c])
            else:
                d = col - self.dnear
                g = int(np.minimum(d, 0).sum())
            best = min(best, (g, 0, c))
        self._write(*best)

    def build_select(self, cb):
        g, _, c = parallel.lexmin_records(self._recs())
        owner = int(np.searchsorted(cb, c, side="right") - 1)
        self._pending = c
        self._gain = g
        return c, owner, g

    def build_decide(self, step):
        g, _, c = parallel.lexmin_records(self._recs())
        self._pending = c
        self._gain = g
        col = self._col()
        if self.c0 <= c < self.c1:
            col[:] = self.D[:, c]
        else:
            col[:] = 0

    def build_apply_async(self, step):
        self.build_apply(step)

    def get_state(self):
        import types
        return types.SimpleNamespace(medoids=np.asarray(self.M, np.int32))

    def build_apply(self, step):
        col = self._col().astype(np.int64)
        self.M.append(self._pending)
        if step == 0:
            self.dnear = col.copy()
        else:
            self.dnear = np.minimum(self.dnear, col)
        self.dnear[self.M] = 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, seed, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(seed)
        n, k = 57, 4
        D = rand_int(rng, n, 300)
        cb = parallel.column_bounds(n, world)
        comm = parallel.TorchComm()
        h = MockShard(D, rank, cb, k)
        M = parallel.build_async([h], comm, cb, k)                  # device-decided (all-reduce)
        chosen = parallel.build([h], comm, cb, k)                   # host-decided (broadcast)
        if [c for c, _ in chosen] != M:
            raise AssertionError("the two sharded BUILD protocols disagree")
        parallel.set_medoids([h], comm, cb, M, n)
        trace, iters, conv = parallel.run([h], comm, cb)            # device-decided (all-reduce)
        res = (M, trace, iters, conv, list(h.M), h.td)
        parallel.set_medoids([h], comm, cb, M, n)
        trace2, iters2, conv2 = parallel.run_sync([h], comm, cb)    # host-decided (broadcast)
        if (trace2, iters2, conv2, list(h.M), h.td) != res[1:]:
            raise AssertionError("the two sharded protocols disagree")
        q.put((rank,) + res)
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, "error", repr(e), 0, 0, 0, 0))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seed", [0, 1])
def test_gloo_world2_sharded_protocol_equals_oracle(seed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, seed, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=240) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda t: t[0])
    assert all(t[1] != "error" for t in out), out
    rng = np.random.default_rng(seed)
    D = rand_int(rng, 57, 300)
    Mb, _, _ = oracle.build_init(D, 4)
    ref = oracle.swap_run(D, Mb, oracle.FASTPAM1)
    for (rank, M, trace, iters, conv, Mf, td) in out:
        assert M == Mb.tolist()
        assert [(s, c, int(v)) for s, c, v in trace] == [(s, c, int(v)) for s, c, v in ref.trace]
        assert iters == ref.n_iter and conv
        assert Mf == ref.medoids.tolist() and td == ref.td


def test_column_bounds_and_records():
    cb = parallel.column_bounds(50000, 8)
    assert cb[0] == 0 and cb[-1] == 50000 and all(int(x) % 4 == 0 for x in cb[:-1])
    assert np.all(np.diff(cb) > 0)
    with pytest.raises(ValueError):
        parallel.column_bounds(3, 8)
    raw = np.zeros(32, np.uint8)
    raw[0:8] = np.array([-5], np.int64).view(np.uint8)
    raw[8:12] = np.array([2], np.int32).view(np.uint8)
    raw[12:16] = np.array([40], np.int32).view(np.uint8)
    raw[16:24] = np.array([-5], np.int64).view(np.uint8)
    raw[24:28] = np.array([1], np.int32).view(np.uint8)
    raw[28:32] = np.array([99], np.int32).view(np.uint8)
    recs = parallel.decode_records(raw, np.int64)
    assert recs == [(-5, 2, 40), (-5, 1, 99)]
    assert parallel.lexmin_records(recs) == (-5, 1, 99)     # smaller slot wins (reading R1)


class BufShard:
    """Only the FastPAM2 exchange buffers (CPU tensors), rank-tagged contents."""

    def __init__(self, rank, world, k, n):
        self.rank = rank
        colb = 4 * n
        self.x = (torch.full((16 * k,), rank + 1, dtype=torch.uint8), torch.zeros(16 * k * world, dtype=torch.uint8),
                  torch.zeros(k * colb, dtype=torch.uint8), torch.zeros(k * colb * world, dtype=torch.uint8), colb)
        for j in range(k):
            self.x[2][j * colb:(j + 1) * colb] = (10 * rank + j) % 251

    def fp2_exchange_tensors(self, world, need=0):
        return self.x


def _fp2_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        k, n, maxcnt = 5, 7, 3
        h = BufShard(rank, world, k, n)
        comm = parallel.TorchComm()
        comm.allgather_fp2_records([h])
        comm.allgather_fp2_columns([h], maxcnt)
        q.put((rank, h.x[1].numpy().copy(), h.x[3].numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_fp2_exchange_layout():
    """Records land in rank order; rank r's first maxcnt columns land at
    [r*maxcnt*colbytes, (r+1)*maxcnt*colbytes) -- the layout
    kmedoids_fp2_shard_plan's column indices assume."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_fp2_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted([q.get(timeout=120) for _ in ps], key=lambda t: t[0])
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    k, n, maxcnt, colb = 5, 7, 3, 28
    for rank, rec, cols in out:
        assert (rec[:16 * k] == 1).all() and (rec[16 * k:] == 2).all()
        for r in range(2):
            for j in range(maxcnt):
                blk = cols[(r * maxcnt + j) * colb:(r * maxcnt + j + 1) * colb]
                assert (blk == (10 * r + j) % 251).all()


class RoundShard:
    """Only the owner-side FastPAM2 round buffers (CPU tensors), rank-tagged."""

    def __init__(self, rank, world, stride):
        self.x = (torch.full((stride,), 7 + rank, dtype=torch.uint8), torch.zeros(stride * world, dtype=torch.uint8),
                  stride)
        self.x[0][:4] = torch.tensor([rank, 0, 0, 0], dtype=torch.uint8)

    def fp2_round_tensors(self, world):
        return self.x


def _round_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h = RoundShard(rank, world, 48)
        parallel.TorchComm().allgather_fp2_round([h])
        q.put((rank, h.x[1].numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_fp2_round_layout():
    """Owner-side rounds: rank r's round buffer (header + column) lands at
    [r*stride, (r+1)*stride) of every rank's receive buffer -- the layout
    k_fp2_round_apply reads -- and LocalComm (virtual ranks) does the same."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_round_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted([q.get(timeout=120) for _ in ps], key=lambda t: t[0])
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    local = [RoundShard(r, 3, 48) for r in range(3)]
    parallel.LocalComm(3).allgather_fp2_round(local)
    for got, world in [(out[0][1], 2), (out[1][1], 2), (local[0].x[1].numpy(), 3), (local[2].x[1].numpy(), 3)]:
        for r in range(world):
            blk = got[r * 48:(r + 1) * 48]
            assert blk[0] == r and (blk[4:] == 7 + r).all()


# ---------- FastCLARA from points over ranks (NEXT-3) ----------

def _oracle_runner(X, metric, k, samples, variant):
    t, j, M, _ = oracle.clara_points(X, metric, k, samples, variant)
    return M, t, j


def _clara_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(91)
        X = rng.integers(0, 400, size=(160, 3)).astype(np.int32)
        samples = np.stack([rng.choice(160, size=30, replace=False) for _ in range(5)])
        M, td, j = parallel.clara_points(X, "l1", 4, samples, parallel.TorchComm(), runner=_oracle_runner)
        q.put((rank, M.tolist(), int(td), j))
    except Exception as e:
        q.put((rank, "error", repr(e), 0))
        raise
    finally:
        dist.destroy_process_group()


def test_gloo_world2_clara_points_equals_oracle():
    """Samples split over 2 ranks (r, r+2, ...), one all-gather of (TD,
    sample, medoids): every rank returns oracle.clara_points over ALL samples."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_clara_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted([q.get(timeout=240) for _ in ps], key=lambda t: t[0])
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(t[1] != "error" for t in out), out
    rng = np.random.default_rng(91)
    X = rng.integers(0, 400, size=(160, 3)).astype(np.int32)
    samples = np.stack([rng.choice(160, size=30, replace=False) for _ in range(5)])
    t, j, M, _ = oracle.clara_points(X, "l1", 4, samples)
    for (rank, Mr, tr, jr) in out:
        assert (Mr, tr, jr) == (M.tolist(), int(t), j)
