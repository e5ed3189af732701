"""Column-sharded multi-GPU SWAP / BUILD.

Rank r of R holds the column slab [cb[r], cb[r+1]) of the n x n matrix D
(all n rows): its candidates are those columns.  Every rank keeps the full
nearest/second cache and the k medoid columns MC (replicated), so after the
one exchange per step every rank updates its own copy and no symmetry of D
is needed.  One SWAP iteration (FastPAM1, Alg.3) is:

  1. kmedoids_shard_eval      local stream over the slab -> 16-byte record (dTD, slot, c)
  2. all-gather the R records (NCCL over NVLink; 16*R bytes)
  3. kmedoids_shard_select    identical lexicographic min on every rank (reading R1)
  4. owner of c*: kmedoids_shard_pack_column; broadcast the n-element column
  5. kmedoids_shard_apply     M, TD and the nearest/second cache (identical on every rank)

``swap_iter_async`` / ``run`` use the device-decided form instead: the
lexicographic min is taken on the device (kmedoids_shard_decide), the owner
packs column c* and every other rank zeros, and one SUM all-reduce of the
column buffers delivers c* everywhere -- no host round trip inside an
iteration, so the host keeps one iteration queued ahead of the one whose
status it reads (the decision is sticky after convergence, so the extra
iteration changes and counts nothing).

BUILD (Alg.1) uses the same gather / pack / broadcast pattern per step.

The protocol is written once over ``handles`` (the shard handles this process
drives) and a ``comm``:
  * ``TorchComm``  one handle per process, torch.distributed (nccl on GPUs,
                    gloo for the CPU tests of this host logic);
  * ``LocalComm``  all R handles in one process (virtual ranks on one GPU,
                    sequential, no kernels waiting on each other).
The exchange buffers are whatever ``h.exchange_tensors(R)`` returns (device
memory owned by the library handle for the CUDA path).
"""
from __future__ import annotations

import os
import time

import numpy as np

RECORD_BYTES = 16


def column_bounds(n: int, world: int) -> np.ndarray:
    """Contiguous column slabs: rank r owns [cb[r], cb[r+1]) (multiples of 4 except the last)."""
    cb = np.zeros(world + 1, np.int64)
    for r in range(1, world):
        cb[r] = min(n, (r * n // world + 3) // 4 * 4)
    cb[world] = n
    if np.any(np.diff(cb) <= 0):
        raise ValueError(f"n={n} too small for {world} ranks")
    return cb


def decode_records(raw: np.ndarray, acc_dtype) -> list:
    """(R*16,) uint8 -> [(v, slot, c)] in rank order."""
    R = raw.size // RECORD_BYTES
    rec = raw.reshape(R, RECORD_BYTES)
    v = rec[:, 0:8].copy().view(acc_dtype).ravel()
    slot = rec[:, 8:12].copy().view(np.int32).ravel()
    c = rec[:, 12:16].copy().view(np.int32).ravel()
    return [(v[r].item(), int(slot[r]), int(c[r])) for r in range(R)]


def lexmin_records(recs):
    """Reading R1: the lexicographic minimum of (dTD, slot, candidate)."""
    return min(recs, key=lambda t: (t[0], t[1], t[2]))


def column_view(col, dtype: str):
    """The exchange column (uint8 bytes) as float32 ("f32") or int32 ("u32":
    the uint32 bits; a SUM with zeros leaves them unchanged)."""
    import torch
    return col.view(torch.float32 if dtype == "f32" else torch.int32)


def on_handle_stream(handles):
    """Context in which a collective or copy over the handles' exchange
    buffers is enqueued on the library handle's CUDA stream (the stream the
    shard kernels that produce and consume those buffers run on), so it is
    ordered with them whatever torch's current stream is.  CPU (mock) handles:
    no-op."""
    import contextlib
    km = getattr(handles[0], "km", None)
    if km is None or getattr(km, "stream", None) is None:
        return contextlib.nullcontext()
    import torch
    return torch.cuda.stream(km.stream)


def _streamed(method):
    def wrapper(self, handles, *a, **kw):
        with on_handle_stream(handles):
            return method(self, handles, *a, **kw)
    wrapper.__name__ = method.__name__
    wrapper.__doc__ = method.__doc__
    return wrapper


class LocalComm:
    """All ranks' handles in one process (virtual ranks)."""

    def __init__(self, world: int):
        self.world = world

    @_streamed
    def allgather_records(self, handles):
        xs = [h.exchange_tensors(self.world) for h in handles]
        cat = [x[0] for x in xs]
        for (send, recv, col) in xs:
            for r, s in enumerate(cat):
                recv[r * RECORD_BYTES:(r + 1) * RECORD_BYTES].copy_(s)

    @_streamed
    def broadcast_column(self, handles, owner: int):
        xs = [h.exchange_tensors(self.world) for h in handles]
        src = xs[owner][2]
        for r, (_, _, col) in enumerate(xs):
            if r != owner:
                col.copy_(src)

    @_streamed
    def allreduce_column(self, handles):
        xs = [h.exchange_tensors(self.world) for h in handles]
        cols = [column_view(x[2], h.column_dtype) for x, h in zip(xs, handles)]
        tot = cols[0].clone()
        for c in cols[1:]:
            tot += c
        for c in cols:
            c.copy_(tot)

    @_streamed
    def allgather_fp2_records(self, handles):
        xs = [h.fp2_exchange_tensors(self.world) for h in handles]
        nb = xs[0][0].numel()
        for x in xs:
            for r, y in enumerate(xs):
                x[1][r * nb:(r + 1) * nb].copy_(y[0])

    @_streamed
    def allgather_fp2_columns(self, handles, maxcnt: int):
        xs = [h.fp2_exchange_tensors(self.world) for h in handles]
        cb = xs[0][4] * maxcnt                     # bytes per rank
        for x in xs:
            for r, y in enumerate(xs):
                x[3][r * cb:(r + 1) * cb].copy_(y[2][:cb])

    @_streamed
    def allgather_fp2_round(self, handles):
        xs = [h.fp2_round_tensors(self.world) for h in handles]
        for x in xs:
            for r, y in enumerate(xs):
                x[1][r * y[2]:(r + 1) * y[2]].copy_(y[0])

    def max_over_ranks(self, x: float) -> float:
        return x


class TorchComm:
    """One handle per process; torch.distributed collectives (nccl or gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    @_streamed
    def allgather_records(self, handles):
        (h,) = handles
        send, recv, _ = h.exchange_tensors(self.world)
        self.dist.all_gather_into_tensor(recv, send, group=self.group)

    @_streamed
    def broadcast_column(self, handles, owner: int):
        (h,) = handles
        _, _, col = h.exchange_tensors(self.world)
        self.dist.broadcast(col, src=owner, group=self.group)

    @_streamed
    def allreduce_column(self, handles):
        (h,) = handles
        _, _, col = h.exchange_tensors(self.world)
        self.dist.all_reduce(column_view(col, h.column_dtype), op=self.dist.ReduceOp.SUM, group=self.group)

    @_streamed
    def allgather_fp2_records(self, handles):
        (h,) = handles
        send, recv, _, _, _ = h.fp2_exchange_tensors(self.world)
        self.dist.all_gather_into_tensor(recv, send, group=self.group)

    @_streamed
    def allgather_fp2_columns(self, handles, maxcnt: int):
        (h,) = handles
        _, _, csend, crecv, colb = h.fp2_exchange_tensors(self.world)
        cb = colb * maxcnt
        self.dist.all_gather_into_tensor(crecv[:cb * self.world], csend[:cb], group=self.group)

    @_streamed
    def allgather_fp2_round(self, handles):
        (h,) = handles
        send, recv, _ = h.fp2_round_tensors(self.world)
        self.dist.all_gather_into_tensor(recv, send, group=self.group)

    def allgather_object(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def max_over_ranks(self, x: float) -> float:
        import torch
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())


# ---------------------------------------------------------------------------
# the protocol (identical on every rank)
# ---------------------------------------------------------------------------
def set_medoids(handles, comm, cb, medoids, n: int):
    """Gather the k medoid columns from their owners (k broadcasts) and set them."""
    import torch
    M = np.asarray(medoids, dtype=np.int64)
    k = len(M)
    cols = []
    for h in handles:
        _, _, col = h.exchange_tensors(comm.world)
        cols.append(torch.empty((k, col.numel()), dtype=col.dtype, device=col.device))
    for j, m in enumerate(M):
        owner = int(np.searchsorted(cb, m, side="right") - 1)
        for h in handles:
            if h.rank == owner:
                h.shard_pack_column(int(m))
        comm.broadcast_column(handles, owner)
        with on_handle_stream(handles):          # ordered with the pack / set kernels
            for h, buf in zip(handles, cols):
                buf[j].copy_(h.exchange_tensors(comm.world)[2])
    for h, buf in zip(handles, cols):
        h.shard_set_medoids(M.astype(np.int32), buf)


def swap_iter(handles, comm, cb):
    """One sharded FastPAM1 SWAP iteration; returns (converged, (slot, c, dTD) or None)."""
    for h in handles:
        h.shard_eval()
    comm.allgather_records(handles)
    sel = [h.shard_select(cb) for h in handles]
    found, slot, cand, owner, dtd = sel[0]
    if any(s != sel[0] for s in sel):
        raise RuntimeError(f"ranks disagree on the swap: {sel}")
    if not found:
        return True, None
    for h in handles:
        if h.rank == owner:
            h.shard_pack_column(cand)
    comm.broadcast_column(handles, owner)
    for h in handles:
        h.shard_apply()
    return False, (slot, cand, dtd)


def build(handles, comm, cb, k: int):
    """Sharded PAM BUILD (Alg.1): k steps of local eval / gather / select / broadcast."""
    chosen = []
    for step in range(k):
        for h in handles:
            h.build_eval(step)
        comm.allgather_records(handles)
        sel = [h.build_select(cb) for h in handles]
        cand, owner, gain = sel[0]
        if any(s != sel[0] for s in sel):
            raise RuntimeError(f"ranks disagree on the BUILD step: {sel}")
        for h in handles:
            if h.rank == owner:
                h.shard_pack_column(cand)
        comm.broadcast_column(handles, owner)
        for h in handles:
            h.build_apply(step)
        chosen.append((cand, gain))
    return chosen


def build_async(handles, comm, cb, k: int):
    """Sharded BUILD with the decisions on the device (no host round trip in
    any step); returns the chosen medoids (identical on every rank)."""
    for step in range(k):
        for h in handles:
            h.build_eval(step)
        comm.allgather_records(handles)
        for h in handles:
            h.build_decide(step)
        comm.allreduce_column(handles)
        for h in handles:
            h.build_apply_async(step)
    Ms = [h.get_state().medoids.tolist() for h in handles]
    if any(m != Ms[0] for m in Ms):
        raise RuntimeError(f"ranks disagree on the BUILD medoids: {Ms}")
    return Ms[0]


FP2_MODES = ("gather", "owner")


def fp2_iter(handles, comm, cb, mode: str = "gather"):
    """One sharded FastPAM2 iteration (reading R6); returns (converged, swaps).

    per-slot bests of the local candidates -> all-gather (k*16 B per rank) ->
    identical plan on every rank, then the sequential phase:

    * ``owner``: rounds of owner-side re-evaluation
      (kmedoids_fp2_round_eval: each rank re-checks its own plan entries on
      the current state and publishes its first improving one with its
      column) -> all-gather of the round buffers -> every rank applies the
      published entry with the smallest plan position
      (kmedoids_fp2_round_apply).  Rounds = applied swaps + 1; one column
      per applied swap crosses the interconnect.
    * ``gather`` (default): all-gather of the columns of the planned
      candidates (distinct candidates only; each rank sends the ones it
      owns), then every rank runs the whole sequential phase redundantly on
      the gathered columns.

    Both give the single-GPU trace.  Measured on virtual ranks (C5 / C3,
    G = 8): the planned slots share few distinct
    candidates (2-3 columns per rank), so ``gather`` moves 6-10 MB per rank
    in one collective while ``owner`` needs swaps + 1 collectives and host
    round trips per iteration -- ``gather`` is the default; ``owner`` moves
    one column per applied swap, the better choice when the plan names many
    distinct candidates."""
    if mode not in FP2_MODES:
        raise ValueError(f"mode must be one of {FP2_MODES}")
    for h in handles:
        h.fp2_exchange_tensors(comm.world)      # sizes the exchange buffers once
        h.fp2_shard_eval()
    comm.allgather_fp2_records(handles)
    plans = [h.fp2_shard_plan(cb) for h in handles]
    m, maxcnt = plans[0]
    if any(p != plans[0] for p in plans):
        raise RuntimeError(f"ranks disagree on the FastPAM2 plan: {plans}")
    if m > 0 and mode == "owner":
        while True:
            for h in handles:
                h.fp2_round_eval()
            comm.allgather_fp2_round(handles)
            res = [h.fp2_round_apply() for h in handles]
            if any(r != res[0] for r in res):
                raise RuntimeError(f"ranks disagree on a FastPAM2 round: {res}")
            more, swaps, _ = res[0]
            if not more:
                return False, swaps
    if m > 0:
        for h in handles:                       # the column buffers grow on demand (kmedoids.h)
            h.fp2_exchange_tensors(comm.world, need=maxcnt)
        comm.allgather_fp2_columns(handles, maxcnt)
    res = [h.fp2_shard_apply() for h in handles]
    if any(r[:2] != res[0][:2] for r in res):
        raise RuntimeError(f"ranks disagree on the FastPAM2 swaps: {res}")
    conv, swaps, td = res[0]
    return conv, swaps


def run_sync(handles, comm, cb, max_iter: int = 2000):
    """The host-decided protocol (swap_iter) to convergence: same result as run()."""
    trace = []
    it = 0
    while it < max_iter:
        it += 1
        conv, sw = swap_iter(handles, comm, cb)
        if conv:
            return trace, it, True
        trace.append(sw)
    return trace, it, False


def swap_iter_async(handles, comm):
    """One device-decided sharded FastPAM1 iteration, enqueued (no host sync)."""
    for h in handles:
        h.shard_eval()
    comm.allgather_records(handles)
    for h in handles:
        h.shard_decide()
    comm.allreduce_column(handles)
    for h in handles:
        h.shard_apply_async()


def status(handles, comm, wait: int = 1):
    """(converged, n_iter, n_swaps, td) -- identical on every rank (checked here)."""
    st = [h.shard_status(wait) for h in handles]
    if any(s != st[0] for s in st):
        raise RuntimeError(f"ranks disagree on the run status: {st}")
    return st[0]


def run(handles, comm, cb, max_iter: int = 2000):
    """Sharded FastPAM1 to convergence: iterations enqueued one ahead of the
    status the host inspects.  Returns (trace [(slot, c, dTD)], n_iter, converged)."""
    enq = 0
    conv, it = False, 0
    while enq < max_iter:
        swap_iter_async(handles, comm)
        enq += 1
        conv, it, _, _ = status(handles, comm, wait=2)     # the iteration before the last one
        if conv:
            break
    if not conv:
        conv, it, _, _ = status(handles, comm, wait=1)
    traces = [h.shard_trace() for h in handles]
    if any(t != traces[0] for t in traces):
        raise RuntimeError("ranks disagree on the swap trace")
    return traces[0], it, conv


class IterationGraph:
    """The device-decided sharded FastPAM1 iteration (eval -> all-gather ->
    decide -> all-reduce -> apply, swap_iter_async) captured ONCE into a CUDA
    graph together with its collectives, then replayed per iteration: one
    graph launch instead of ~10 kernel launches and two collective calls per
    iteration.  The state lives on the device (the decision is sticky after
    convergence), so replaying the same graph K times is K iterations.

    The handles must share one non-default stream (capture cannot run on the
    legacy default stream); profiling is switched off (its event ring is
    host-side bookkeeping).  The capture itself executes nothing; resync()
    after the replays brings the library's host-side counters up to date
    (kmedoids_shard_resync) before status() / shard_trace().  Collectives:
    any comm whose calls are stream-ordered on the handle stream
    (LocalComm copies, TorchComm over NCCL)."""

    def __init__(self, handles, comm):
        import torch
        st = handles[0].km.stream
        if any(h.km.stream != st for h in handles):
            raise ValueError("all handles of the graph must run on one stream")
        if st == torch.cuda.default_stream(st.device):
            raise ValueError("capture needs the handles on a non-default stream (KMedoids(..., stream=...))")
        for h in handles:
            # decide steps since the last set_medoids / BUILD (syncs the stream)
            if getattr(h, "_x", None) is None or h.km.shard_resync() == 0:
                raise ValueError("run one sharded iteration (swap_iter_async) before the capture: the exchange "
                                 "buffers and the library's scratch are allocated on first use")
            h.km.set_profiling(False)
        self.handles = handles
        self.stream = st
        l0 = [h.km.launch_count() for h in handles]
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=st, capture_error_mode="thread_local"):
            swap_iter_async(handles, comm)
        # kernels of one iteration per handle (the capture counted them once)
        self.kernels_per_iter = [h.km.launch_count() - a for h, a in zip(handles, l0)]

    def replay(self, count: int = 1):
        import torch
        with torch.cuda.stream(self.stream):      # CUDAGraph.replay launches on the current stream
            for _ in range(count):
                self.graph.replay()

    def resync(self):
        """Host bookkeeping after replays; returns the decide steps per handle."""
        return [h.km.shard_resync() for h in self.handles]


def run_graph(handles, comm, graph: IterationGraph, max_iter: int = 2000, chunk: int = 8):
    """Sharded FastPAM1 to convergence by graph replays, `chunk` iterations
    between status checks (iterations after convergence are no-ops).
    Returns (trace, n_iter, converged) as run()."""
    conv, it, done = False, 0, 0
    while done < max_iter and not conv:
        c = min(chunk, max_iter - done)
        graph.replay(c)
        done += c
        graph.resync()
        conv, it, _, _ = status(handles, comm, wait=1)
    traces = [h.shard_trace() for h in handles]
    if any(t != traces[0] for t in traces):
        raise RuntimeError("ranks disagree on the swap trace")
    return traces[0], it, conv


# ---------------------------------------------------------------------------
# CUDA shard handle: KMedoids on a column slab + exchange tensors
# ---------------------------------------------------------------------------
class _DevBytes:
    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


class CudaShard:
    """A KMedoids handle on columns [cb[rank], cb[rank+1]) of D."""

    def __init__(self, D_slab, n: int, k: int, rank: int, cb, stream=None):
        from .kmedoids import KMedoids
        self.rank = rank
        self.km = KMedoids(D_slab, n, k, int(cb[rank]), int(cb[rank + 1]), stream=stream)
        self._x = None

    def exchange_tensors(self, world: int):
        import torch
        if self._x is None:
            x = self.km.shard_exchange(world)
            dev = self.km.D.device
            send = torch.as_tensor(_DevBytes(x.record_send, x.record_bytes), device=dev)
            recv = torch.as_tensor(_DevBytes(x.record_recv, x.record_bytes * world), device=dev)
            col = torch.as_tensor(_DevBytes(x.column, x.column_bytes), device=dev)
            self._x = (send, recv, col)
        return self._x

    def fp2_exchange_tensors(self, world: int, need: int = 0):
        """(record_send, record_recv, col_send, col_recv, bytes per column) as
        uint8 tensors; re-queried when a plan needs more columns per rank than
        the buffers held (the library grew them)."""
        import torch
        if getattr(self, "_f2", None) is None or need > getattr(self, "_f2_cap", 0):
            x = self.km.fp2_shard_exchange(world)
            self._f2_cap = int(x.col_capacity)
            dev = self.km.D.device
            cap = x.col_capacity * x.col_bytes_per_column
            self._f2 = (torch.as_tensor(_DevBytes(x.record_send, x.record_bytes), device=dev),
                        torch.as_tensor(_DevBytes(x.record_recv, x.record_bytes * world), device=dev),
                        torch.as_tensor(_DevBytes(x.col_send, cap), device=dev),
                        torch.as_tensor(_DevBytes(x.col_recv, cap * world), device=dev),
                        int(x.col_bytes_per_column))
        return self._f2

    def fp2_round_tensors(self, world: int):
        """(round send, round recv, stride) of the owner-side FastPAM2 rounds
        as uint8 tensors (kmedoids_fp2_round_buffers)."""
        import torch
        if getattr(self, "_f2r", None) is None:
            sp, rp, stride = self.km.fp2_round_buffers()
            dev = self.km.D.device
            self._f2r = (torch.as_tensor(_DevBytes(sp, stride), device=dev),
                         torch.as_tensor(_DevBytes(rp, stride * world), device=dev), stride)
        return self._f2r

    @property
    def column_dtype(self) -> str:
        from .kmedoids import KM_U32
        return "u32" if self.km.dtype == KM_U32 else "f32"

    def __getattr__(self, name):       # shard_eval, shard_select, ... -> the handle
        return getattr(self.km, name)


# ---------------------------------------------------------------------------
# FastCLARA from points over several GPUs (NEXT-3; "CLARA can be
# trivially parallelized")
# ---------------------------------------------------------------------------
def clara_points(X, metric: str, k: int, samples, comm, variant: str = "fastpam1", runner=None):
    """Samples are independent units: rank r runs samples r, r + R, ... on its
    GPU (kmedoids_clara_points over its share; X replicated, no D anywhere),
    then one all-gather of (TD, sample index, medoids) per rank and every rank
    takes the same smallest (TD, sample index).  No data-path collective other
    than that one small exchange.  Returns (medoids, TD, best sample index).

    ``runner(X, metric, k, samples, variant) -> (medoids, TD, local best)``
    defaults to the CUDA library call (the CPU tests pass their own)."""
    if runner is None:
        from .kmedoids import kmedoids_clara_points

        def runner(X_, m_, k_, s_, v_):
            M, td, b, _ = kmedoids_clara_points(X_, m_, k_, s_, v_)
            return M, td, b
    samples = np.asarray(samples)
    mine = list(range(comm.rank, len(samples), comm.world))
    rec = None
    if mine:
        M, td, b = runner(X, metric, k, samples[mine], variant)
        rec = (td, mine[b], [int(x) for x in M])
    recs = [r for r in comm.allgather_object(rec) if r is not None]
    td, j, M = min(recs, key=lambda r: (r[0], r[1]))
    return np.asarray(M, np.int32), td, j
