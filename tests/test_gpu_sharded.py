"""Column-sharded path on one GPU with virtual ranks (LocalComm, sequential,
no kernels waiting on each other): R handles on the column slabs of one
matrix must reproduce the single-GPU result bit for bit on integer data."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import kmsynth  # noqa: E402
import oracle  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def shards(Dt, n, k, world):
    from paper_2008_05171_b200 import parallel
    cb = parallel.column_bounds(n, world)
    hs = [parallel.CudaShard(Dt[:, int(cb[r]):], n, k, r, cb) for r in range(world)]
    return hs, cb


@pytest.mark.parametrize("world,cid,n,k", [(2, 1, 500, 5), (3, 1, 500, 5), (4, 5, 1200, 9), (2, 4, 900, 7),
                                            (1, 4, 900, 7)])
def test_sharded_build_and_swap_equal_single_gpu(world, cid, n, k):
    from paper_2008_05171_b200 import KMedoids, parallel
    cfg = kmsynth.CONFIGS[cid]
    X = kmsynth.make_points(cfg, n=n)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    single = KMedoids(Dt, n, k)
    Mb, tdb = single.init_build()
    tr1 = []
    while True:
        conv, sw, td = single.swap_iter()
        tr1 += single.last_swaps()
        if conv:
            break
    st1 = single.get_state()
    hs, cb = shards(Dt, n, k, world)
    comm = parallel.LocalComm(world)
    chosen = parallel.build(hs, comm, cb, k)
    assert [c for c, _ in chosen] == Mb.tolist()
    tdb = [h.km.get_state().td for h in hs]
    assert parallel.build_async(hs, comm, cb, k) == Mb.tolist()       # device-decided BUILD
    assert [h.km.get_state().td for h in hs] == tdb
    trace, iters, conv = parallel.run(hs, comm, cb)
    assert conv and iters == st1.n_iter
    for h in hs:
        assert h.km.get_state().n_iter == st1.n_iter
    if cfg.metric == kmsynth.L1_INT:
        assert [(s, c, int(v)) for s, c, v in trace] == [(s, c, int(v)) for s, c, v in tr1]
    else:
        assert [(s, c) for s, c, v in trace] == [(s, c) for s, c, v in tr1]
    for h in hs:
        st = h.km.get_state()
        assert st.medoids.tolist() == st1.medoids.tolist()
        assert st.assignment.tolist() == st1.assignment.tolist()
        if cfg.metric == kmsynth.L1_INT:
            assert st.td == st1.td
        else:
            assert st.td == pytest.approx(st1.td, rel=1e-12)
    if cfg.metric == kmsynth.L1_INT:
        D = kmsynth.as_numpy_D(Dt)[:, :n]
        ref = oracle.swap_run(D, Mb, oracle.FASTPAM1)
        assert st1.medoids.tolist() == ref.medoids.tolist() and st1.td == ref.td


def test_sharded_random_init_set_medoids():
    from paper_2008_05171_b200 import parallel
    cfg = kmsynth.CONFIGS[5]
    n, k, world = 800, 12, 3
    X = kmsynth.make_points(cfg, n=n)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    D = kmsynth.as_numpy_D(Dt)[:, :n]
    M0 = kmsynth.random_medoids(cfg, k=k, n=n)
    ref = oracle.swap_run(D, M0, oracle.FASTPAM1)
    hs, cb = shards(Dt, n, k, world)
    comm = parallel.LocalComm(world)
    parallel.set_medoids(hs, comm, cb, M0, n)
    trace, iters, conv = parallel.run(hs, comm, cb)
    assert [(s, c, int(v)) for s, c, v in trace] == [(s, c, int(v)) for s, c, v in ref.trace]
    st = hs[1].km.get_state()
    assert st.medoids.tolist() == ref.medoids.tolist() and st.td == ref.td
    assert st.assignment.tolist() == ref.assignment.tolist()


@pytest.mark.parametrize("mode", ["owner", "gather"])
@pytest.mark.parametrize("world,cid,n,k", [(2, 5, 900, 11), (3, 5, 1300, 17), (4, 3, 800, 9), (2, 5, 1600, 90),
                                          (8, 3, 2000, 40)])
def test_sharded_fastpam2_equals_single_gpu(world, cid, n, k, mode):
    from paper_2008_05171_b200 import KMedoids, parallel
    cfg = kmsynth.CONFIGS[cid]
    X = kmsynth.make_points(cfg, n=n)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    M0 = kmsynth.random_medoids(cfg, k=k, n=n)
    single = KMedoids(Dt, n, k)
    single.set_medoids(M0)
    tr1 = []
    while True:
        conv, sw, td = single.swap_iter("fastpam2")
        tr1.append(single.last_swaps())
        if conv:
            break
    st1 = single.get_state()
    hs, cb = shards(Dt, n, k, world)
    comm = parallel.LocalComm(world)
    parallel.set_medoids(hs, comm, cb, M0, n)
    tr2 = []
    while True:
        conv, sw = parallel.fp2_iter(hs, comm, cb, mode=mode)
        tr2.append(hs[0].km.last_swaps())
        if conv:
            break
    if cfg.metric == kmsynth.L1_INT:
        assert tr2 == tr1
    else:
        assert [[t[:2] for t in it] for it in tr2] == [[t[:2] for t in it] for it in tr1]
    for h in hs:
        st = h.km.get_state()
        assert st.medoids.tolist() == st1.medoids.tolist()
        assert st.assignment.tolist() == st1.assignment.tolist()
        assert st.n_iter == st1.n_iter and st.n_swaps == st1.n_swaps
    if cfg.metric == kmsynth.L1_INT:
        D = kmsynth.as_numpy_D(Dt)[:, :n]
        ref = oracle.swap_run(D, M0, oracle.FASTPAM2)
        assert st1.medoids.tolist() == ref.medoids.tolist() and st1.td == ref.td


@pytest.mark.parametrize("world,cid,n,k", [(2, 5, 700, 9), (3, 4, 900, 12)])
def test_sharded_device_decided_equals_host_decided(world, cid, n, k):
    """run() (device-decided, SUM all-reduce of the column, one iteration
    queued ahead) and run_sync() (host-decided, broadcast) give the same swaps,
    iteration count and state; the status is sticky after convergence."""
    from paper_2008_05171_b200 import parallel
    cfg = kmsynth.CONFIGS[cid]
    X = kmsynth.make_points(cfg, n=n)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    M0 = kmsynth.random_medoids(cfg, k=k, n=n)
    hs, cb = shards(Dt, n, k, world)
    comm = parallel.LocalComm(world)
    parallel.set_medoids(hs, comm, cb, M0, n)
    t1, it1, c1 = parallel.run(hs, comm, cb)
    s1 = [h.km.get_state() for h in hs]
    # extra iterations after convergence change and count nothing
    parallel.swap_iter_async(hs, comm)
    parallel.swap_iter_async(hs, comm)
    conv, it, sw, td = parallel.status(hs, comm, wait=1)
    assert conv and it == it1 and sw == len(t1)
    parallel.set_medoids(hs, comm, cb, M0, n)
    t2, it2, c2 = parallel.run_sync(hs, comm, cb)
    assert c1 and c2 and it1 == it2
    if cfg.metric == kmsynth.L1_INT:
        assert [(a, b, int(v)) for a, b, v in t1] == [(a, b, int(v)) for a, b, v in t2]
    else:
        assert [(a, b) for a, b, v in t1] == [(a, b) for a, b, v in t2]
    for h, s in zip(hs, s1):
        st = h.km.get_state()
        assert st.medoids.tolist() == s.medoids.tolist()
        assert st.assignment.tolist() == s.assignment.tolist()


@pytest.mark.parametrize("world,cid,n,k", [(2, 5, 1200, 9), (3, 1, 500, 5), (1, 4, 900, 7)])
def test_sharded_iteration_graph_replays_equal_direct(world, cid, n, k):
    """The device-decided iteration captured once into a CUDA graph with its
    collectives (parallel.IterationGraph) and replayed: the same swaps,
    iteration count and state as the directly enqueued run; replays after
    convergence are no-ops; status / trace read correctly after resync."""
    from paper_2008_05171_b200 import parallel
    cfg = kmsynth.CONFIGS[cid]
    X = kmsynth.make_points(cfg, n=n)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    M0 = kmsynth.random_medoids(cfg, k=k, n=n)
    hs, cb = shards(Dt, n, k, world)
    comm = parallel.LocalComm(world)
    parallel.set_medoids(hs, comm, cb, M0, n)
    t1, it1, c1 = parallel.run(hs, comm, cb)
    s1 = [h.km.get_state() for h in hs]
    side = torch.cuda.Stream()
    cbs = parallel.column_bounds(n, world)
    hg = [parallel.CudaShard(Dt[:, int(cbs[r]):], n, k, r, cbs, stream=side) for r in range(world)]
    parallel.set_medoids(hg, comm, cbs, M0, n)
    with pytest.raises(ValueError):
        parallel.IterationGraph(hg, comm)          # before the first iteration
    parallel.swap_iter_async(hg, comm)             # one direct iteration: buffers allocated
    g = parallel.IterationGraph(hg, comm)
    assert all(x > 0 for x in g.kernels_per_iter)
    t2, it2, c2 = parallel.run_graph(hg, comm, g, chunk=5)
    assert c1 and c2 and it1 == it2
    if cfg.metric == kmsynth.L1_INT:
        assert [(a, b, int(v)) for a, b, v in t1] == [(a, b, int(v)) for a, b, v in t2]
    else:
        assert [(a, b) for a, b, v in t1] == [(a, b) for a, b, v in t2]
    g.replay(3)                                    # after convergence: no-ops
    g.resync()
    conv, it, sw, td = parallel.status(hg, comm, wait=1)
    assert conv and it == it1 and sw == len(t1)
    for h, a in zip(hg, s1):
        st = h.km.get_state()
        assert st.medoids.tolist() == a.medoids.tolist() and st.assignment.tolist() == a.assignment.tolist()
        assert st.td == a.td
