"""Incremental FastPAM1 (KM_FASTPAM1_INC): the swaps of Alg.3 (best swap per
iteration, key R1) from k-vectors kept across iterations and corrected after
every swap.  Bit-exact to the oracle's FastPAM1 on uint32 (the same trace,
iterations, medoids, assignment, TD); on float32 the same trajectory as the
streaming FastPAM1 up to the rounding of the re-associated sums."""
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


def KM(*a, **kw):
    from paper_2008_05171_b200 import KMedoids
    return KMedoids(*a, **kw)


def to_dev(D):
    n = D.shape[0]
    ld = kmsynth.round_ld(n)
    buf = np.zeros((n, ld), D.dtype)
    buf[:, :n] = D
    return torch.from_numpy(buf.view(np.int32) if D.dtype == np.uint32 else buf).cuda()


def rand_int(rng, n, hi, symmetric=True):
    A = rng.integers(0, hi, size=(n, n)).astype(np.uint32)
    if symmetric:
        A = np.triu(A, 1)
        A = A + A.T
    np.fill_diagonal(A, 0)
    return A


@pytest.mark.parametrize("seed", range(10))
def test_inc_int_trace_exact(seed):
    rng = np.random.default_rng(7000 + seed)
    n = int(rng.choice([7, 64, 300, 1031, 3000]))
    k = int(rng.integers(2, min(40, n - 1) + 1))
    D = rand_int(rng, n, int(rng.choice([3, 60, 100000])), symmetric=bool(seed % 3))
    M0 = rng.choice(n, size=k, replace=False).astype(np.int32)
    ref = oracle.swap_run(D, M0, oracle.FASTPAM1)
    km = KM(to_dev(D), n, k)
    km.set_medoids(M0)
    trace = []
    for _ in range(5000):
        conv, sw, td = km.swap_iter("fastpam1_inc")
        trace += km.last_swaps()
        if conv:
            break
    assert [(i, c, int(v)) for i, c, v in trace] == [(i, c, int(v)) for i, c, v in ref.trace]
    st = km.get_state()
    assert st.medoids.tolist() == ref.medoids.tolist() and st.td == ref.td
    assert (st.n_iter, st.n_swaps) == (ref.n_iter, ref.n_swaps)
    assert st.assignment.tolist() == ref.assignment.tolist()
    # kmedoids_run in one cooperative launch gives the same
    km2 = KM(to_dev(D), n, k)
    km2.set_medoids(M0)
    r = km2.run(use_build=False, variant="fastpam1_inc")
    assert r.medoids.tolist() == ref.medoids.tolist() and r.td == ref.td and r.n_iter == ref.n_iter


def test_inc_c5_recipe_build_exact_and_mixed_variants():
    """C5 recipe (u32 L1, outliers) at n = 6000, k = 60: BUILD + incremental
    FastPAM1 equals the oracle; switching variants midway stays exact."""
    cfg = kmsynth.CONFIGS[5]
    n, k = 6000, 60
    X = kmsynth.make_points(cfg, n=n)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    D = kmsynth.as_numpy_D(Dt)[:, :n]
    km = KM(Dt, n, k)
    Mb, _ = km.init_build()
    ref = oracle.swap_run(D, Mb, oracle.FASTPAM1)
    for it in range(4):
        km.swap_iter("fastpam1")                  # streaming iterations first
    r = km.run(use_build=False, variant="fastpam1_inc")
    assert r.medoids.tolist() == ref.medoids.tolist() and r.td == ref.td
    assert (r.n_iter, r.n_swaps) == (ref.n_iter, ref.n_swaps)


def test_inc_float_matches_streaming_fastpam1():
    cfg = kmsynth.CONFIGS[2]
    n, k = 3000, 20
    X = kmsynth.make_points(cfg, n=n)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    D = kmsynth.as_numpy_D(Dt)[:, :n]
    M0 = kmsynth.random_medoids(cfg, k=k, n=n)
    a = KM(Dt, n, k); a.set_medoids(M0); ra = a.run(use_build=False, variant="fastpam1")
    b = KM(Dt, n, k); b.set_medoids(M0); rb = b.run(use_build=False, variant="fastpam1_inc")
    assert rb.medoids.tolist() == ra.medoids.tolist() and rb.n_iter == ra.n_iter
    assert rb.td == pytest.approx(ra.td, rel=1e-12)
    assert rb.td == pytest.approx(oracle.td(D, rb.medoids), rel=1e-12)
