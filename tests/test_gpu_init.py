"""NEXT-4 initialisations on the GPU (kmedoids_init_weighted / _lab) vs the
oracle (readings I1, I2).  The random numbers are inputs, so
the integer path is bit-exact; LAB sums in the oracle's order and is exact on
float too; distance-weighted seeding on float agrees up to the rounding of
the prefix sums (each pick is checked against the sampling definition)."""
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


def rand_int(rng, n, hi):
    A = rng.integers(0, hi, size=(n, n)).astype(np.uint32)
    A = np.triu(A, 1)
    A = A + A.T
    np.fill_diagonal(A, 0)
    return A


@pytest.mark.parametrize("seed", range(6))
def test_weighted_int_exact(seed):
    rng = np.random.default_rng(4000 + seed)
    n = int(rng.choice([5, 64, 333, 2500]))
    k = int(rng.integers(2, min(30, n - 1) + 1))
    D = rand_int(rng, n, int(rng.choice([2, 100, 100000])))
    u = rng.random(k)
    ref = oracle.init_weighted(D, k, u)
    km = KM(to_dev(D), n, k)
    M, td = km.init_weighted(u)
    assert M.tolist() == ref.tolist()
    assert td == oracle.td(D, ref)
    near, sec, dn, ds = km.get_cache()
    c = oracle.assign(D, ref)
    assert near.tolist() == c.nearest.tolist() and dn.tolist() == c.dn.tolist()


def test_weighted_float_picks_follow_the_definition():
    cfg = kmsynth.CONFIGS[2]
    n, k = 3000, 25
    X = kmsynth.make_points(cfg, n=n)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    D = kmsynth.as_numpy_D(Dt)[:, :n].astype(np.float64)
    u = np.random.default_rng(12).random(k)
    M, td = KM(Dt, n, k).init_weighted(u)
    assert M[0] == int(u[0] * n) and len(set(M.tolist())) == k
    w = D[:, M[0]].copy()
    for i in range(1, k):
        W = w.sum()
        r = u[i] * W
        pref = np.cumsum(w)
        c = int(M[i])
        lo = pref[c - 1] if c > 0 else 0.0
        assert lo <= r + 1e-9 * W and pref[c] > r - 1e-9 * W and w[c] > 0
        w = np.minimum(w, D[:, c])
    assert td == pytest.approx(D[:, M].min(axis=1).sum(), rel=1e-9)


@pytest.mark.parametrize("cid,n,k", [(1, 500, 5), (5, 3000, 30), (3, 2500, 40), (4, 4000, 60)])
def test_lab_exact_int_and_float(cid, n, k):
    cfg = kmsynth.CONFIGS[cid]
    X = kmsynth.make_points(cfg, n=n)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    D = kmsynth.as_numpy_D(Dt)[:, :n]
    s, rows = oracle.lab_sample_rows(n, k, seed=cfg.seed + 2000)
    ref = oracle.init_lab(D, k, s, rows)
    km = KM(Dt, n, k)
    M, td = km.init_lab(s, rows)
    assert M.tolist() == ref.tolist()
    assert td == pytest.approx(oracle.td(D, ref), rel=1e-12)


def test_lab_full_sample_equals_gpu_build_and_fasterpam_from_lab():
    rng = np.random.default_rng(31)
    n, k = 700, 9
    D = rand_int(rng, n, 5000)
    rows = np.stack([np.concatenate([rng.permutation(n), -np.ones(k, np.int64)]) for _ in range(k)]).astype(np.int32)
    km = KM(to_dev(D), n, k)
    Mb, _ = km.init_build()
    km2 = KM(to_dev(D), n, k)
    Ml, _ = km2.init_lab(n, rows)
    assert Ml.tolist() == Mb.tolist()
    # the paper's recommended pipeline: a cheap init, then FasterPAM
    s, rows = oracle.lab_sample_rows(n, k, seed=7)
    M0 = oracle.init_lab(D, k, s, rows)
    ref = oracle.fasterpam_run(D, M0)
    km3 = KM(to_dev(D), n, k)
    km3.init_lab(s, rows)
    r = km3.run(use_build=False, variant="fasterpam")
    assert r.medoids.tolist() == ref.medoids.tolist() and r.td == ref.td


def test_init_argument_errors():
    from paper_2008_05171_b200 import KMError
    D = np.zeros((10, 10), np.uint32)
    km = KM(to_dev(D), 10, 3)
    with pytest.raises(KMError):
        km.init_weighted([0.1, 1.5, 0.2])
    with pytest.raises(KMError):
        km.init_lab(3, np.full((3, 6), 11, np.int32))


@pytest.mark.parametrize("which", ["weighted", "lab"])
def test_single_block_and_cooperative_kernels_agree(monkeypatch, which):
    """The cooperative seeding kernels (default) and the single-block ones
    (KM_INIT_*=block) give the oracle's medoids on integer data."""
    rng = np.random.default_rng(91)
    n, k = 2100, 17
    D = rand_int(rng, n, 3000)
    u = rng.random(k)
    s, rows = oracle.lab_sample_rows(n, k, seed=5)
    ref = oracle.init_weighted(D, k, u) if which == "weighted" else oracle.init_lab(D, k, s, rows)
    for mode in ("", "block"):
        monkeypatch.setenv("KM_INIT_WEIGHTED" if which == "weighted" else "KM_INIT_LAB", mode)
        km = KM(to_dev(D), n, k)
        M, td = km.init_weighted(u) if which == "weighted" else km.init_lab(s, rows)
        assert M.tolist() == ref.tolist(), mode
        assert td == oracle.td(D, ref)
