"""NEXT-2: dissimilarity materialisation (kmedoids_dissimilarity) vs the
oracle's plain definitions.  L1 on integer coordinates is exact; L2 runs on
the tensor cores (tcgen05 kind::tf32 with a hi/lo split) and is checked on
squared distances against the bound its arithmetic gives (header of
csrc/km_dist.cuh): |d2_gpu - d2| <= (6d + 16) 2^-24 (|x|^2 + |y|^2) plus the
f32 output rounding."""
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


def l2_bound(X, d):
    """The arithmetic's bound on squared distances with the points centred
    (km_dist.cuh: x - mu, mu = the f32-rounded fp64 mean) -- the norms are
    those of the centred points."""
    Xd = X.astype(np.float64)
    mu = Xd.mean(axis=0).astype(np.float32).astype(np.float64)
    nrm = ((X - mu.astype(np.float32)).astype(np.float64) ** 2).sum(axis=1)
    return (6 * d + 16) * 2.0 ** -24 * (nrm[:, None] + nrm[None, :])


@pytest.mark.parametrize("n,d,c0,c1", [(1, 1, 0, 1), (7, 2, 0, 7), (129, 10, 0, 129), (300, 27, 0, 300),
                                       (1000, 32, 0, 1000), (513, 64, 0, 513), (700, 33, 128, 515),
                                       (260, 5, 256, 260), (3001, 17, 0, 3001), (900, 8, 300, 899)])
def test_l2_tensor_core_matches_definition(n, d, c0, c1):
    from paper_2008_05171_b200 import kmedoids_dissimilarity
    rng = np.random.default_rng(n * 100 + d)
    X = (rng.normal(size=(n, d)) * rng.choice([0.1, 1.0, 8.0]) + rng.normal(size=d) * 3).astype(np.float32)
    Dg = kmedoids_dissimilarity(torch.from_numpy(X).cuda(), "l2", col_begin=c0, col_end=c1)
    Dg = Dg[:, :c1 - c0].double().cpu().numpy()
    Dx = oracle.dist_l2(X)[:, c0:c1]
    tol = l2_bound(X, d)[:, c0:c1] + 2.0 ** -20 * Dx ** 2
    err = np.abs(Dg ** 2 - Dx ** 2)
    assert (err <= tol).all(), (err.max(), np.unravel_index(np.argmax(err - tol), err.shape))
    for i in range(max(c0, 0), min(c1, n)):
        assert Dg[i, i - c0] == 0.0
    assert (Dg >= 0).all()


@pytest.mark.parametrize("n,d,c0,c1", [(1, 1, 0, 1), (65, 2, 0, 65), (300, 64, 0, 300), (257, 3, 64, 200)])
def test_l1_exact(n, d, c0, c1):
    from paper_2008_05171_b200 import kmedoids_dissimilarity
    rng = np.random.default_rng(7 + n)
    Xq = rng.integers(-20000, 20000, size=(n, d)).astype(np.int32)
    Dg = kmedoids_dissimilarity(torch.from_numpy(Xq).cuda(), "l1", col_begin=c0, col_end=c1)
    Dg = Dg[:, :c1 - c0].cpu().numpy().view(np.uint32).astype(np.int64)
    assert (Dg == oracle.dist_l1(Xq)[:, c0:c1]).all()


def test_l2_config_points_close_to_generator_and_swap_runs():
    """C4 recipe points (n=2000): the tensor-core D is within the bound of the
    definition; FastPAM1 on it (through the C ABI) equals the oracle's
    FastPAM1 on the same (downloaded) D."""
    from paper_2008_05171_b200 import KMedoids, kmedoids_dissimilarity
    cfg = kmsynth.CONFIGS[4]
    n, k = 2000, 20
    X = kmsynth.make_points(cfg, n=n).astype(np.float32)
    Dt = kmedoids_dissimilarity(torch.from_numpy(X).cuda(), "l2")
    D = Dt[:, :n].cpu().numpy()
    Dx = oracle.dist_l2(X)
    assert (np.abs(D.astype(np.float64) ** 2 - Dx ** 2) <= l2_bound(X, X.shape[1]) + 2.0 ** -20 * Dx ** 2).all()
    M0 = kmsynth.random_medoids(cfg, k=k, n=n)
    km = KMedoids(Dt, n, k)
    km.set_medoids(M0)
    r = km.run(use_build=False)
    ref = oracle.swap_run(np.ascontiguousarray(D), M0, oracle.FASTPAM1)
    assert r.td == pytest.approx(ref.td, rel=1e-9)
    assert r.medoids.tolist() == ref.medoids.tolist()


def test_l1_config_points_exact_pipeline():
    """C5 recipe points quantised x100 (n=1500): the GPU L1 matrix equals the
    oracle's; FastPAM1 on it is bit-exact to the oracle."""
    from paper_2008_05171_b200 import KMedoids, kmedoids_dissimilarity
    cfg = kmsynth.CONFIGS[5]
    n, k = 1500, 12
    Xq = np.ascontiguousarray(kmsynth.make_points(cfg, n=n), dtype=np.int32)   # already x100-quantised
    Dt = kmedoids_dissimilarity(torch.from_numpy(Xq).cuda(), "l1")
    D = Dt[:, :n].cpu().numpy().view(np.uint32)
    assert (D.astype(np.int64) == oracle.dist_l1(Xq)).all()
    M0 = kmsynth.random_medoids(cfg, k=k, n=n)
    km = KMedoids(Dt, n, k)
    km.set_medoids(M0)
    r = km.run(use_build=False)
    ref = oracle.swap_run(np.ascontiguousarray(D), M0, oracle.FASTPAM1)
    assert r.medoids.tolist() == ref.medoids.tolist() and r.td == ref.td
    assert r.assignment.tolist() == ref.assignment.tolist()


def test_dissimilarity_argument_errors():
    from paper_2008_05171_b200 import KMError, kmedoids_dissimilarity
    X = torch.zeros((10, 65), dtype=torch.float32, device="cuda")
    with pytest.raises(KMError):
        kmedoids_dissimilarity(X, "l2")                   # d > 64 on the tensor-core path
    with pytest.raises(KMError):
        kmedoids_dissimilarity(X[:, :4].contiguous(), "l2", col_begin=5, col_end=3)


@pytest.mark.parametrize("n,d,lo,hi,c0,c1", [
    (300, 2, 0, 2 ** 23 - 1, 0, 300),           # sum of ranges 2^24 - 2: the fp32 kernel, at its limit
    (300, 3, 0, 2 ** 23 - 1, 0, 300),           # 1.5 x 2^24: the integer kernel
    (200, 4, -2 ** 25, 2 ** 25, 0, 200),        # ranges 2^26: the integer kernel
    (150, 3, 2 ** 30, 2 ** 30 + 1000, 0, 150),  # large |x|, small ranges: fp32 after translation
    (1000, 5, -3000, 3000, 3, 997),             # ragged 128-tiles, unaligned slab start
    (385, 64, 0, 5000, 0, 385),                 # C5-like range, three row tiles + 1 row
    (129, 40, -100, 100, 1, 2),                 # one column
    (260, 7, 0, 65535, 0, 260),                 # ranges 2^16 - 1: the packed 16-bit kernel at its limit
    (260, 7, 0, 65536, 0, 260),                 # ranges 2^16: the fp32 kernel
])
def test_l1_fp32_path_exact_and_integer_fallback(n, d, lo, hi, c0, c1):
    """The translated-coordinate L1 kernels (S_i + S_j - 2 sum min) are used
    only where exact: packed 16-bit when every range < 2^16, fp32 when the
    sum of ranges < 2^24 (decided on the device), else the integer kernel;
    every side of both limits must equal the integer definition exactly."""
    from paper_2008_05171_b200 import kmedoids_dissimilarity
    rng = np.random.default_rng(n + d)
    Xq = rng.integers(lo, hi, size=(n, d), endpoint=True).astype(np.int32)
    Xq[0, :] = lo                              # the extremes occur
    Xq[-1, :] = hi
    Dg = kmedoids_dissimilarity(torch.from_numpy(Xq).cuda(), "l1", col_begin=c0, col_end=c1)
    Dg = Dg[:, :c1 - c0].cpu().numpy().view(np.uint32).astype(np.int64)
    assert (Dg == oracle.dist_l1(Xq)[:, c0:c1]).all()


def test_l1_integer_kernel_forced(monkeypatch):
    from paper_2008_05171_b200 import kmedoids_dissimilarity
    monkeypatch.setenv("KM_DIST_L1", "int")
    rng = np.random.default_rng(5)
    Xq = rng.integers(-5000, 5000, size=(333, 17)).astype(np.int32)
    Dg = kmedoids_dissimilarity(torch.from_numpy(Xq).cuda(), "l1")
    assert (Dg[:, :333].cpu().numpy().view(np.uint32).astype(np.int64) == oracle.dist_l1(Xq)).all()


@pytest.mark.parametrize("n,d,c0,c1", [(333, 17, 0, 333), (1000, 5, 3, 997), (129, 64, 0, 129)])
def test_l1_fp32_kernel_forced(monkeypatch, n, d, c0, c1):
    """KM_DIST_L1=f32 disables the packed kernel: the fp32 one on small ranges."""
    from paper_2008_05171_b200 import kmedoids_dissimilarity
    monkeypatch.setenv("KM_DIST_L1", "f32")
    rng = np.random.default_rng(n + 3 * d)
    Xq = rng.integers(-5000, 5000, size=(n, d)).astype(np.int32)
    Dg = kmedoids_dissimilarity(torch.from_numpy(Xq).cuda(), "l1", col_begin=c0, col_end=c1)
    assert (Dg[:, :c1 - c0].cpu().numpy().view(np.uint32).astype(np.int64) == oracle.dist_l1(Xq)[:, c0:c1]).all()


def test_l2_centering_removes_the_offset_error(monkeypatch):
    """Distances are translation invariant; the norm expansion's error scales
    with |x|^2 + |y|^2 unless the points are centred first.  Points near
    (1000, ..., 1000): relative error below 1e-5 with centring, far above it
    without (KM_DIST_CENTER=0, measurement override)."""
    from paper_2008_05171_b200 import kmedoids_dissimilarity
    rng = np.random.default_rng(5)
    X = (rng.normal(size=(1500, 16)) + 1000.0).astype(np.float32)
    Dx = oracle.dist_l2(X)
    off = ~np.eye(1500, dtype=bool)

    def rel(env, metric="l2"):
        monkeypatch.setenv("KM_DIST_CENTER", env)
        Dg = kmedoids_dissimilarity(torch.from_numpy(X).cuda(), metric)[:, :1500].double().cpu().numpy()
        assert (np.diag(Dg) == 0).all()
        return (np.abs(Dg - Dx)[off] / Dx[off]).max()

    assert rel("1") < 1e-5
    assert rel("0") > 1e-3
    # "l2exact" recomputes the cancelling pairs from the points (here: every
    # pair): accurate even uncentred
    assert rel("0", "l2exact") < 1e-6


@pytest.mark.parametrize("cid,n,c0,c1", [(2, 3000, 0, 3000), (3, 3000, 0, 3000), (4, 3000, 0, 3000),
                                         (4, 2600, 517, 2001)])
def test_l2exact_relative_error_on_config_recipes(cid, n, c0, c1):
    """SURVEY 8(f) NEXT-2 / VERDICT r1 item 9: with "l2exact" every pair of
    the config recipes -- within-cluster pairs included, where |x|^2 + |y|^2
    - 2<x,y> cancels -- is within 1e-5 relative of the definition
    (oracle.dist_l2, fp64, rounded to f32), also on a ragged column slab;
    the plain "l2" is not (the tensor cores' fp32 accumulation)."""
    from paper_2008_05171_b200 import kmedoids_dissimilarity
    cfg = kmsynth.CONFIGS[cid]
    X = kmsynth.make_points(cfg, n=n).astype(np.float32)
    Dx = oracle.dist_l2(X).astype(np.float32).astype(np.float64)[:, c0:c1]
    Xt = torch.from_numpy(X).cuda()
    Dg = kmedoids_dissimilarity(Xt, "l2exact", col_begin=c0, col_end=c1)[:, :c1 - c0].double().cpu().numpy()
    off = np.ones_like(Dx, dtype=bool)
    off[np.arange(c0, c1), np.arange(c1 - c0)] = False
    assert (Dg[~off] == 0).all()
    rel = np.abs(Dg - Dx)[off] / Dx[off]
    assert rel.max() <= 1e-5, rel.max()
    Dp = kmedoids_dissimilarity(Xt, "l2", col_begin=c0, col_end=c1)[:, :c1 - c0].double().cpu().numpy()
    assert (np.abs(Dp - Dx)[off] / Dx[off]).max() > 1e-5
