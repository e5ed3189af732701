"""NEXT-3 FastCLARA from points (kmedoids_clara_points): no n x n matrix.

Parity with oracle.clara_points (reading C2): the
sample sub-matrices are computed from the points by the same definitions on
both sides (L2: fp64 sums rounded to float32; L1: exact), so medoids, the
winning sample and the assignment are identical for both metrics; TD is
bit-exact on L1 and agrees to 1e-12 relative on L2 (only the order of the
fp64 sum over objects differs).  At n = 1e6 the call runs without any
n x n matrix and its TD / assignment equal the oracle's definition."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def mixture(rng, n, d, c, metric, spread=8.0):
    centres = spread * rng.standard_normal((c, d))
    X = centres[rng.integers(0, c, size=n)] + rng.standard_normal((n, d))
    if metric == "l1":
        return np.rint(100 * X).astype(np.int32)
    return X.astype(np.float32)


@pytest.mark.parametrize("metric", ["l1", "l2"])
@pytest.mark.parametrize("variant", ["fastpam1", "fasterpam"])
def test_clara_points_equals_oracle(metric, variant):
    from paper_2008_05171_b200 import kmedoids_clara_points
    rng = np.random.default_rng(11 if metric == "l1" else 12)
    n, d, k = 3000, 8, 6
    X = mixture(rng, n, d, 9, metric)
    samples = np.stack([rng.choice(n, size=80 + 4 * k, replace=False) for _ in range(5)])
    M, td, best, asg = kmedoids_clara_points(torch.from_numpy(X).cuda(), metric, k, samples, variant,
                                             assignment=True)
    t, j, Mo, asgo = oracle.clara_points(X, metric, k, samples, variant)
    assert best == j and M.tolist() == Mo.tolist()
    assert asg.tolist() == asgo.tolist()
    if metric == "l1":
        assert td == t
    else:
        assert td == pytest.approx(t, rel=1e-12)


def test_clara_points_ragged_and_edge_sizes():
    """s not a multiple of the 32 x 32 tiles, d = 1 and d = 128, one sample,
    k = s - 1: still equal to the oracle (L1, exact)."""
    from paper_2008_05171_b200 import kmedoids_clara_points
    rng = np.random.default_rng(13)
    for n, d, k, s, ns in [(500, 1, 3, 37, 3), (700, 128, 4, 65, 2), (300, 5, 20, 21, 1)]:
        X = mixture(rng, n, d, 5, "l1")
        samples = np.stack([rng.choice(n, size=s, replace=False) for _ in range(ns)])
        M, td, best, _ = kmedoids_clara_points(torch.from_numpy(X).cuda(), "l1", k, samples)
        t, j, Mo, _ = oracle.clara_points(X, "l1", k, samples)
        assert (M.tolist(), td, best) == (Mo.tolist(), t, j)


def test_clara_points_validation():
    from paper_2008_05171_b200 import KMError, kmedoids_clara_points
    X = torch.zeros((50, 3), dtype=torch.int32, device="cuda")
    with pytest.raises(KMError):
        kmedoids_clara_points(X, "l1", 5, np.arange(5).reshape(1, 5))          # s <= k
    with pytest.raises(KMError):
        kmedoids_clara_points(X, "l1", 2, np.array([[0, 1, 1, 3]]))             # duplicate index
    with pytest.raises(KMError):
        kmedoids_clara_points(X, "l1", 2, np.array([[0, 1, 2, 50]]))            # out of range


def test_clara_points_one_million_points():
    """n = 1e6 (a 4 TB float32 matrix if materialised): 5 samples of
    s = 80 + 4k, k = 20.  The returned TD and assignment equal the oracle's
    definition for the returned medoids, and no sample's own solution beats it
    (each sample's PAM is checked on its sub-matrix by the oracle)."""
    from paper_2008_05171_b200 import kmedoids_clara_points
    rng = np.random.default_rng(14)
    n, d, k = 1_000_000, 16, 20
    X = mixture(rng, n, d, 40, "l2")
    s = 80 + 4 * k
    samples = np.stack([rng.choice(n, size=s, replace=False) for _ in range(5)])
    free0 = torch.cuda.mem_get_info()[0]
    M, td, best, asg = kmedoids_clara_points(torch.from_numpy(X).cuda(), "l2", k, samples, assignment=True)
    assert torch.cuda.mem_get_info()[0] >= free0 - (1 << 30)       # nothing near n^2 bytes stayed allocated
    t, _, asgo = oracle.td_points(X, "l2", M)
    assert td == pytest.approx(t, rel=1e-12)
    assert asg.tolist() == asgo.tolist()
    for jj, S in enumerate(samples):
        Dj = oracle.sub_dissimilarity(X, "l2", S)
        Mb, _, _ = oracle.build_init(Dj, k)
        r = oracle.swap_run(Dj, Mb, oracle.FASTPAM1)
        tj, _, _ = oracle.td_points(X, "l2", S[r.medoids])
        assert tj >= td * (1 - 1e-12)
        if jj == best:
            assert S[r.medoids].tolist() == M.tolist()


def test_clara_points_medoid_chunks_and_repeat_calls():
    """k larger than one shared-memory chunk of medoid points in the TD pass
    (d = 64: 184 medoids per chunk, k = 300), several samples per slot, and a
    second identical call (cached slots, BUILD replayed from graphs): both
    equal the oracle (L1, exact)."""
    from paper_2008_05171_b200 import kmedoids_clara_points
    rng = np.random.default_rng(15)
    n, d, k, s = 20000, 64, 300, 400
    X = mixture(rng, n, d, 60, "l1", spread=6.0)
    samples = np.stack([rng.choice(n, size=s, replace=False) for _ in range(10)])
    t, j, Mo, asgo = oracle.clara_points(X, "l1", k, samples)
    Xt = torch.from_numpy(X).cuda()
    for _ in range(2):
        M, td, best, asg = kmedoids_clara_points(Xt, "l1", k, samples, assignment=True)
        assert (M.tolist(), td, best) == (Mo.tolist(), t, j)
        assert asg.tolist() == asgo.tolist()
