"""NEXT-3 FastCLARA on the GPU (kmedoids_clara) vs oracle.clara (P:1109-1129,
reading C1): the same caller-drawn samples; bit-exact on uint32 for FastPAM1
and FasterPAM, TD within 1e-9 on float32."""
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


def samples_for(n, k, ns, seed, s=None):
    s = s or min(n, 80 + 4 * k)
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.stack([rng.choice(n, size=s, replace=False) for _ in range(ns)]).astype(np.int32)


@pytest.mark.parametrize("cid,n,k,variant", [(1, 500, 5, "fastpam1"), (5, 3000, 12, "fastpam1"),
                                             (5, 3000, 12, "fasterpam"), (1, 500, 5, "fasterpam")])
def test_clara_int_exact(cid, n, k, variant):
    cfg = kmsynth.CONFIGS[cid]
    X = kmsynth.make_points(cfg, n=n)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    D = kmsynth.as_numpy_D(Dt)[:, :n]
    S = samples_for(n, k, 5, cfg.seed + 4000)
    t, j, M = oracle.clara(D, k, S, variant)
    km = KM(Dt, n, k)
    Mg, tg, jg = km.clara(S, variant)
    assert (Mg.tolist(), tg, jg) == (M.tolist(), t, j)
    st = km.get_state()
    assert st.medoids.tolist() == M.tolist() and st.td == t


def test_clara_float_and_full_sample():
    cfg = kmsynth.CONFIGS[3]
    n, k = 2000, 20
    X = kmsynth.make_points(cfg, n=n)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    D = kmsynth.as_numpy_D(Dt)[:, :n]
    S = samples_for(n, k, 3, 99)
    t, j, M = oracle.clara(D, k, S)
    Mg, tg, jg = KM(Dt, n, k).clara(S)
    assert tg == pytest.approx(t, rel=1e-9) and jg == j and Mg.tolist() == M.tolist()
    # one sample = all points: the PAM of the whole set
    km = KM(Dt, n, k)
    Mf, tf, _ = km.clara(np.arange(n, dtype=np.int32)[None, :])
    r = KM(Dt, n, k).run(use_build=True)
    assert Mf.tolist() == r.medoids.tolist() and tf == pytest.approx(r.td, rel=1e-12)


def test_clara_argument_errors():
    from paper_2008_05171_b200 import KMError
    D = torch.zeros((20, 20), dtype=torch.int32, device="cuda")
    km = KM(D, 20, 3)
    with pytest.raises(KMError):
        km.clara(np.array([[0, 1, 2]], np.int32))            # s <= k
    with pytest.raises(KMError):
        km.clara(np.array([[0, 1, 2, 2, 5]], np.int32))      # duplicate


@pytest.mark.parametrize("variant", ["fastpam1", "fasterpam"])
def test_clara_many_samples_reuse_nested_handles(variant):
    """More samples than concurrent slots: nested handles run several samples
    (their BUILD is replayed from a captured CUDA graph from the second one
    on); every sample must still equal the oracle exactly (int)."""
    cfg = kmsynth.CONFIGS[5]
    n, k = 1500, 8
    X = kmsynth.make_points(cfg, n=n)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    D = kmsynth.as_numpy_D(Dt)[:, :n]
    S = samples_for(n, k, 19, cfg.seed + 4100)
    t, j, M = oracle.clara(D, k, S, variant)
    km = KM(Dt, n, k)
    Mg, tg, jg = km.clara(S, variant)
    assert (Mg.tolist(), tg, jg) == (M.tolist(), t, j)
    Mg2, tg2, jg2 = km.clara(S, variant)                     # the same handle again (all replays)
    assert (Mg2.tolist(), tg2, jg2) == (M.tolist(), t, j)
