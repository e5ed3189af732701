"""FasterPAM (Alg.4; readings F1-F5) on the GPU vs the oracle.

The GPU evaluates the candidates of consecutive scan positions in
speculative batches and accepts the first improving one, which is exactly
the candidate Alg.4's sequential loop swaps.  On
uint32 dissimilarities the whole run is therefore bit-exact to
oracle.fasterpam_run: the same swaps (slot, candidate, dTD) in the same
order, the same passes, medoids, assignment and int64 TD -- for any batch
width (KM_FASTER_W0 / KM_FASTER_WMAX force one-tile windows here).  On
float32 the sums differ in the last bits (reading R9): swaps must agree
until a decision lies within the tolerance of the north_star (1e-5*TD).
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import kmsynth  # noqa: E402
import oracle  # noqa: E402

FTOL = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.fixture
def windows(request):
    """(W0, WMAX) batch widths in columns for the handles created in a test."""
    w0, wmax = request.param
    old = {k: os.environ.get(k) for k in ("KM_FASTER_W0", "KM_FASTER_WMAX")}
    if w0:
        os.environ["KM_FASTER_W0"], os.environ["KM_FASTER_WMAX"] = str(w0), str(wmax)
    yield request.param
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def KM(*a, **kw):
    from paper_2008_05171_b200 import KMedoids
    return KMedoids(*a, **kw)


def to_dev(D: np.ndarray, ld=None):
    n = D.shape[0]
    ld = ld or kmsynth.round_ld(n)
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


def gpu_passes(km, max_iter=2000):
    """Run FasterPAM passes to convergence; (swap trace, passes, converged)."""
    trace, passes = [], 0
    for _ in range(max_iter):
        conv, sw, td = km.swap_iter("fasterpam")
        got = km.last_swaps()
        assert len(got) == sw
        trace += got
        passes += 1
        if conv:
            return trace, passes, True
    return trace, passes, False


ONE_TILE = (896, 896)          # every batch one 896-column tile
DEFAULT = (0, 0)               # library defaults (2 tiles, doubling to 16)


@pytest.mark.parametrize("windows", [ONE_TILE, DEFAULT], indirect=True)
@pytest.mark.parametrize("seed", range(8))
def test_fasterpam_int_trace_exact(seed, windows):
    rng = np.random.default_rng(3100 + seed)
    n = int(rng.choice([9, 64, 300, 1031, 2500]))
    k = int(rng.integers(2, min(20, n - 1) + 1))
    D = rand_int(rng, n, int(rng.choice([3, 60, 100000])), symmetric=bool(seed % 3))
    M0 = rng.choice(n, size=k, replace=False).astype(np.int32)
    ref = oracle.fasterpam_run(D, M0)
    km = KM(to_dev(D), n, k)
    km.set_medoids(M0)
    tr, passes, conv = gpu_passes(km)
    assert conv and ref.converged
    assert [(i, c, int(v)) for i, c, v in tr] == [(i, c, int(v)) for i, c, v, _ in ref.trace]
    st = km.get_state()
    assert st.medoids.tolist() == ref.medoids.tolist()
    assert st.assignment.tolist() == ref.assignment.tolist()
    assert st.td == ref.td and st.n_swaps == ref.n_swaps
    assert st.n_iter == ref.n_iter == passes
    near, sec, dn, ds = km.get_cache()
    c = oracle.assign(D, ref.medoids)
    assert near.tolist() == c.nearest.tolist() and sec.tolist() == c.second.tolist()
    assert dn.tolist() == c.dn.tolist() and ds.tolist() == c.ds.tolist()


def test_fasterpam_c1_build_then_eager_exact():
    """C1 (u32 Manhattan x100): BUILD on the GPU, then FasterPAM, bit-exact
    to the oracle's BUILD + Alg.4, through kmedoids_run."""
    cfg = kmsynth.CONFIGS[1]
    X = kmsynth.make_points(cfg)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    D = kmsynth.as_numpy_D(Dt)[:, :cfg.n]
    Mb, _, _ = oracle.build_init(D, cfg.k)
    ref = oracle.fasterpam_run(D, Mb)
    km = KM(Dt, cfg.n, cfg.k)
    r = km.run(use_build=True, variant="fasterpam")
    assert r.converged
    assert r.medoids.tolist() == ref.medoids.tolist() and r.td == ref.td
    assert r.assignment.tolist() == ref.assignment.tolist()
    assert (r.n_iter, r.n_swaps) == (ref.n_iter, ref.n_swaps)


def test_fasterpam_c5_recipe_random_init_exact():
    """C5 recipe (u32 L1 x100 with 5% outliers) at an oracle-sized n, random
    init: many swaps in the first pass, bit-exact."""
    cfg = kmsynth.CONFIGS[5]
    n, k = 6000, 40
    X = kmsynth.make_points(cfg, n=n)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    D = kmsynth.as_numpy_D(Dt)[:, :n]
    M0 = kmsynth.random_medoids(cfg, k=k, n=n)
    ref = oracle.fasterpam_run(D, M0)
    km = KM(Dt, n, k)
    km.set_medoids(M0)
    tr, passes, conv = gpu_passes(km)
    assert conv
    assert [(i, c, int(v)) for i, c, v in tr] == [(i, c, int(v)) for i, c, v, _ in ref.trace]
    st = km.get_state()
    assert st.td == ref.td and st.n_iter == ref.n_iter and st.medoids.tolist() == ref.medoids.tolist()


def test_fasterpam_max_iter_and_edge_cases():
    rng = np.random.default_rng(9)
    D = rand_int(rng, 400, 1000)
    M0 = rng.choice(400, size=7, replace=False).astype(np.int32)
    for cap in (1, 2):
        ref = oracle.fasterpam_run(D, M0, max_iter=cap)
        km = KM(to_dev(D), 400, 7)
        km.set_medoids(M0)
        r = km.run(use_build=False, variant="fasterpam", max_iter=cap)
        assert r.converged == ref.converged
        assert (r.n_iter, r.n_swaps, r.td) == (ref.n_iter, ref.n_swaps, ref.td)
        assert r.medoids.tolist() == ref.medoids.tolist()
    # all-zero matrix: one pass, no swap
    km = KM(to_dev(np.zeros((9, 9), np.uint32)), 9, 3)
    km.set_medoids([0, 1, 2])
    r = km.run(use_build=False, variant="fasterpam")
    assert r.converged and r.n_swaps == 0 and r.n_iter == 1 and r.td == 0
    # after convergence further passes do nothing
    conv, sw, td = km.swap_iter("fasterpam")
    assert conv and sw == 0
    # duplicates and k = n - 1
    x = np.array([0, 0, 5, 5, 9, 9, 14])
    D = np.abs(x[:, None] - x[None, :]).astype(np.uint32)
    for k in (2, 6):
        ref = oracle.fasterpam_run(D, list(range(k)))
        km = KM(to_dev(D), 7, k)
        km.set_medoids(list(range(k)))
        r = km.run(use_build=False, variant="fasterpam")
        assert r.medoids.tolist() == ref.medoids.tolist() and r.td == ref.td
        assert (r.n_iter, r.n_swaps) == (ref.n_iter, ref.n_swaps)
        assert r.assignment.tolist() == ref.assignment.tolist()


def test_fasterpam_fig1_instance():
    """Fig.1 (reading R7): the eager scan reaches the optimum."""
    import json
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig1_alternating.json")))
    x = np.array(g["points"], np.int64)
    D = np.abs(x[:, None] - x[None, :]).astype(np.uint32)
    ref = oracle.fasterpam_run(D, g["medoids"])
    km = KM(to_dev(D), len(x), len(g["medoids"]))
    km.set_medoids(g["medoids"])
    r = km.run(use_build=False, variant="fasterpam")
    assert r.td == ref.td == g["losses"][-1]
    assert r.medoids.tolist() == ref.medoids.tolist()
    assert (r.n_iter, r.n_swaps) == (ref.n_iter, ref.n_swaps)


def check_float_against_oracle(D, Dt, n, k, M0):
    """GPU FasterPAM vs oracle.fasterpam_run on float data: identical swaps
    until a near tie (1e-5*TD), every applied dTD = TD change from the
    definition, final local optimum, TD within 1e-5; returns the GPU trace."""
    ref = oracle.fasterpam_run(D, M0)
    km = KM(Dt, n, k)
    km.set_medoids(M0)
    tr, passes, conv = gpu_passes(km)
    assert conv
    M = np.array(M0, np.int32)
    diverged = False
    for j, (i, c, v) in enumerate(tr):
        td_before = oracle.td(D, M)
        if not diverged:
            ri, rc, rv, _ = ref.trace[j] if j < len(ref.trace) else (-1, -1, 0.0, -1)
            if (ri, rc) != (i, c):
                cache = oracle.assign(D, M)
                R = oracle.removal_loss(cache, k)
                vec, plus = oracle.fastpam1_candidate(D, c, cache, R)
                full = np.sort(vec + plus)
                near_tie = abs(full[0]) <= FTOL * td_before or full[1] - full[0] <= FTOL * td_before
                if rc >= 0:
                    vr, pr = oracle.fastpam1_candidate(D, rc, cache, R)
                    near_tie |= abs(np.min(vr + pr)) <= FTOL * td_before
                assert near_tie, (j, (i, c, v), ref.trace[j] if j < len(ref.trace) else None)
                diverged = True
        M[i] = c
        assert v == pytest.approx(oracle.td(D, M) - td_before, rel=1e-9, abs=1e-9 * td_before)
    st = km.get_state()
    assert st.medoids.tolist() == M.tolist()
    assert st.td == pytest.approx(oracle.td(D, M), rel=1e-12)
    assert st.td == pytest.approx(ref.td, rel=FTOL)
    if not diverged:
        assert len(tr) == len(ref.trace) and st.n_iter == ref.n_iter
    v, s = km.eval_candidates()
    assert np.min(np.where(s >= 0, v, np.inf)) >= -1e-9 * st.td
    return tr


def test_fasterpam_float_c4_recipe_from_build_deterministic():
    """C4 recipe (32-D mixture, f32 Euclidean) at n=12000, k=200, GPU BUILD
    start: oracle agreement as above, and two GPU runs are bitwise equal."""
    cfg = kmsynth.CONFIGS[4]
    n, k = 12000, 200
    X = kmsynth.make_points(cfg, n=n)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    D = kmsynth.as_numpy_D(Dt)[:, :n]
    M0, _ = KM(Dt, n, k).init_build()
    tr = check_float_against_oracle(D, Dt, n, k, M0)
    km = KM(Dt, n, k)
    km.set_medoids(M0)
    tr2, _, _ = gpu_passes(km)
    assert tr2 == tr


@pytest.mark.parametrize("windows", [ONE_TILE, DEFAULT], indirect=True)
def test_fasterpam_float_c2_recipe(windows):
    """C2 recipe (f32 Euclidean), oracle-sized: the GPU's swap sequence equals
    the oracle's until a decision is a near tie (|dTD| or the slot gap within
    1e-5*TD); every applied dTD equals the TD change recomputed from its
    definition; the final state is a local optimum; TD within 1e-5."""
    cfg = kmsynth.CONFIGS[2]
    n, k = 2000, cfg.k
    X = kmsynth.make_points(cfg, n=n)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    D = kmsynth.as_numpy_D(Dt)[:, :n]
    M0 = kmsynth.random_medoids(cfg, k=k, n=n)
    ref = oracle.fasterpam_run(D, M0)
    km = KM(Dt, n, k)
    km.set_medoids(M0)
    tr, passes, conv = gpu_passes(km)
    assert conv
    M = np.array(M0, np.int32)
    diverged = False
    for j, (i, c, v) in enumerate(tr):
        td_before = oracle.td(D, M)
        if not diverged:
            ri, rc, rv, _ = ref.trace[j] if j < len(ref.trace) else (-1, -1, 0.0, -1)
            if (ri, rc) != (i, c):
                cache = oracle.assign(D, M)
                R = oracle.removal_loss(cache, k)
                vec, plus = oracle.fastpam1_candidate(D, c, cache, R)
                full = np.sort(vec + plus)
                near_tie = abs(full[0]) <= FTOL * td_before or full[1] - full[0] <= FTOL * td_before
                if rc >= 0:
                    vr, pr = oracle.fastpam1_candidate(D, rc, cache, R)
                    near_tie |= abs(np.min(vr + pr)) <= FTOL * td_before
                assert near_tie, (j, (i, c, v), ref.trace[j] if j < len(ref.trace) else None)
                diverged = True
        M[i] = c
        assert v == pytest.approx(oracle.td(D, M) - td_before, rel=1e-9, abs=1e-9 * td_before)
    st = km.get_state()
    assert st.medoids.tolist() == M.tolist()
    assert st.td == pytest.approx(oracle.td(D, M), rel=1e-12)
    assert st.td == pytest.approx(ref.td, rel=FTOL)
    if not diverged:
        assert len(tr) == len(ref.trace) and st.n_iter == ref.n_iter
    v, s = km.eval_candidates()
    assert np.min(np.where(s >= 0, v, np.inf)) >= -1e-9 * st.td
