"""Parity at BASELINE.json's full sizes (C3, C4, C5), in the launch
configuration bench.py times, on outputs the oracle can compute one by one:
per-candidate dTD for sampled candidates, the chosen swap of an iteration,
BUILD steps and the nearest/second cache for sampled objects.  The oracle
works on columns of D fetched from the device (d(., x_c) = D[:, c]); no
symmetry is assumed."""
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


def cols(Dt, idx, n):
    """Columns d(., x_c) for c in idx as a (len(idx), n) host array."""
    t = Dt[:, torch.as_tensor(np.asarray(idx, np.int64), device=Dt.device)][:n].T.contiguous().cpu().numpy()
    return t.view(np.uint32) if t.dtype == np.int32 else t


def check_candidates(km, Dt, n, k, M, rng, nsample, exact):
    """GPU per-candidate (min_i dTD, argmin) == oracle on sampled candidates."""
    v, s = km.eval_candidates()
    cache = oracle.assign_cols(cols(Dt, M, n))
    R = oracle.removal_loss(cache, k)
    td = float(cache.dn.sum())
    pool = np.setdiff1d(np.arange(n), M)
    best = int(np.argmin(np.where(s >= 0, v, np.inf)))
    sample = np.unique(np.concatenate([rng.choice(pool, size=nsample, replace=False), [best]]))
    C = cols(Dt, sample, n)
    for c, col in zip(sample, C):
        vec, plus = oracle.fastpam1_candidate_col(col, cache, R)
        full = vec + plus
        if exact:
            i = int(np.argmin(full))
            assert (int(v[c]), int(s[c])) == (int(full[i]), i), c
        else:
            assert v[c] == pytest.approx(full.min(), rel=1e-9, abs=1e-9 * td)
            srt = np.sort(full)
            if srt[1] - srt[0] > 1e-9 * td:
                assert s[c] == int(np.argmin(full))
    for j in range(k):
        assert s[M[j]] == -1
    return v, s, cache


def check_cache(km, Dt, n, M, rng, nsample=4000):
    near, sec, dn, ds = km.get_cache()
    objs = rng.choice(n, size=nsample, replace=False)
    C = cols(Dt, M, n)                          # (k, n): C[j, o] = d(x_o, m_j)
    sub = oracle.assign_cols(np.ascontiguousarray(C[:, objs]))
    assert near[objs].tolist() == sub.nearest.tolist()
    assert sec[objs].tolist() == sub.second.tolist()
    assert dn[objs].tolist() == sub.dn.tolist() and ds[objs].tolist() == sub.ds.tolist()


def test_c4_fullsize_build_and_swap():
    from paper_2008_05171_b200 import KMedoids
    cfg = kmsynth.CONFIGS[4]
    n, k = cfg.n, cfg.k
    X = kmsynth.make_points(cfg)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    rng = np.random.default_rng(44)
    km = KMedoids(Dt, n, k)
    M, td = km.init_build()
    assert len(set(M.tolist())) == k
    # BUILD: TD bookkeeping vs definition; sampled steps pick the best of a sample
    C = cols(Dt, M, n)
    assert td == pytest.approx(float(C.astype(np.float64).min(axis=0).sum()), rel=1e-9)
    for t in (1, 2, 50, 199):
        dnear = C[:t].astype(np.float64).min(axis=0)
        pool = np.setdiff1d(np.arange(n), M[:t])
        samp = rng.choice(pool, size=64, replace=False)
        Cs = cols(Dt, samp, n).astype(np.float64)
        gains = np.minimum(Cs - dnear[None, :], 0).sum(axis=1)
        g_chosen = np.minimum(C[t].astype(np.float64) - dnear, 0).sum()
        assert g_chosen <= gains.min() + 1e-9 * td
    check_cache(km, Dt, n, M, rng)
    v, s, cache = check_candidates(km, Dt, n, k, M, rng, 96, exact=False)
    # one SWAP iteration: the applied swap is the minimum and its dTD is exact
    conv, sw, td1 = km.swap_iter()
    (i, c, dtd), = km.last_swaps()
    assert (v[c], s[c]) == (pytest.approx(dtd, rel=1e-12), i)
    assert dtd == pytest.approx(np.nanmin(np.where(s >= 0, v, np.inf)), rel=1e-12)
    M2 = M.copy()
    M2[i] = c
    assert td1 == pytest.approx(float(cols(Dt, M2, n).astype(np.float64).min(axis=0).sum()), rel=1e-9)
    check_cache(km, Dt, n, M2, rng)


def test_c5_fullsize_fastpam2_exact():
    from paper_2008_05171_b200 import KMedoids
    cfg = kmsynth.CONFIGS[5]
    n, k = cfg.n, cfg.k
    X = kmsynth.make_points(cfg)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    rng = np.random.default_rng(55)
    M = kmsynth.random_medoids(cfg)
    km = KMedoids(Dt, n, k)
    km.set_medoids(M)
    check_candidates(km, Dt, n, k, M, rng, 48, exact=True)
    check_cache(km, Dt, n, M, rng)
    # two FastPAM2 iterations: every applied swap's dTD is exact (brute force on
    # the current state via the oracle's column form), TD exact
    M = M.copy()
    for it in range(2):
        conv, sw, td = km.swap_iter("fastpam2")
        swaps = km.last_swaps()
        assert len(swaps) == sw
        for (i, c, dtd) in swaps[:6]:
            cache = oracle.assign_cols(cols(Dt, M, n))
            R = oracle.removal_loss(cache, k)
            vec, plus = oracle.fastpam1_candidate_col(cols(Dt, [c], n)[0], cache, R)
            assert int(vec[i] + plus) == dtd
            M[i] = c
        for (i, c, dtd) in swaps[6:]:
            M[i] = c
        assert km.get_state().medoids.tolist() == M.tolist()
        assert td == int(cols(Dt, M, n).astype(np.int64).min(axis=0).sum())
    check_cache(km, Dt, n, M, rng)


def test_c3_fullsize_fastpam1_lockstep_prefix():
    """C3 at full size: three FastPAM1 iterations in lockstep with the full
    oracle (table over all k x (n-k) pairs on the host copy of D)."""
    from paper_2008_05171_b200 import KMedoids
    cfg = kmsynth.CONFIGS[3]
    n, k = cfg.n, cfg.k
    X = kmsynth.make_points(cfg)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    D = kmsynth.as_numpy_D(Dt)[:, :n]
    M = kmsynth.random_medoids(cfg).copy()
    km = KMedoids(Dt, n, k)
    km.set_medoids(M)
    for it in range(3):
        c = oracle.assign(D, M)
        R = oracle.removal_loss(c, k)
        td_ref = oracle.td(D, M)
        bd, bi, bc = oracle.fastpam1_best(D, M, c, R)
        conv, sw, td = km.swap_iter()
        assert not conv and bi >= 0
        (gi, gc, gdtd), = km.last_swaps()
        vec, plus = oracle.fastpam1_candidate(D, gc, c, R)
        assert vec[gi] + plus <= bd + 1e-5 * abs(td_ref)
        assert gdtd == pytest.approx(vec[gi] + plus, rel=1e-9, abs=1e-9 * td_ref)
        M[gi] = gc
        assert td == pytest.approx(oracle.td(D, M), rel=1e-9)


def test_c4_every_candidate_exact_and_deterministic():
    """C4 at full size, EVERY candidate of an iteration: the per-candidate
    (min_i dTD, argmin) equals the oracle's Alg.3 evaluation (reading R9:
    fp64 sums in another order, 1e-9 relative), two evaluations of the same
    state are bitwise identical, and the TD tracked over a whole run to
    convergence equals TD recomputed from its definition (Eq. eqn:td)."""
    from paper_2008_05171_b200 import KMedoids
    cfg = kmsynth.CONFIGS[4]
    n, k = cfg.n, cfg.k
    X = kmsynth.make_points(cfg)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    km = KMedoids(Dt, n, k)
    M, td = km.init_build()
    for _ in range(3):
        km.swap_iter()
    M = km.get_state().medoids
    v1, s1 = km.eval_candidates()
    v2, s2 = km.eval_candidates()
    assert np.array_equal(v1, v2) and np.array_equal(s1, s2)
    cache = oracle.assign_cols(cols(Dt, M, n))
    R = oracle.removal_loss(cache, k)
    tdr = float(cache.dn.sum())
    med = set(M.tolist())
    bad = []
    for c0 in range(0, n, 2500):
        idx = np.arange(c0, min(n, c0 + 2500))
        C = cols(Dt, idx, n)
        for c, col in zip(idx, C):
            if c in med:
                assert s1[c] == -1
                continue
            vec, plus = oracle.fastpam1_candidate_col(col, cache, R)
            full = vec + plus
            i = int(np.argmin(full))
            srt = np.partition(full, 1)
            ok = abs(v1[c] - full[i]) <= 1e-9 * tdr and (s1[c] == i or srt[1] - srt[0] <= 1e-9 * tdr)
            if not ok:
                bad.append((int(c), float(v1[c]), int(s1[c]), float(full[i]), i))
    assert not bad, bad[:10]
    r = km.run(use_build=False)
    assert r.converged
    td_def = float(cols(Dt, r.medoids, n).astype(np.float64).min(axis=0).sum())
    assert r.td == pytest.approx(td_def, rel=1e-9)
    v, s = km.eval_candidates()
    assert np.min(np.where(s >= 0, v, np.inf)) >= -1e-12 * abs(r.td)
