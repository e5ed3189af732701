"""Parity of the CUDA path (through the C ABI) with the CPU oracle.

Bar (BASELINE.json north_star): uint32 dissimilarities bit-exact (medoids,
assignment, swap sequence, int64 TD); float32 TD within relative 1e-5 and
identical medoids wherever the best and second-best dTD differ by more than
that tolerance (lockstep protocol, reading R8).
"""
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


def KM(*a, **kw):
    from paper_2008_05171_b200 import KMedoids
    return KMedoids(*a, **kw)


def to_dev(D: np.ndarray, ld=None):
    """(n, n) numpy -> padded (n, ld) CUDA tensor (uint32 carried as int32 bits)."""
    n = D.shape[0]
    ld = ld or kmsynth.round_ld(n)
    buf = np.zeros((n, ld), D.dtype)
    buf[:, :n] = D
    t = torch.from_numpy(buf.view(np.int32) if D.dtype == np.uint32 else buf).cuda()
    return t


def rand_int(rng, n, hi, symmetric=True):
    A = rng.integers(0, hi, size=(n, n)).astype(np.uint32)
    if symmetric:
        A = np.triu(A, 1)
        A = A + A.T
    np.fill_diagonal(A, 0)
    return A


def gpu_trace(km, k, variant="fastpam1", max_iter=2000):
    """Step the GPU one SWAP iteration at a time; return the swap trace."""
    trace = []
    prev = km.get_state().medoids.copy()
    for _ in range(max_iter):
        conv, swaps, td = km.swap_iter(variant)
        cur = km.get_state().medoids
        changed = [i for i in range(k) if cur[i] != prev[i]]
        trace.append((changed, [int(cur[i]) for i in changed], td))
        prev = cur.copy()
        if conv:
            break
    return trace


# ---------------- input generator: GPU == numpy, bit for bit ----------------

@pytest.mark.parametrize("cid,n,c0,c1", [(1, 500, 0, 500), (2, 700, 0, 700), (3, 333, 0, 333),
                                         (5, 257, 0, 257), (4, 301, 100, 251), (5, 129, 64, 129)])
def test_synth_cuda_matches_numpy(cid, n, c0, c1):
    cfg = kmsynth.CONFIGS[cid]
    X = kmsynth.make_points(cfg, n=n)
    a = kmsynth.as_numpy_D(kmsynth.dist_cuda(X, cfg.metric, c0, c1))
    b = kmsynth.dist_numpy(X, cfg.metric, c0, c1)
    assert a.shape == b.shape and a.tobytes() == b.tobytes()
    if c0 == 0 and c1 == n:
        S = a[:, :n]
        assert (S == S.T).all() and (np.diag(S) == 0).all()


# ---------------- integer path: bit-exact ----------------

def test_c1_build_fastpam1_bit_exact():
    cfg = kmsynth.CONFIGS[1]
    X = kmsynth.make_points(cfg)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    D = kmsynth.as_numpy_D(Dt)[:, :cfg.n]
    Mb, tdb, _ = oracle.build_init(D, cfg.k)
    ref = oracle.swap_run(D, Mb, oracle.FASTPAM1)
    km = KM(Dt, cfg.n, cfg.k)
    Mg, tdg = km.init_build()
    assert Mg.tolist() == Mb.tolist() and tdg == tdb
    near, sec, dn, ds = km.get_cache()
    c = oracle.assign(D, Mb)
    assert near.tolist() == c.nearest.tolist() and sec.tolist() == c.second.tolist()
    assert dn.tolist() == c.dn.tolist() and ds.tolist() == c.ds.tolist()
    tr = gpu_trace(km, cfg.k)
    got = [(ch[0], cs[0]) for ch, cs, _ in tr if ch]
    assert got == [(i, c) for i, c, _ in ref.trace]
    st = km.get_state()
    assert st.medoids.tolist() == ref.medoids.tolist()
    assert st.assignment.tolist() == ref.assignment.tolist()
    assert st.td == ref.td and st.n_iter == ref.n_iter and st.n_swaps == ref.n_swaps


@pytest.mark.parametrize("parts", [None, "1", "3", "37"])
def test_part_counts_trace_exact(parts, monkeypatch):
    """Any number of stream row parts (one part; ragged parts; the default)
    gives the oracle's exact trace on integer data with many ties, on several
    column tiles (n > 896): the combine (a4) completes every segment cut by a
    part boundary."""
    if parts:
        monkeypatch.setenv("KM_PARTS", parts)
    rng = np.random.default_rng(77)
    for n, k, hi in [(2100, 9, 4), (1031, 17, 100000), (3001, 5, 50)]:
        D = rand_int(rng, n, hi, symmetric=bool(n % 2))
        M0 = rng.choice(n, size=k, replace=False).astype(np.int32)
        ref = oracle.swap_run(D, M0, oracle.FASTPAM1)
        km = KM(to_dev(D), n, k)
        km.set_medoids(M0)
        tr = gpu_trace(km, k)
        got = [(ch[0], cs[0]) for ch, cs, _ in tr if ch]
        assert got == [(i, c) for i, c, _ in ref.trace], (n, k)
        st = km.get_state()
        assert st.td == ref.td and st.n_iter == ref.n_iter and st.medoids.tolist() == ref.medoids.tolist()
        km.close()


@pytest.mark.parametrize("seed", range(4))
def test_swap_iters_pipelined_equals_oracle(seed):
    """kmedoids_swap_iters (FastPAM1 iterations queued one ahead, sticky
    convergence) reaches the oracle's exact end state and counts; a bounded
    call stops after `count` passes and the next call continues; after
    convergence further calls are no-ops (no pass counted); other variants and
    set_medoids clear the sticky flag."""
    rng = np.random.default_rng(4000 + seed)
    n, k = int(rng.choice([300, 1500, 2500])), int(rng.integers(3, 12))
    D = rand_int(rng, n, int(rng.choice([4, 1000])), symmetric=bool(seed % 2))
    M0 = rng.choice(n, size=k, replace=False).astype(np.int32)
    ref = oracle.swap_run(D, M0, oracle.FASTPAM1)
    km = KM(to_dev(D), n, k)
    km.set_medoids(M0)
    first = min(3, ref.n_iter)
    conv, it, sw, td = km.swap_iters(first)
    assert it == first and sw == min(first, ref.n_swaps) and conv == (first == ref.n_iter)
    conv, it2, sw2, td = km.swap_iters(2000)
    assert conv or first == ref.n_iter
    st = km.get_state()
    assert st.medoids.tolist() == ref.medoids.tolist() and st.td == ref.td == td
    assert st.n_iter == ref.n_iter and st.n_swaps == ref.n_swaps
    assert st.assignment.tolist() == ref.assignment.tolist()
    conv, it3, sw3, _ = km.swap_iters(5)                     # sticky: nothing runs, nothing counted
    assert conv and sw3 == 0 and km.get_state().n_iter == ref.n_iter
    c2 = km.swap_iter("fastpam2")                            # other variant: a real (non-improving) pass
    assert c2[0] and km.get_state().n_iter == ref.n_iter + 1
    km.set_medoids(M0)                                       # fresh state: FastPAM1 runs again
    tr = gpu_trace(km, k)
    got = [(ch[0], cs[0]) for ch, cs, _ in tr if ch]
    assert got == [(i, c) for i, c, _ in ref.trace]


@pytest.mark.parametrize("seed", range(12))
def test_random_int_instances_trace_exact(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.choice([7, 37, 130, 257, 600, 1031]))
    k = int(rng.integers(2, min(12, n - 1) + 1))
    hi = int(rng.choice([3, 50, 100000]))          # hi=3: massive ties
    D = rand_int(rng, n, hi, symmetric=bool(seed % 3))
    M0 = rng.choice(n, size=k, replace=False).astype(np.int32)
    ref = oracle.swap_run(D, M0, oracle.FASTPAM1)
    km = KM(to_dev(D), n, k)
    km.set_medoids(M0)
    tr = gpu_trace(km, k)
    got = [(ch[0], cs[0]) for ch, cs, _ in tr if ch]
    assert got == [(i, c) for i, c, _ in ref.trace]
    st = km.get_state()
    assert st.medoids.tolist() == ref.medoids.tolist()
    assert st.assignment.tolist() == ref.assignment.tolist()
    assert st.td == ref.td and st.n_iter == ref.n_iter and st.n_swaps == ref.n_swaps
    # cache after convergence equals a from-scratch assignment
    near, sec, dn, ds = km.get_cache()
    c = oracle.assign(D, ref.medoids)
    assert near.tolist() == c.nearest.tolist() and sec.tolist() == c.second.tolist()
    assert dn.tolist() == c.dn.tolist() and ds.tolist() == c.ds.tolist()


@pytest.mark.parametrize("seed", range(6))
def test_per_candidate_values_exact(seed):
    rng = np.random.default_rng(77 + seed)
    n = int(rng.choice([64, 513, 2000]))
    k = int(rng.integers(2, 40))
    D = rand_int(rng, n, int(rng.choice([10, 1000])))
    M0 = rng.choice(n, size=k, replace=False)
    km = KM(to_dev(D), n, k)
    km.set_medoids(M0)
    v, s = km.eval_candidates()
    c = oracle.assign(D, M0)
    R = oracle.removal_loss(c, k)
    for x in range(n):
        if x in M0:
            assert s[x] == -1
            continue
        vec, plus = oracle.fastpam1_candidate(D, x, c, R)
        i = int(np.argmin(vec))                       # smallest slot on ties
        assert (int(v[x]), int(s[x])) == (int(vec[i] + plus), i)


def test_build_int_bit_exact_random():
    rng = np.random.default_rng(5)
    for trial in range(6):
        n = int(rng.choice([9, 100, 777]))
        k = int(rng.integers(1, min(9, n - 1) + 1))
        D = rand_int(rng, n, int(rng.choice([4, 1000])), symmetric=bool(trial % 2))
        Mb, tdb, _ = oracle.build_init(D, k)
        km = KM(to_dev(D), n, k)
        Mg, tdg = km.init_build()
        assert Mg.tolist() == Mb.tolist()
        if k >= 2:
            assert tdg == oracle.td(D, Mb)
        else:
            assert tdg == tdb


def test_edge_cases():
    # all-zero matrix: nothing improves
    D = np.zeros((9, 9), np.uint32)
    km = KM(to_dev(D), 9, 3)
    km.set_medoids([0, 1, 2])
    r = km.run(use_build=False)
    assert r.n_swaps == 0 and r.n_iter == 1 and r.td == 0 and r.converged
    # duplicated points and k = n - 1
    x = np.array([0, 0, 5, 5, 9, 9, 14])
    D = np.abs(x[:, None] - x[None, :]).astype(np.uint32)
    for k in (2, 6):
        M0 = list(range(k))
        ref = oracle.swap_run(D, M0, oracle.FASTPAM1)
        km = KM(to_dev(D), 7, k)
        km.set_medoids(M0)
        r = km.run(use_build=False)
        assert r.medoids.tolist() == ref.medoids.tolist() and r.td == ref.td
        assert r.assignment.tolist() == ref.assignment.tolist()
    # padded rows (ld > n) and an asymmetric matrix
    rng = np.random.default_rng(3)
    D = rand_int(rng, 45, 60, symmetric=False)
    ref = oracle.swap_run(D, [1, 2, 3], oracle.FASTPAM1)
    km = KM(to_dev(D, ld=64), 45, 3)
    km.set_medoids([1, 2, 3])
    r = km.run(use_build=False)
    assert r.medoids.tolist() == ref.medoids.tolist() and r.td == ref.td


def test_invalid_arguments():
    from paper_2008_05171_b200 import KMError
    D = to_dev(np.zeros((8, 8), np.uint32))
    with pytest.raises(KMError):
        KM(D, 8, 8)                       # k >= n
    km = KM(D, 8, 3)
    with pytest.raises(KMError):
        km.set_medoids([0, 0, 1])         # duplicate
    with pytest.raises(KMError):
        km.set_medoids([0, 1, 8])         # out of range
    with pytest.raises(KMError):
        km.swap_iter()                    # no medoids yet


# ---------------- float path: tolerance + lockstep ----------------

def lockstep_fastpam1(D, Dt, n, k, M0, max_iter=10_000, table=True):
    """Lockstep protocol (reading R8): at every iteration the GPU's chosen swap
    must be within FTOL*TD of the oracle's best; the oracle then follows it."""
    km = KM(Dt, n, k)
    km.set_medoids(M0)
    M = np.array(M0, np.int32)
    iters = 0
    while iters < max_iter:
        iters += 1
        c = oracle.assign(D, M)
        R = oracle.removal_loss(c, k)
        td_ref = oracle.td(D, M)
        bd, bi, bc = oracle.fastpam1_best(D, M, c, R)
        conv, swaps, td_gpu = km.swap_iter()
        if conv:                                # a non-improving pass leaves TD unchanged
            assert td_gpu == pytest.approx(td_ref, rel=FTOL)
        st = km.get_state()
        if conv:
            assert bi < 0 or bd >= -FTOL * abs(td_ref), "GPU converged but the oracle improves"
            assert st.td == pytest.approx(td_ref, rel=FTOL)
            return st, iters
        changed = [i for i in range(k) if st.medoids[i] != M[i]]
        assert len(changed) == 1
        gi, gc = changed[0], int(st.medoids[changed[0]])
        vec, plus = oracle.fastpam1_candidate(D, gc, c, R)
        assert vec[gi] + plus <= bd + FTOL * abs(td_ref)
        if (gi, gc) != (bi, bc) and table:
            # only allowed on a near tie
            assert abs((vec[gi] + plus) - bd) <= FTOL * abs(td_ref)
        M[gi] = gc
        assert td_gpu == pytest.approx(oracle.td(D, M), rel=FTOL)
    raise AssertionError("no convergence")


def test_c2_float_build_and_lockstep():
    cfg = kmsynth.CONFIGS[2]
    n = 2000                                  # C2 recipe, oracle-sized prefix
    X = kmsynth.make_points(cfg, n=n)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    D = kmsynth.as_numpy_D(Dt)[:, :n]
    Mb, tdb, gains = oracle.build_init(D, cfg.k)
    km = KM(Dt, n, cfg.k)
    Mg, tdg = km.init_build()
    assert tdg == pytest.approx(tdb, rel=FTOL)
    assert Mg.tolist() == Mb.tolist()        # no near ties in BUILD on this input
    st, iters = lockstep_fastpam1(D, Dt, n, cfg.k, Mg)
    ref = oracle.swap_run(D, Mg, oracle.FASTPAM1)
    assert st.td == pytest.approx(ref.td, rel=FTOL)
    assert st.medoids.tolist() == ref.medoids.tolist()
    assert st.assignment.tolist() == ref.assignment.tolist()


def test_float_per_candidate_values():
    rng = np.random.default_rng(8)
    n, k = 1500, 17
    X = rng.normal(size=(n, 5))
    D = kmsynth.dist_numpy(X, kmsynth.L2_F32)[:, :n]
    M0 = rng.choice(n, size=k, replace=False)
    km = KM(to_dev(D), n, k)
    km.set_medoids(M0)
    v, s = km.eval_candidates()
    c = oracle.assign(D, M0)
    R = oracle.removal_loss(c, k)
    td = oracle.td(D, M0)
    for x in range(0, n, 7):
        if x in M0:
            continue
        vec, plus = oracle.fastpam1_candidate(D, x, c, R)
        full = vec + plus
        assert v[x] == pytest.approx(full.min(), rel=1e-9, abs=1e-9 * td)
        srt = np.sort(full)
        if srt[1] - srt[0] > 1e-9 * td:
            assert s[x] == int(np.argmin(full))


# ---------------- FastPAM2 (reading R6) ----------------

def gpu_swaps(km, variant, max_iter=2000):
    """Run SWAP iterations to convergence; return the full swap trace."""
    trace = []
    for _ in range(max_iter):
        conv, swaps, td = km.swap_iter(variant)
        got = km.last_swaps()
        assert len(got) == swaps
        trace += got
        if conv:
            break
    return trace


@pytest.mark.parametrize("seed", range(10))
def test_fastpam2_int_trace_exact(seed):
    rng = np.random.default_rng(500 + seed)
    n = int(rng.choice([9, 64, 257, 700]))
    k = int(rng.integers(2, min(16, n - 1) + 1))
    D = rand_int(rng, n, int(rng.choice([3, 40, 10000])), symmetric=bool(seed % 2))
    M0 = rng.choice(n, size=k, replace=False).astype(np.int32)
    ref = oracle.swap_run(D, M0, oracle.FASTPAM2)
    km = KM(to_dev(D), n, k)
    km.set_medoids(M0)
    tr = gpu_swaps(km, "fastpam2")
    assert [(i, c, int(v)) for i, c, v in tr] == [(i, c, int(v)) for i, c, v in ref.trace]
    st = km.get_state()
    assert st.medoids.tolist() == ref.medoids.tolist()
    assert st.assignment.tolist() == ref.assignment.tolist()
    assert st.td == ref.td and st.n_iter == ref.n_iter and st.n_swaps == ref.n_swaps
    near, sec, dn, ds = km.get_cache()
    c = oracle.assign(D, ref.medoids)
    assert near.tolist() == c.nearest.tolist() and sec.tolist() == c.second.tolist()


def test_fastpam1_last_swaps_trace():
    rng = np.random.default_rng(42)
    n, k = 300, 6
    D = rand_int(rng, n, 500)
    M0 = rng.choice(n, size=k, replace=False)
    ref = oracle.swap_run(D, M0, oracle.FASTPAM1)
    km = KM(to_dev(D), n, k)
    km.set_medoids(M0)
    tr = gpu_swaps(km, "fastpam1")
    assert [(i, c, int(v)) for i, c, v in tr] == [(i, c, int(v)) for i, c, v in ref.trace]


def test_fastpam2_float_c3_prefix():
    """C3 recipe (oracle-sized prefix): FastPAM2 final TD within 1e-5 of the
    oracle, every applied dTD exact up to fp64 rounding, final state a local
    optimum (a GPU FastPAM1 pass finds nothing improving)."""
    cfg = kmsynth.CONFIGS[3]
    n, k = 1500, 30
    X = kmsynth.make_points(cfg, n=n)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    D = kmsynth.as_numpy_D(Dt)[:, :n]
    M0 = kmsynth.random_medoids(cfg, k=k, n=n)
    ref = oracle.swap_run(D, M0, oracle.FASTPAM2)
    km = KM(Dt, n, k)
    km.set_medoids(M0)
    M = list(M0)
    for _ in range(500):
        conv, swaps, td = km.swap_iter("fastpam2")
        for (i, c, v) in km.last_swaps():
            td_before = oracle.td(D, M)
            M[i] = c
            assert v == pytest.approx(oracle.td(D, M) - td_before, rel=1e-9, abs=1e-9 * td_before)
        if conv:
            break
    st = km.get_state()
    assert st.medoids.tolist() == M
    assert st.td == pytest.approx(ref.td, rel=FTOL)
    assert st.td == pytest.approx(oracle.td(D, M), rel=1e-12)
    v, s = km.eval_candidates()
    assert np.nanmin(np.where(s >= 0, v, np.inf)) >= -1e-9 * st.td


@pytest.mark.parametrize("variant", ["fastpam1", "fastpam2", "fasterpam"])
def test_large_k_and_tiny_n(variant):
    """Many slots (k = 900 of n = 2501: segments of ~3 rows, many empty-slot
    and part-boundary cases) and the smallest problems (n = 3, k = 2)."""
    rng = np.random.default_rng(8080)
    n, k = 2501, 900
    D = rand_int(rng, n, 1 << 20)
    M0 = rng.choice(n, size=k, replace=False).astype(np.int32)
    ref = (oracle.fasterpam_run(D, M0) if variant == "fasterpam"
           else oracle.swap_run(D, M0, oracle.FASTPAM1 if variant == "fastpam1" else oracle.FASTPAM2, max_iter=6))
    km = KM(to_dev(D), n, k)
    km.set_medoids(M0)
    r = km.run(use_build=False, variant=variant, max_iter=2000 if variant == "fasterpam" else 6)
    assert r.medoids.tolist() == ref.medoids.tolist() and r.td == ref.td
    assert (r.n_iter, r.n_swaps) == (ref.n_iter, ref.n_swaps)
    D3 = np.array([[0, 5, 1], [5, 0, 4], [1, 4, 0]], np.uint32)
    ref3 = (oracle.fasterpam_run(D3, [1, 2]) if variant == "fasterpam"
            else oracle.swap_run(D3, [1, 2], oracle.FASTPAM1 if variant == "fastpam1" else oracle.FASTPAM2))
    km3 = KM(to_dev(D3), 3, 2)
    km3.set_medoids([1, 2])
    r3 = km3.run(use_build=False, variant=variant)
    assert r3.medoids.tolist() == ref3.medoids.tolist() and r3.td == ref3.td


@pytest.mark.parametrize("skew", ["0", "7", "15"])
def test_part_tilt_does_not_change_results(monkeypatch, skew):
    """The stream's row parts are arbitrary row ranges (km::part_lo): any tilt
    (KM_PART_SKEW, 16ths) and any part count give the oracle's exact trace."""
    monkeypatch.setenv("KM_PART_SKEW", skew)
    for parts in ("0", "9"):
        monkeypatch.setenv("KM_PARTS", parts)
        rng = np.random.default_rng(77)
        n, k = 1500, 9
        D = rand_int(rng, n, 5000, symmetric=True)
        M0 = rng.choice(n, size=k, replace=False).astype(np.int32)
        ref = oracle.swap_run(D, M0, oracle.FASTPAM1)
        km = KM(to_dev(D), n, k)
        km.set_medoids(M0)
        r = km.run(use_build=False)
        assert r.medoids.tolist() == ref.medoids.tolist() and r.td == ref.td and r.n_iter == ref.n_iter
        km.close()


def test_run_host_jobs_reuse_buffer_and_handle():
    """kmedoids_run_host (H2D of D, init, SWAP to convergence, D2H): repeated
    jobs of one shape reuse the device buffer and the handle; every job equals
    the oracle on ITS matrix (BUILD and given-medoid inits, FastPAM1 and
    FastPAM2), a job whose D has a nonzero diagonal is refused (KM_EINVAL)
    even on a reused handle, and the cache can be released."""
    from paper_2008_05171_b200 import KMError, kmedoids_release_host_cache, kmedoids_run_host
    rng = np.random.default_rng(808)
    n, k = 700, 6
    for job in range(4):
        D = rand_int(rng, n, [5, 1000][job % 2], symmetric=bool(job % 3))
        Dh = np.zeros((n, kmsynth.round_ld(n)), np.uint32)
        Dh[:, :n] = D
        if job % 2 == 0:
            r = kmedoids_run_host(Dh, k, use_build=True)
            Mb, _, _ = oracle.build_init(D, k)
            ref = oracle.swap_run(D, Mb, oracle.FASTPAM1)
        else:
            M0 = rng.choice(n, size=k, replace=False)
            r = kmedoids_run_host(Dh, k, use_build=False, medoids=M0, variant="fastpam2")
            ref = oracle.swap_run(D, M0, oracle.FASTPAM2)
        assert r.medoids.tolist() == ref.medoids.tolist() and r.td == ref.td
        assert r.assignment.tolist() == ref.assignment.tolist()
        assert (r.n_iter, r.n_swaps) == (ref.n_iter, ref.n_swaps)
    Dh[3, 3] = 1
    with pytest.raises(KMError):
        kmedoids_run_host(Dh, k, use_build=True)
    kmedoids_release_host_cache()
    Dh[3, 3] = 0
    r = kmedoids_run_host(Dh, k, use_build=True)
    assert r.td == oracle.td(Dh[:, :n], r.medoids)
    kmedoids_release_host_cache()


def test_input_validation_diagonal_nan_negative():
    """The documented preconditions are checked (include/kmedoids.h): a
    nonzero or NaN diagonal is refused at create (also for a column slab),
    a negative or NaN dissimilarity in a medoid column at set_medoids (float
    path); valid inputs pass."""
    from paper_2008_05171_b200 import KMError
    rng = np.random.default_rng(31)
    D = rand_int(rng, 40, 100)
    Dbad = D.copy()
    Dbad[7, 7] = 3
    with pytest.raises(KMError):
        KM(to_dev(Dbad), 40, 3)
    # a column slab [8, 40): its diagonal entries D[o][o - 8]
    slab = np.ascontiguousarray(D[:, 8:])
    slab[20, 12] = 1
    with pytest.raises(KMError):
        KM(torch.from_numpy(np.ascontiguousarray(np.pad(slab, ((0, 0), (0, 0)))).view(np.int32)).cuda(), 40, 3,
           col_begin=8, col_end=40)
    F = rand_int(rng, 40, 100).astype(np.float32)
    Fn = F.copy()
    Fn[5, 5] = np.nan
    with pytest.raises(KMError):
        KM(to_dev(Fn), 40, 3)
    Fm = F.copy()
    Fm[11, 2] = -1.0                              # d(x_11, m) < 0 for the medoid m = 2
    km = KM(to_dev(Fm), 40, 3)
    with pytest.raises(KMError):
        km.set_medoids([2, 4, 6])
    Fm[11, 2] = np.nan
    km = KM(to_dev(Fm), 40, 3)
    with pytest.raises(KMError):
        km.set_medoids([2, 4, 6])
    km.set_medoids([3, 4, 6])                     # columns without the bad value: accepted
    KM(to_dev(F), 40, 3).set_medoids([2, 4, 6])


@pytest.mark.parametrize("seed", range(3))
def test_fastpam2_symmetric_rows_equal_oracle(seed):
    """kmedoids_set_symmetric: verified on the device (an asymmetric D is
    refused), after which the FastPAM2 re-evaluations read candidate rows --
    the trace is still the oracle's, bit for bit."""
    from paper_2008_05171_b200 import KMError
    rng = np.random.default_rng(6100 + seed)
    n, k = int(rng.choice([513, 1500, 2222])), int(rng.integers(5, 60))
    D = rand_int(rng, n, int(rng.choice([6, 1000])))
    M0 = rng.choice(n, size=k, replace=False).astype(np.int32)
    ref = oracle.swap_run(D, M0, oracle.FASTPAM2)
    km = KM(to_dev(D), n, k)
    km.set_symmetric(True)
    km.set_medoids(M0)
    r = km.run(use_build=False, variant="fastpam2")
    assert r.medoids.tolist() == ref.medoids.tolist() and r.td == ref.td
    assert (r.n_iter, r.n_swaps) == (ref.n_iter, ref.n_swaps)
    A = rand_int(rng, 300, 50, symmetric=False)
    km2 = KM(to_dev(A), 300, 4)
    with pytest.raises(KMError):
        km2.set_symmetric(True)
    A[np.tril_indices(300, -1)] = A.T[np.tril_indices(300, -1)]      # now symmetric
    KM(to_dev(A), 300, 4).set_symmetric(True)


@pytest.mark.parametrize("variant", ["fastpam1", "fastpam2"])
def test_post_chunk_loop_path_equals_oracle(variant, monkeypatch):
    """The post kernel's chunk-loop path (taken when a block owns more than 256
    objects, n > ~113,000 on a B200; forced here with KM_POST_REG=0) gives the
    oracle's exact trace, on several sizes and many ties."""
    monkeypatch.setenv("KM_POST_REG", "0")
    rng = np.random.default_rng(9100)
    for n, k, hi in [(2500, 11, 5), (777, 40, 1000), (3000, 3, 100000)]:
        D = rand_int(rng, n, hi, symmetric=bool(k % 2))
        M0 = rng.choice(n, size=k, replace=False).astype(np.int32)
        ref = oracle.swap_run(D, M0, oracle.FASTPAM1 if variant == "fastpam1" else oracle.FASTPAM2)
        km = KM(to_dev(D), n, k)
        km.set_medoids(M0)
        r = km.run(use_build=False, variant=variant)
        assert r.medoids.tolist() == ref.medoids.tolist() and r.td == ref.td
        assert (r.n_iter, r.n_swaps) == (ref.n_iter, ref.n_swaps)
        assert r.assignment.tolist() == ref.assignment.tolist()
        km.close()
