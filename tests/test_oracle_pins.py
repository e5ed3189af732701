"""Pins of the CPU oracle against what the paper and the mathematics fix.

Nothing here compares the oracle with itself: every expected value comes from
a golden fixture (cited), from brute force written here independently (full
recomputation of TD after a swap, exhaustive search over medoid sets), from
the paper's Appendix-A decomposition, or from an invariant the paper states.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def line_matrix(points):
    x = np.asarray(points, dtype=np.int64)
    return np.abs(x[:, None] - x[None, :]).astype(np.uint32)


# ---------- brute force, written independently of oracle/ ----------

def bf_td(D, M):
    """TD by definition: every object to its closest medoid (Eq. eqn:td)."""
    n = D.shape[0]
    tot = 0
    for o in range(n):
        tot += min(int(D[o, m]) if D.dtype == np.uint32 else float(D[o, m]) for m in M)
    return tot


def bf_delta(D, M, i, c):
    M2 = list(M)
    M2[i] = c
    return bf_td(D, M2) - bf_td(D, M)


def rand_int_matrix(rng, n, hi=50, symmetric=True):
    A = rng.integers(0, hi, size=(n, n)).astype(np.uint32)
    if symmetric:
        A = np.triu(A, 1)
        A = A + A.T
    np.fill_diagonal(A, 0)
    return A


# ---------- golden worked examples ----------

def test_spec_line_example_cache_and_removal_loss():
    g = _gold("spec_line_0_5_6_10.json")
    D = line_matrix(g["points"])
    c = oracle.assign(D, g["medoids"])
    assert c.nearest.tolist() == g["nearest"]
    assert c.dn.tolist() == g["dn"]
    assert c.ds.tolist() == g["ds"]
    assert oracle.td(D, g["medoids"]) == g["td"]
    assert oracle.removal_loss(c, 2).tolist() == g["removal_loss"]


def test_spec_line_example_change_function():
    g = _gold("spec_line_0_5_6_10.json")
    D = line_matrix(g["points"])
    c = oracle.assign(D, g["medoids"])
    s = g["swap_slot0_with_point1"]
    per = [oracle.change(int(D[o, 1]), int(c.nearest[o]), int(c.dn[o]), int(c.ds[o]), 0) for o in range(4)]
    assert per == s["per_object_change"]
    assert sum(per) == s["delta_td"] == bf_delta(D, g["medoids"], 0, 1)
    assert bf_td(D, [1, 3]) == s["td_after"]


def test_spec_line_example_fastpam1_vectors_and_trace():
    g = _gold("spec_line_0_5_6_10.json")
    D = line_matrix(g["points"])
    c = oracle.assign(D, g["medoids"])
    R = oracle.removal_loss(c, 2)
    for cand in (1, 2):
        gg = g[f"fastpam1_candidate_{cand}"]
        vec, plus = oracle.fastpam1_candidate(D, cand, c, R)
        assert vec.tolist() == gg["vec"] and plus == gg["plus"]
        assert [int(v + plus) for v in vec] == gg["delta_td"]
        assert gg["delta_td"] == [bf_delta(D, g["medoids"], i, cand) for i in range(2)]
    for variant in (oracle.PAM, oracle.FASTPAM1, oracle.FASTPAM2):
        r = oracle.swap_run(D, g["medoids"], variant)
        assert [list(t) for t in r.trace] == g["trace"]
        assert r.medoids.tolist() == g["final_medoids"] and r.td == g["final_td"]
    # the final state is the exhaustive optimum over all C(4,2) medoid sets
    assert g["final_td"] == min(bf_td(D, list(s)) for s in itertools.combinations(range(4), 2))


def test_fig1_trace_reproduces_printed_losses():
    g = _gold("fig1_alternating.json")
    D = line_matrix(g["points"])
    assert bf_td(D, g["medoids"]) == g["losses"][0]
    for variant in (oracle.PAM, oracle.FASTPAM1):
        r = oracle.swap_run(D, g["medoids"], variant)
        assert [list(t) for t in r.trace] == g["trace"]
        M = list(g["medoids"])
        losses = [bf_td(D, M)]
        for (i, cnd, dtd) in r.trace:
            M[i] = cnd
            losses.append(bf_td(D, M))
        assert losses == g["losses"]
        assert r.medoids.tolist() == g["final_medoids"]
        assert r.td == min(bf_td(D, list(s)) for s in itertools.combinations(range(6), 2))


def test_build_golden():
    g = _gold("spec_build_0_1_2_10.json")
    D = line_matrix(g["points"])
    assert [int(D[:, c].sum()) for c in range(4)] == g["first_medoid_sums"]
    M, td, gains = oracle.build_init(D, g["k"])
    assert M.tolist() == g["medoids"] and td == g["td"] and gains.tolist() == g["gains"]
    assert bf_td(D, g["medoids"]) == g["td"]


# ---------- Appendix A: decomposition == four-case change ----------

def test_appendix_a_identity():
    rng = np.random.default_rng(7)
    for _ in range(1000):
        dn = int(rng.integers(0, 20))
        ds = dn + int(rng.integers(0, 20))
        doc = int(rng.integers(0, 45))
        k = int(rng.integers(2, 6))
        near = int(rng.integers(0, k))
        i = int(rng.integers(0, k))
        minus = (ds - dn) if near == i else 0
        plus = (doc - dn) if doc < dn else 0
        if near == i and doc < dn:
            corr = dn - ds
        elif near == i and doc < ds:
            corr = doc - ds
        else:
            corr = 0
        assert oracle.change(doc, near, dn, ds, i) == minus + plus + corr


# ---------- brute force on random instances ----------

@pytest.mark.parametrize("symmetric", [True, False])
def test_change_sum_and_fastpam1_table_equal_bruteforce(symmetric):
    rng = np.random.default_rng(11 + symmetric)
    for trial in range(60):
        n = int(rng.integers(5, 18))
        k = int(rng.integers(2, min(6, n - 1) + 1))
        D = rand_int_matrix(rng, n, hi=30, symmetric=symmetric)
        M = rng.choice(n, size=k, replace=False).astype(np.int32)
        c = oracle.assign(D, M)
        R = oracle.removal_loss(c, k)
        T = oracle.fastpam1_table(D, M, c, R)
        for i in range(k):
            for x in range(n):
                if x in M:
                    continue
                bf = bf_delta(D, M, i, x)
                # Eq. eqn:td2 with Alg.2's object set (x_o not in M \ m_i)
                s = sum(oracle.change(int(D[o, x]), int(c.nearest[o]), int(c.dn[o]), int(c.ds[o]), i)
                        for o in range(n) if o == M[i] or o not in M)
                assert s == bf
                assert T[i, x] == bf


def test_assign_against_sorting():
    rng = np.random.default_rng(3)
    for _ in range(100):
        n = int(rng.integers(3, 30))
        k = int(rng.integers(2, n))
        D = rand_int_matrix(rng, n, hi=8)    # many ties
        M = rng.choice(n, size=k, replace=False)
        c = oracle.assign(D, M)
        for o in range(n):
            order = sorted(range(k), key=lambda j: (int(D[o, M[j]]), j))
            assert c.nearest[o] == order[0] and c.second[o] == order[1]
            assert c.dn[o] == D[o, M[order[0]]] and c.ds[o] == D[o, M[order[1]]]
        R = oracle.removal_loss(c, k)
        assert (R >= 0).all()
        assert R.sum() == (c.ds - c.dn).sum()
        for i in range(k):
            # removal loss = TD increase when medoid i is simply deleted
            Mi = [m for j, m in enumerate(M) if j != i]
            assert R[i] == bf_td(D, Mi) - bf_td(D, M)


def test_pam_equals_fastpam1_traces_and_local_optimum():
    rng = np.random.default_rng(2008)
    for trial in range(200):
        n = int(rng.integers(10, 41))
        k = int(rng.integers(2, 9))
        D = rand_int_matrix(rng, n, hi=int(rng.choice([5, 20, 1000])), symmetric=bool(trial % 4))
        M0 = rng.choice(n, size=k, replace=False)
        a = oracle.swap_run(D, M0, oracle.PAM)
        b = oracle.swap_run(D, M0, oracle.FASTPAM1)
        assert a.trace == b.trace and a.td == b.td and a.medoids.tolist() == b.medoids.tolist()
        assert a.converged and a.n_iter == a.n_swaps + 1
        assert b.td == bf_td(D, b.medoids)                          # TD bookkeeping
        M = list(M0)
        prev = bf_td(D, M)
        for (i, c, dtd) in b.trace:                                  # each applied dTD is exact
            assert dtd == bf_delta(D, M, i, c) and dtd < 0
            M[i] = c
            cur = bf_td(D, M)
            assert cur < prev
            prev = cur
        if trial % 5 == 0:                                           # local optimality (exhaustive)
            Mf = b.medoids.tolist()
            for i in range(k):
                for x in range(n):
                    if x not in Mf:
                        assert bf_delta(D, Mf, i, x) >= 0
            assert b.assignment.tolist() == oracle.assign(D, Mf).nearest.tolist()


def test_best_swap_key_is_delta_slot_candidate():
    """Reading R1: on exact ties the smaller slot, then the smaller candidate wins."""
    rng = np.random.default_rng(5)
    seen_tie = 0
    for _ in range(300):
        n = int(rng.integers(6, 16))
        k = int(rng.integers(2, 5))
        D = rand_int_matrix(rng, n, hi=4)
        M = rng.choice(n, size=k, replace=False)
        c = oracle.assign(D, M)
        R = oracle.removal_loss(c, k)
        cands = [(bf_delta(D, M, i, x), i, x) for i in range(k) for x in range(n) if x not in M]
        best = min(cands)
        if sum(1 for t in cands if t[0] == best[0]) > 1:
            seen_tie += 1
        got_p = oracle.pam_best(D, M, c)
        got_f = oracle.fastpam1_best(D, M, c, R)
        if best[0] < 0:
            assert (got_p[0], got_p[1], got_p[2]) == best
            assert (got_f[0], got_f[1], got_f[2]) == best
        else:
            assert got_p[1] == -1 and got_f[1] == -1
    assert seen_tie > 20


def test_degenerate_inputs():
    # all-zero matrix: every dTD is 0, nothing is accepted (strict <)
    D = np.zeros((7, 7), np.uint32)
    r = oracle.swap_run(D, [0, 1, 2], oracle.FASTPAM1)
    assert r.n_swaps == 0 and r.n_iter == 1 and r.td == 0
    # exact duplicate points: the duplicate of a medoid is a valid candidate with dTD 0
    D = line_matrix([0, 0, 5, 5, 9])
    r = oracle.swap_run(D, [0, 2], oracle.FASTPAM1)
    assert r.td == bf_td(D, r.medoids)
    # k = n - 1
    D = line_matrix([0, 1, 3, 7, 15])
    r = oracle.swap_run(D, [0, 1, 2, 3], oracle.PAM)
    r2 = oracle.swap_run(D, [0, 1, 2, 3], oracle.FASTPAM1)
    assert r.trace == r2.trace and r.td == min(bf_td(D, list(s)) for s in itertools.combinations(range(5), 4))
    with pytest.raises(ValueError):
        oracle.swap_run(D, [0], oracle.FASTPAM1)


# ---------- BUILD (Alg.1) ----------

def test_build_is_greedy_exact_td_reduction():
    """Reading R3: each BUILD step adds argmin_c TD(M + {c}) (exact TD change, smallest c)."""
    rng = np.random.default_rng(17)
    for trial in range(60):
        n = int(rng.integers(4, 25))
        k = int(rng.integers(1, min(7, n - 1) + 1))
        D = rand_int_matrix(rng, n, hi=int(rng.choice([4, 100])), symmetric=bool(trial % 3))
        M, td, gains = oracle.build_init(D, k)
        # first medoid: smallest column sum, smallest index on ties
        sums = [int(D[:, c].sum()) for c in range(n)]
        assert M[0] == int(np.argmin(sums)) and gains[0] == min(sums)
        cur = [int(M[0])]
        for i in range(1, k):
            opts = [(bf_td(D, cur + [c]) - bf_td(D, cur), c) for c in range(n) if c not in cur]
            g, cbest = min(opts)
            assert (gains[i], M[i]) == (g, cbest)
            cur.append(cbest)
        assert td == bf_td(D, cur)
        assert len(set(M.tolist())) == k


# ---------- float path ----------

def test_float_path_bruteforce_and_traces():
    rng = np.random.default_rng(99)
    for trial in range(40):
        n = int(rng.integers(8, 30))
        k = int(rng.integers(2, 6))
        X = rng.normal(size=(n, 3))
        D = np.sqrt(((X[:, None, :] - X[None, :, :]) ** 2).sum(-1)).astype(np.float32)
        M0 = rng.choice(n, size=k, replace=False)
        c = oracle.assign(D, M0)
        R = oracle.removal_loss(c, k)
        T = oracle.fastpam1_table(D, M0, c, R)
        for i in range(k):
            for x in range(n):
                if x not in M0:
                    assert T[i, x] == pytest.approx(bf_delta(D, M0, i, x), rel=1e-9, abs=1e-9)
        a = oracle.swap_run(D, M0, oracle.PAM)
        b = oracle.swap_run(D, M0, oracle.FASTPAM1)
        assert [t[:2] for t in a.trace] == [t[:2] for t in b.trace]
        assert b.td == pytest.approx(bf_td(D, b.medoids), rel=1e-12)


# ---------- FastPAM2 (reading R6; parity unpinned by the paper) ----------

def test_fastpam2_reading_properties():
    rng = np.random.default_rng(45)
    for trial in range(80):
        n = int(rng.integers(10, 40))
        k = int(rng.integers(2, 8))
        D = rand_int_matrix(rng, n, hi=int(rng.choice([6, 200])))
        M0 = rng.choice(n, size=k, replace=False)
        r2 = oracle.swap_run(D, M0, oracle.FASTPAM2)
        r1 = oracle.swap_run(D, M0, oracle.FASTPAM1)
        if r1.trace:
            assert r2.trace[0] == r1.trace[0]             # first swap = FastPAM1's choice
        M = list(M0)
        for (i, c, dtd) in r2.trace:                       # every applied dTD is exact and < 0
            assert c not in M and dtd == bf_delta(D, M, i, c) and dtd < 0
            M[i] = c
        assert M == r2.medoids.tolist()
        assert r2.td == bf_td(D, M)
        for i in range(k):                                 # final state is a local optimum
            for x in range(n):
                if x not in M:
                    assert bf_delta(D, M, i, x) >= 0
        assert r2.converged and r2.n_iter >= 1


def bf_fastpam2(D, M0, max_iter=2000, eps_rel=None):
    """FastPAM2 as DESIGN.md reading R6 states it,
    written from the definitions only -- every dTD is a full recomputation of
    TD (Eq. eqn:td), no cache, no removal loss, no FastPAM1 vector:

    1-3. per slot i, (v_i, c_i) = lexicographic min over non-medoid c of
         (TD(M with m_i <- c) - TD(M), c);
    4.   stop if no v_i improves;
    5.   slots in ascending (v_i, i);
    6.   the first is applied with v_i;
    7.   every later slot whose v_i improved at the start of the iteration is
         skipped if c_i is a medoid by now, else re-evaluated on the current
         medoids and applied iff that value improves.
    Returns (medoids, td, n_iter, trace[(i, c, dTD)], converged)."""
    Dw = D.astype(np.int64) if D.dtype == np.uint32 else D.astype(np.float64)
    n = D.shape[0]
    M = list(M0)
    k = len(M)

    def td_of(MM):
        return Dw[:, MM].min(axis=1).sum()

    def improving(v, t):
        return v < 0 if eps_rel is None else v < -eps_rel * abs(t)

    def delta(MM, i, c):
        M2 = list(MM)
        M2[i] = c
        return td_of(M2) - td_of(MM)

    td = td_of(M)
    trace, iters, converged = [], 0, False
    while iters < max_iter:
        iters += 1
        best = []
        for i in range(k):
            vals = [(delta(M, i, c), c) for c in range(n) if c not in M]
            best.append(min(vals))
        if not any(improving(v, td) for v, _ in best):
            converged = True
            break
        td0 = td
        order = sorted(range(k), key=lambda i: (best[i][0], i))
        for r, i in enumerate(order):
            v, c = best[i]
            if not improving(v, td0):
                continue
            if r > 0:
                if c in M:
                    continue
                v = delta(M, i, c)
                if not improving(v, td):
                    continue
            trace.append((i, c, v))
            M[i] = c
            td = td_of(M)
    return M, td, iters, trace, converged


@pytest.mark.parametrize("symmetric", [True, False])
def test_fastpam2_equals_bruteforce_reading_r6(symmetric):
    """The oracle's FastPAM2 procedure (swap ORDER, skips and re-evaluations,
    not only its end state) equals bf_fastpam2, a from-definition restatement
    of reading R6, on integer instances with many exact ties (values 0..3)
    and without them."""
    rng = np.random.default_rng(620 + symmetric)
    multi = 0
    for trial in range(80):
        n = int(rng.integers(8, 30))
        k = int(rng.integers(2, min(8, n - 2) + 1))
        D = rand_int_matrix(rng, n, hi=int(rng.choice([4, 4, 30, 1000])), symmetric=symmetric)
        M0 = rng.choice(n, size=k, replace=False).tolist()
        r = oracle.swap_run(D, M0, oracle.FASTPAM2)
        M, td, iters, trace, conv = bf_fastpam2(D, M0)
        assert [tuple(t) for t in r.trace] == trace
        assert r.medoids.tolist() == M and r.td == td
        assert r.n_iter == iters and r.converged == conv
        assert r.assignment.tolist() == oracle.assign(D, M).nearest.tolist()
        if r.n_swaps > r.n_iter - 1 + (not r.converged):
            multi += 1             # some iteration applied more than one swap
    assert multi > 20


def test_fastpam2_float_equals_bruteforce_reading_r6():
    rng = np.random.default_rng(626)
    for _ in range(30):
        n = int(rng.integers(10, 28))
        k = int(rng.integers(2, 6))
        X = rng.normal(size=(n, 3))
        D = np.sqrt(((X[:, None, :] - X[None, :, :]) ** 2).sum(-1)).astype(np.float32)
        M0 = rng.choice(n, size=k, replace=False).tolist()
        r = oracle.swap_run(D, M0, oracle.FASTPAM2)
        M, td, iters, trace, conv = bf_fastpam2(D, M0, eps_rel=oracle.EPS_REL)
        assert [t[:2] for t in r.trace] == [t[:2] for t in trace]
        assert np.allclose([t[2] for t in r.trace], [t[2] for t in trace], rtol=0, atol=1e-9)
        assert r.medoids.tolist() == M and r.td == pytest.approx(td, rel=1e-12)
        assert r.n_iter == iters and r.converged == conv


def test_bf_fastpam2_detects_injected_deviations():
    """bf_fastpam2 is sensitive to the two alternatives R6 rules out (slot
    order instead of dTD order; no re-evaluation): on the same instances both
    alternatives produce a different trace somewhere."""
    rng = np.random.default_rng(627)

    def variant(D, M0, by_slot=False, reeval=True):
        Dw = D.astype(np.int64)
        M = list(M0)
        n, k = D.shape[0], len(M)
        td_of = lambda MM: Dw[:, MM].min(axis=1).sum()
        trace = []
        for _ in range(100):
            best = []
            for i in range(k):
                best.append(min((td_of(M[:i] + [c] + M[i + 1:]) - td_of(M), c) for c in range(n) if c not in M))
            if not any(v < 0 for v, _ in best):
                break
            order = sorted(range(k), key=(lambda i: i) if by_slot else (lambda i: (best[i][0], i)))
            for r, i in enumerate(order):
                v, c = best[i]
                if v >= 0 or c in M:
                    continue
                if reeval and r > 0:
                    v = td_of(M[:i] + [c] + M[i + 1:]) - td_of(M)
                    if v >= 0:
                        continue
                trace.append((i, c))
                M[i] = c
        return trace

    diff_order = diff_reeval = 0
    for _ in range(40):
        n = int(rng.integers(12, 30))
        k = int(rng.integers(3, 7))
        D = rand_int_matrix(rng, n, hi=1000)
        M0 = rng.choice(n, size=k, replace=False).tolist()
        ref = [t[:2] for t in bf_fastpam2(D, M0)[3]]
        diff_order += variant(D, M0, by_slot=True) != ref
        diff_reeval += variant(D, M0, reeval=False) != ref
    assert diff_order > 5 and diff_reeval > 5


def test_candidate_col_and_assign_cols_equal_definitions():
    """oracle.fastpam1_candidate_col (explicit column) and oracle.assign_cols
    (explicit medoid columns) against brute force: vec[i] + plus is the exact
    TD change of swapping slot i for the column's point, and the cache is the
    sorted (d, slot) order."""
    rng = np.random.default_rng(628)
    for trial in range(60):
        n = int(rng.integers(5, 20))
        k = int(rng.integers(2, min(6, n - 1) + 1))
        D = rand_int_matrix(rng, n, hi=int(rng.choice([4, 50])), symmetric=bool(trial % 2))
        M = rng.choice(n, size=k, replace=False)
        cols = np.ascontiguousarray(D[:, M].T)
        c = oracle.assign_cols(cols)
        for o in range(n):
            order = sorted(range(k), key=lambda j: (int(D[o, M[j]]), j))
            assert (c.nearest[o], c.second[o]) == (order[0], order[1])
            assert (c.dn[o], c.ds[o]) == (D[o, M[order[0]]], D[o, M[order[1]]])
        R = oracle.removal_loss(c, k)
        for x in range(n):
            if x in M:
                continue
            vec, plus = oracle.fastpam1_candidate_col(np.ascontiguousarray(D[:, x]), c, R)
            assert [int(v + plus) for v in vec] == [bf_delta(D, M, i, x) for i in range(k)]


# ---------- FasterPAM (Alg.4; readings F1-F5) ----------

def bf_eager(D, M0, max_iter=2000, eps_rel=None):
    """Eager swapping written from the definitions only: for every scan
    position t (candidate c = t mod n, medoids skipped), the change of TD for
    replacing each slot i by c is recomputed from scratch (Eq. eqn:td); the
    best slot (smaller slot on ties) is swapped in if it lowers TD.  Stops at
    the first position n past the last swap (readings F1-F3)."""
    n = D.shape[0]
    Dw = D.astype(np.int64) if D.dtype == np.uint32 else D.astype(np.float64)
    M = list(M0)

    def td_of(MM):
        return Dw[:, MM].min(axis=1).sum()

    td = td_of(M)
    t = t_last = 0
    trace = []
    converged = True
    while True:
        if t - t_last == n:
            break
        if t % n == 0 and t // n >= max_iter:
            converged = False
            break
        c = t % n
        if c not in M:
            deltas = []
            for i in range(len(M)):
                M2 = list(M)
                M2[i] = c
                deltas.append(td_of(M2) - td)
            i = int(np.argmin(deltas))      # first minimum = smaller slot
            v = deltas[i]
            ok = v < 0 if eps_rel is None else v < -eps_rel * abs(td)
            if ok:
                trace.append((i, c, v, t))
                M[i] = c
                td = td_of(M)
                t_last = t
        t += 1
    return M, td, (t + n - 1) // n, trace, converged


def _check_eager(D, M0, float_tol=None, **kw):
    r = oracle.fasterpam_run(D, M0, **kw)
    M, td, iters, trace, conv = bf_eager(D, M0, eps_rel=None if float_tol is None else oracle.EPS_REL, **kw)
    assert r.medoids.tolist() == M
    assert [(a, b, d) for a, b, _, d in r.trace] == [(a, b, d) for a, b, _, d in trace]
    if float_tol is None:
        assert [v for _, _, v, _ in r.trace] == [v for _, _, v, _ in trace]
        assert r.td == td
    else:
        assert np.allclose([v for _, _, v, _ in r.trace], [v for _, _, v, _ in trace], rtol=0, atol=float_tol)
        assert abs(r.td - td) <= float_tol
    assert r.n_iter == iters and r.n_swaps == len(trace) and r.converged == conv
    return r


@pytest.mark.parametrize("symmetric", [True, False])
def test_fasterpam_equals_bruteforce_eager(symmetric):
    rng = np.random.default_rng(41 + symmetric)
    for _ in range(60):
        n = int(rng.integers(6, 28))
        k = int(rng.integers(2, min(6, n - 1) + 1))
        D = rand_int_matrix(rng, n, hi=int(rng.choice([4, 30, 1000])), symmetric=symmetric)
        M0 = rng.choice(n, k, replace=False).tolist()
        r = _check_eager(D, M0)
        # several swaps per pass; the result is a local optimum
        for i in range(k):
            for c in range(n):
                if c not in r.medoids.tolist():
                    assert bf_delta(D, r.medoids.tolist(), i, c) >= 0
        assert oracle.td(D, r.medoids) == r.td
        assert r.assignment.tolist() == oracle.assign(D, r.medoids).nearest.tolist()


def test_fasterpam_float_equals_bruteforce_eager():
    rng = np.random.default_rng(7)
    for _ in range(30):
        n = int(rng.integers(8, 26))
        k = int(rng.integers(2, 5))
        X = rng.normal(size=(n, 3))
        D = np.sqrt(((X[:, None, :] - X[None, :, :]) ** 2).sum(-1)).astype(np.float32)
        M0 = rng.choice(n, k, replace=False).tolist()
        _check_eager(D, M0, float_tol=1e-9)


def test_fasterpam_max_iter_and_termination():
    rng = np.random.default_rng(3)
    D = rand_int_matrix(rng, 40, hi=1000)
    M0 = [0, 1, 2, 3]
    full = _check_eager(D, M0)
    assert full.converged and full.n_swaps >= full.n_iter - 1
    capped = _check_eager(D, M0, max_iter=1)
    assert capped.n_iter == 1 and not capped.converged
    # a start at the optimum: one pass, no swap (F2 with x_last invalid)
    again = _check_eager(D, full.medoids.tolist())
    assert again.n_swaps == 0 and again.n_iter == 1 and again.converged


def test_fasterpam_fig1_reaches_the_optimum():
    """SPEC fasterpam_swap example: the Fig.1 instance (reading R7),
    started at its 'Loss: 10' configuration, ends at the exhaustive optimum."""
    g = _gold("fig1_alternating.json")
    D = line_matrix(g["points"])
    r = _check_eager(D, g["medoids"])
    best = min(bf_td(D, list(S)) for S in itertools.combinations(range(len(g["points"])), 2))
    assert best == g["losses"][-1]
    assert r.td == best


# ---------- dissimilarity matrix from points (NEXT-2) ----------

def test_dist_oracle_closed_forms_and_library():
    """oracle.dist_l2 / dist_l1 against closed forms (3-4-5, unit square) and
    scipy's cdist (a library routine of the same definitions), plus the metric
    axioms: zero diagonal, symmetry, triangle inequality."""
    from scipy.spatial.distance import cdist
    X = np.array([[0, 0], [3, 4], [0, 1], [1, 0]], np.float32)
    D = oracle.dist_l2(X)
    assert D[0, 1] == 5.0 and D[2, 3] == np.sqrt(2.0) and D[1, 2] == np.sqrt(9 + 9)
    Xq = np.array([[0, 0], [3, -4], [-1, 2]], np.int32)
    assert oracle.dist_l1(Xq).tolist() == [[0, 7, 3], [7, 0, 10], [3, 10, 0]]
    rng = np.random.default_rng(17)
    for n, d in [(1, 3), (40, 1), (57, 13), (80, 64)]:
        X = rng.normal(size=(n, d)).astype(np.float32)
        D = oracle.dist_l2(X)
        assert np.allclose(D, cdist(X.astype(np.float64), X.astype(np.float64)), rtol=1e-12, atol=1e-12)
        assert (np.diag(D) == 0).all() and (D == D.T).all()
        if n >= 3:
            i, j, l = rng.integers(0, n, size=(3, 200))
            assert (D[i, j] <= D[i, l] + D[l, j] + 1e-12).all()
        Xq = rng.integers(-5000, 5000, size=(n, d)).astype(np.int32)
        assert (oracle.dist_l1(Xq) == cdist(Xq, Xq, "cityblock").astype(np.int64)).all()


# ---------- NEXT-4 initialisations (readings I1, I2) ----------

def test_init_weighted_hand_example_and_intervals():
    """Distance-weighted seeding: the 1-D example by hand, and for every
    candidate c the uniform u at the middle of its interval
    [prefix(c-1), prefix(c)) / W picks exactly c (sampling proportional to
    the distance to the nearest seed)."""
    x = np.array([0, 1, 2, 10, 11, 30])
    D = np.abs(x[:, None] - x[None, :]).astype(np.uint32)
    assert oracle.init_weighted(D, 3, [0.0, 0.5, 0.99]).tolist() == [0, 5, 4]
    rng = np.random.default_rng(4)
    D = rand_int_matrix(rng, 40, 100)
    first = 7
    w = D[:, first].astype(np.int64)
    pref = np.cumsum(w)
    for c in range(40):
        if w[c] == 0:
            continue
        u1 = (pref[c] - w[c] / 2) / pref[-1]
        M = oracle.init_weighted(D, 2, [(first + 0.5) / 40, u1])
        assert M.tolist() == [first, c]
    # all points identical: W = 0 -> smallest non-medoids
    Z = np.zeros((6, 6), np.uint32)
    assert oracle.init_weighted(Z, 3, [0.5, 0.3, 0.3]).tolist() == [3, 0, 1]


@pytest.mark.parametrize("seed", range(4))
def test_init_lab_with_full_samples_equals_build(seed):
    """LAB restricted to a sample equal to all points is PAM BUILD (Alg.1,
    P:281-318, reading R3): same medoids for integer and float inputs."""
    rng = np.random.default_rng(900 + seed)
    n, k = int(rng.integers(8, 60)), int(rng.integers(1, 6))
    D = rand_int_matrix(rng, n, int(rng.choice([5, 1000])), symmetric=bool(seed % 2))
    rows = np.stack([np.concatenate([rng.permutation(n), -np.ones(k, np.int64)]) for _ in range(k)]).astype(np.int32)
    Mb, _, _ = oracle.build_init(D, k)
    assert oracle.init_lab(D, k, n, rows).tolist() == Mb.tolist()
    Df = (D.astype(np.float32) * 0.37).astype(np.float32)
    Mbf, _, _ = oracle.build_init(Df, k)
    assert oracle.init_lab(Df, k, n, rows).tolist() == Mbf.tolist()


# ---------- NEXT-3 FastCLARA (reading C1) ----------

def test_clara_full_sample_is_pam_and_best_sample_wins():
    """A single sample holding every point makes CLARA the PAM of the whole
    set (BUILD + FastPAM1, pinned above); with several samples the returned
    TD is the definition's TD of the returned medoids and no sample's
    solution has a smaller TD."""
    rng = np.random.default_rng(61)
    n, k = 90, 4
    D = rand_int_matrix(rng, n, 300)
    t, j, M = oracle.clara(D, k, [np.arange(n)])
    Mb, _, _ = oracle.build_init(D, k)
    ref = oracle.swap_run(D, Mb, oracle.FASTPAM1)
    assert j == 0 and M.tolist() == ref.medoids.tolist() and t == ref.td
    samples = [rng.choice(n, size=30, replace=False) for _ in range(5)]
    t, j, M = oracle.clara(D, k, samples)
    assert t == bf_td(D, M)
    for S in samples:
        Dj = np.ascontiguousarray(D[np.ix_(S, S)])
        Mj, _, _ = oracle.build_init(Dj, k)
        rj = oracle.swap_run(Dj, Mj, oracle.FASTPAM1)
        assert bf_td(D, S[rj.medoids]) >= t


def test_fastpam2_slot_best_equals_bruteforce():
    """Reading R6 steps 2-3 (oracle.fastpam2_slot_best, the per-slot plan the
    full-size goldens record): (v_i, c_i) = lexicographic min over non-medoid
    c of (TD(M with m_i <- c) - TD(M), c), recomputed from the definition."""
    rng = np.random.default_rng(629)
    for trial in range(60):
        n = int(rng.integers(6, 22))
        k = int(rng.integers(2, min(6, n - 1) + 1))
        D = rand_int_matrix(rng, n, hi=int(rng.choice([4, 100])), symmetric=bool(trial % 2))
        M = rng.choice(n, size=k, replace=False)
        c = oracle.assign(D, M)
        sv, sc = oracle.fastpam2_slot_best(D, M, c, oracle.removal_loss(c, k))
        for i in range(k):
            assert (sv[i], sc[i]) == min((bf_delta(D, M, i, x), x) for x in range(n) if x not in M)


# ---------- NEXT-3 FastCLARA from points (reading C2) ----------

def _cdist_f32(X):
    from scipy.spatial.distance import cdist
    return cdist(X.astype(np.float64), X.astype(np.float64)).astype(np.float32)


def _cdist_u32(Xq):
    from scipy.spatial.distance import cdist
    return cdist(Xq, Xq, "cityblock").astype(np.uint32)


@pytest.mark.parametrize("metric", ["l1", "l2"])
def test_td_points_equals_td_of_the_matrix(metric):
    """oracle.td_points (distances recomputed from the points) equals the
    definition's TD on the dissimilarity matrix built by scipy (a library
    routine of the same distances), with the assignment = sorted (d, slot)."""
    rng = np.random.default_rng(71)
    for n, d, k in [(40, 3, 4), (97, 8, 7), (150, 1, 2)]:
        if metric == "l2":
            X = rng.normal(size=(n, d)).astype(np.float32)
            D = _cdist_f32(X)
        else:
            X = rng.integers(-300, 300, size=(n, d)).astype(np.int32)
            D = _cdist_u32(X)
        M = rng.choice(n, size=k, replace=False)
        t, mins, asg = oracle.td_points(X, metric, M)
        ref = bf_td(D, M)
        if metric == "l2":
            assert t == pytest.approx(ref, rel=1e-12)
        else:
            assert t == ref
        for o in range(n):
            order = sorted(range(k), key=lambda j: (D[o, M[j]], j))
            assert asg[o] == order[0] and mins[o] == D[o, M[order[0]]]


@pytest.mark.parametrize("metric", ["l1", "l2"])
def test_clara_points_full_sample_is_pam_and_best_wins(metric):
    """One sample holding every point makes CLARA-from-points the PAM
    (BUILD + FastPAM1) of the whole set on the scipy-built matrix; with
    several samples no sample's PAM solution has a smaller TD over all
    points than the one returned."""
    rng = np.random.default_rng(72)
    n, d, k = 70, 4, 3
    if metric == "l2":
        X = rng.normal(size=(n, d)).astype(np.float32)
        D = _cdist_f32(X)
    else:
        X = rng.integers(0, 500, size=(n, d)).astype(np.int32)
        D = _cdist_u32(X)
    t, j, M, asg = oracle.clara_points(X, metric, k, [np.arange(n)])
    Mb, _, _ = oracle.build_init(D, k)
    ref = oracle.swap_run(D, Mb, oracle.FASTPAM1)
    assert j == 0 and M.tolist() == ref.medoids.tolist()
    assert (t == ref.td) if metric == "l1" else t == pytest.approx(ref.td, rel=1e-12)
    samples = [rng.choice(n, size=25, replace=False) for _ in range(4)]
    t, j, M, asg = oracle.clara_points(X, metric, k, samples)
    assert (t == bf_td(D, M)) if metric == "l1" else t == pytest.approx(bf_td(D, M), rel=1e-12)
    for S in samples:
        Dj = np.ascontiguousarray(D[np.ix_(S, S)])
        Mj, _, _ = oracle.build_init(Dj, k)
        rj = oracle.swap_run(Dj, Mj, oracle.FASTPAM1)
        assert bf_td(D, S[rj.medoids]) >= t - 1e-9
