"""CPU oracle for FastPAM SWAP / BUILD (Schubert & Rousseeuw, arXiv 2008.05171).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2008_05171_b200``) never imports it, and
it never imports the product path: the two share no code.

This module is argument marshalling (ctypes) around ``liboracle.so``, the
plain single-threaded C restatement of the paper in ``oracle_impl.h``.  The
library is compiled on first use with ``gcc -O2`` if it is missing or older
than its sources.

Conventions (reading R0): ``D`` is an ``(n, n)`` numpy array of
``uint32`` or ``float32`` whose rows may be padded (``D.strides[0]`` may exceed
``n * itemsize``); ``d(x_o, x_c) = D[o, c]``.  uint32 inputs accumulate in
int64, float32 inputs in float64.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRCS = [os.path.join(_HERE, f) for f in ("oracle.c", "oracle_impl.h")]

PAM, FASTPAM1, FASTPAM2 = 0, 1, 2
EPS_REL = 1e-12  # reading R5: float acceptance margin (same value as oracle.c)


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain gcc (IEEE semantics, no fast-math)."""
    newest = max(os.path.getmtime(s) for s in _SRCS)
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c99", "-Wall", "-shared", "-fPIC", "-o", tmp,
             os.path.join(_HERE, "oracle.c"), "-lm"])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
    return _lib


_I32P = ctypes.POINTER(ctypes.c_int32)


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _sfx(D: np.ndarray) -> tuple[str, type]:
    if D.dtype == np.uint32:
        return "_u32", np.int64
    if D.dtype == np.float32:
        return "_f32", np.float64
    raise TypeError(f"oracle supports uint32/float32 dissimilarities, got {D.dtype}")


def _ld(D: np.ndarray) -> int:
    if D.ndim != 2 or D.shape[0] != D.shape[1]:
        raise ValueError("D must be (n, n) (rows may be padded via strides)")
    if D.strides[1] != D.itemsize or D.strides[0] % D.itemsize:
        raise ValueError("D rows must be contiguous")
    return D.strides[0] // D.itemsize


def _fn(D, name):
    sfx, acc = _sfx(D)
    return getattr(_load(), name + sfx), acc


def _acc_ctype(acc):
    return ctypes.c_int64 if acc is np.int64 else ctypes.c_double


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def td(D: np.ndarray, M) -> int | float:
    """Eq. eqn:td."""
    f, acc = _fn(D, "oracle_td")
    f.restype = _acc_ctype(acc)
    M = _i32(M)
    return f(_ptr(D), ctypes.c_int64(_ld(D)), ctypes.c_int32(D.shape[0]), _ptr(M),
             ctypes.c_int32(len(M)))


@dataclass
class Cache:
    """nearest/second slot and distances per object (Alg.2)."""
    nearest: np.ndarray
    second: np.ndarray
    dn: np.ndarray
    ds: np.ndarray


def assign(D: np.ndarray, M) -> Cache:
    f, acc = _fn(D, "oracle_assign")
    f.restype = ctypes.c_int
    M = _i32(M)
    n = D.shape[0]
    near = np.empty(n, np.int32); sec = np.empty(n, np.int32)
    dn = np.empty(n, acc); ds = np.empty(n, acc)
    rc = f(_ptr(D), ctypes.c_int64(_ld(D)), ctypes.c_int32(n), _ptr(M), ctypes.c_int32(len(M)),
           _ptr(near), _ptr(sec), _ptr(dn), _ptr(ds))
    if rc != 0:
        raise ValueError("assign needs k >= 2")
    return Cache(near, sec, dn, ds)


def removal_loss(cache: Cache, k: int) -> np.ndarray:
    """dTD^{-m_i}."""
    acc = cache.dn.dtype.type
    f = getattr(_load(), "oracle_removal_loss" + ("_u32" if acc is np.int64 else "_f32"))
    R = np.empty(k, acc)
    n = len(cache.nearest)
    f(ctypes.c_int32(n), ctypes.c_int32(k), _ptr(cache.nearest), _ptr(cache.dn), _ptr(cache.ds), _ptr(R))
    return R


def change(doc, nearest_o: int, dn_o, ds_o, i: int, dtype=np.uint32):
    """Four-case change function, Eq. eqn:change."""
    f = getattr(_load(), "oracle_change" + ("_u32" if dtype == np.uint32 else "_f32"))
    ct = ctypes.c_int64 if dtype == np.uint32 else ctypes.c_double
    f.restype = ct
    f.argtypes = [ct, ctypes.c_int32, ct, ct, ctypes.c_int32]
    return f(doc, nearest_o, dn_o, ds_o, i)


def fastpam1_candidate(D: np.ndarray, c: int, cache: Cache, R: np.ndarray):
    """Alg.3 P:879-891 for one candidate: returns (vec[k] = dTD_i, plus = dTD^{+x_c})."""
    f, acc = _fn(D, "oracle_fastpam1_candidate")
    k = len(R)
    vec = np.empty(k, acc); plus = np.zeros(1, acc)
    f(_ptr(D), ctypes.c_int64(_ld(D)), ctypes.c_int32(D.shape[0]), ctypes.c_int32(k), ctypes.c_int32(c),
      _ptr(cache.nearest), _ptr(cache.dn), _ptr(cache.ds), _ptr(np.ascontiguousarray(R, acc)),
      _ptr(vec), _ptr(plus))
    return vec, plus[0]


def fastpam1_candidate_col(col: np.ndarray, cache: Cache, R: np.ndarray):
    """Same as fastpam1_candidate with col[o] = d(x_o, x_c) given explicitly."""
    col = np.ascontiguousarray(col)
    sfx, acc = _sfx(col.reshape(1, -1))
    f = getattr(_load(), "oracle_fastpam1_candidate_col" + sfx)
    k = len(R)
    vec = np.empty(k, acc); plus = np.zeros(1, acc)
    f(_ptr(col), ctypes.c_int32(len(col)), ctypes.c_int32(k), _ptr(cache.nearest), _ptr(cache.dn),
      _ptr(cache.ds), _ptr(np.ascontiguousarray(R, acc)), _ptr(vec), _ptr(plus))
    return vec, plus[0]


def assign_cols(cols: np.ndarray) -> Cache:
    """Cache from explicit medoid columns cols[j, o] = d(x_o, m_j) (same rule as assign)."""
    k, n = cols.shape
    # An (n, k) view whose column j is medoid j: D'[o, j] = cols[j, o].
    Dp = np.ascontiguousarray(cols.T)
    f, acc = _fn(Dp, "oracle_assign")
    near = np.empty(n, np.int32); sec = np.empty(n, np.int32)
    dn = np.empty(n, acc); ds = np.empty(n, acc)
    M = np.arange(k, dtype=np.int32)
    f.restype = ctypes.c_int
    rc = f(_ptr(Dp), ctypes.c_int64(k), ctypes.c_int32(n), _ptr(M), ctypes.c_int32(k),
           _ptr(near), _ptr(sec), _ptr(dn), _ptr(ds))
    if rc != 0:
        raise ValueError("assign needs k >= 2")
    return Cache(near, sec, dn, ds)


def _best(name, D, M, cache, R=None):
    f, acc = _fn(D, name)
    f.restype = ctypes.c_int
    M = _i32(M)
    bd = np.zeros(1, acc); bi = np.zeros(1, np.int32); bc = np.zeros(1, np.int32)
    args = [_ptr(D), ctypes.c_int64(_ld(D)), ctypes.c_int32(D.shape[0]), _ptr(M), ctypes.c_int32(len(M)),
            _ptr(cache.nearest), _ptr(cache.dn), _ptr(cache.ds)]
    if R is not None:
        args.append(_ptr(np.ascontiguousarray(R, acc)))
    f(*args, _ptr(bd), _ptr(bi), _ptr(bc))
    return bd[0], int(bi[0]), int(bc[0])


def pam_best(D, M, cache):
    """Alg.2 P:351-364 best swap (dTD*, slot, candidate); slot = -1 if none < 0."""
    return _best("oracle_pam_best", D, M, cache)


def fastpam1_best(D, M, cache, R):
    """Alg.3 P:876-897 best swap under key (dTD, i, c)."""
    return _best("oracle_fastpam1_best", D, M, cache, R)


def fastpam1_table(D, M, cache, R) -> np.ndarray:
    """table[i, c] = dTD(m_i, x_c) for non-medoid c (medoid columns = NaN / int64 max)."""
    f, acc = _fn(D, "oracle_fastpam1_table")
    M = _i32(M)
    n, k = D.shape[0], len(M)
    fill = np.iinfo(np.int64).max if acc is np.int64 else np.nan
    table = np.full((k, n), fill, acc)
    f(_ptr(D), ctypes.c_int64(_ld(D)), ctypes.c_int32(n), _ptr(M), ctypes.c_int32(k),
      _ptr(cache.nearest), _ptr(cache.dn), _ptr(cache.ds), _ptr(np.ascontiguousarray(R, acc)), _ptr(table))
    return table


def fastpam2_slot_best(D, M, cache, R):
    """Reading R6 steps 2-3: per slot i, (v_i, c_i) = lexicographic min over
    non-medoid c of (dTD(m_i, x_c), c).  Returns (v[k], c[k])."""
    f, acc = _fn(D, "oracle_fastpam2_slot_best")
    M = _i32(M)
    k = len(M)
    sv = np.zeros(k, acc); sc = np.zeros(k, np.int32)
    f(_ptr(D), ctypes.c_int64(_ld(D)), ctypes.c_int32(D.shape[0]), _ptr(M), ctypes.c_int32(k),
      _ptr(cache.nearest), _ptr(cache.dn), _ptr(cache.ds), _ptr(np.ascontiguousarray(R, acc)), _ptr(sv), _ptr(sc))
    return sv, sc


@dataclass
class RunResult:
    medoids: np.ndarray
    assignment: np.ndarray
    td: int | float
    n_iter: int
    n_swaps: int
    converged: bool
    trace: list = field(default_factory=list)   # [(slot, candidate, dTD)]


def swap_run(D: np.ndarray, M0, variant: int = FASTPAM1, max_iter: int = 2000) -> RunResult:
    """SWAP to convergence: variant PAM (Alg.2), FASTPAM1 (Alg.3), FASTPAM2 (reading R6)."""
    f, acc = _fn(D, "oracle_swap_run")
    f.restype = ctypes.c_int
    M = _i32(M0).copy()
    n, k = D.shape[0], len(M)
    cap = 1 << 20
    ti = np.zeros(cap, np.int32); tc = np.zeros(cap, np.int32); tdv = np.zeros(cap, acc)
    it = np.zeros(1, np.int32); sw = np.zeros(1, np.int32); tdo = np.zeros(1, acc)
    asg = np.zeros(n, np.int32)
    rc = f(_ptr(D), ctypes.c_int64(_ld(D)), ctypes.c_int32(n), _ptr(M), ctypes.c_int32(k),
           ctypes.c_int32(variant), ctypes.c_int32(max_iter), _ptr(ti), _ptr(tc), _ptr(tdv),
           ctypes.c_int32(cap), _ptr(it), _ptr(sw), _ptr(tdo), _ptr(asg))
    if rc < 0:
        raise ValueError("swap_run needs 2 <= k < n")
    ns = int(sw[0])
    trace = [(int(ti[j]), int(tc[j]), tdv[j].item()) for j in range(min(ns, cap))]
    return RunResult(M, asg, tdo[0].item(), int(it[0]), ns, rc == 0, trace)


def fasterpam_run(D: np.ndarray, M0, max_iter: int = 2000) -> RunResult:
    """FasterPAM, Alg.4 with readings F1-F5 (oracle_impl.h).

    ``trace`` entries are (slot, candidate, dTD, scan position t)."""
    f, acc = _fn(D, "oracle_fasterpam_run")
    f.restype = ctypes.c_int
    M = _i32(M0).copy()
    n, k = D.shape[0], len(M)
    cap = 1 << 20
    ti = np.zeros(cap, np.int32); tc = np.zeros(cap, np.int32); tdv = np.zeros(cap, acc)
    tp = np.zeros(cap, np.int64)
    it = np.zeros(1, np.int32); sw = np.zeros(1, np.int32); tdo = np.zeros(1, acc)
    asg = np.zeros(n, np.int32)
    rc = f(_ptr(D), ctypes.c_int64(_ld(D)), ctypes.c_int32(n), _ptr(M), ctypes.c_int32(k),
           ctypes.c_int32(max_iter), _ptr(ti), _ptr(tc), _ptr(tdv), _ptr(tp), ctypes.c_int32(cap),
           _ptr(it), _ptr(sw), _ptr(tdo), _ptr(asg))
    if rc < 0:
        raise ValueError("fasterpam_run needs 2 <= k < n")
    ns = int(sw[0])
    trace = [(int(ti[j]), int(tc[j]), tdv[j].item(), int(tp[j])) for j in range(min(ns, cap))]
    return RunResult(M, asg, tdo[0].item(), int(it[0]), ns, rc == 0, trace)


def build_init(D: np.ndarray, k: int):
    """PAM BUILD, Alg.1 with readings R3/R4.

    Returns (medoids[k], TD, gains[k]) where gains[0] is the first medoid's
    distance sum and gains[i] the dTD* of step i."""
    f, acc = _fn(D, "oracle_build")
    f.restype = ctypes.c_int
    n = D.shape[0]
    M = np.zeros(k, np.int32); tdo = np.zeros(1, acc); gains = np.zeros(k, acc)
    rc = f(_ptr(D), ctypes.c_int64(_ld(D)), ctypes.c_int32(n), ctypes.c_int32(k), _ptr(M), _ptr(tdo), _ptr(gains))
    if rc != 0:
        raise ValueError("build needs 1 <= k < n")
    return M, tdo[0].item(), gains


def dist_l2(X: np.ndarray) -> np.ndarray:
    """Euclidean dissimilarities by definition, fp64 (oracle_dist_l2)."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    n, d = X.shape
    D = np.empty((n, n), np.float64)
    _load().oracle_dist_l2(_ptr(X), ctypes.c_int32(n), ctypes.c_int32(d), _ptr(D))
    return D


def dist_l1(Xq: np.ndarray) -> np.ndarray:
    """Manhattan dissimilarities of integer coordinates by definition, int64 (oracle_dist_l1)."""
    Xq = np.ascontiguousarray(Xq, dtype=np.int32)
    n, d = Xq.shape
    D = np.empty((n, n), np.int64)
    _load().oracle_dist_l1(_ptr(Xq), ctypes.c_int32(n), ctypes.c_int32(d), _ptr(D))
    return D


def init_weighted(D: np.ndarray, k: int, u) -> np.ndarray:
    """Distance-weighted seeding (reading I1) with the uniforms u[k]."""
    f, acc = _fn(D, "oracle_init_weighted")
    f.restype = ctypes.c_int
    M = np.zeros(k, np.int32)
    uu = np.ascontiguousarray(u, np.float64)
    if f(_ptr(D), ctypes.c_int64(_ld(D)), ctypes.c_int32(D.shape[0]), ctypes.c_int32(k), _ptr(uu), _ptr(M)) != 0:
        raise ValueError("init_weighted needs 1 <= k <= n")
    return M


def init_lab(D: np.ndarray, k: int, s: int, seq) -> np.ndarray:
    """LAB (reading I2) with the per-step index rows seq[k][s+k]."""
    f, acc = _fn(D, "oracle_init_lab")
    f.restype = ctypes.c_int
    M = np.zeros(k, np.int32)
    q = np.ascontiguousarray(seq, np.int32)
    if f(_ptr(D), ctypes.c_int64(_ld(D)), ctypes.c_int32(D.shape[0]), ctypes.c_int32(k), ctypes.c_int32(s),
         _ptr(q), _ptr(M)) != 0:
        raise ValueError("init_lab needs 1 <= k <= n, s >= 1")
    return M


def lab_sample_rows(n: int, k: int, seed: int, s: int | None = None):
    """The caller-side random input of LAB: s = 10 + ceil(sqrt(n)) and, per step,
    s + k distinct uniform indices (numpy Generator(PCG64(seed)))."""
    import math
    s = s if s is not None else 10 + math.ceil(math.sqrt(n))
    s = min(s, n)
    rng = np.random.Generator(np.random.PCG64(seed))
    w = min(n, s + k)
    rows = np.stack([rng.choice(n, size=w, replace=False) for _ in range(k)]).astype(np.int32)
    if w < s + k:                                   # fewer than s + k points: pad with -1 (skipped)
        rows = np.concatenate([rows, np.full((k, s + k - w), -1, np.int32)], axis=1)
    return s, rows


def clara(D: np.ndarray, k: int, samples, variant: str = "fastpam1"):
    """FastCLARA (reading C1): PAM (BUILD, Alg.1, then SWAP:
    FastPAM1 Alg.3 or FasterPAM Alg.4) on the sub-matrix D[S][S] of every
    sample S (caller-drawn, distinct indices), medoids mapped back to point
    indices, TD over ALL points (Eq. eqn:td); the sample with the smallest
    (TD, sample index) wins.  Returns (TD, best sample index, medoids)."""
    best = None
    for j, S in enumerate(samples):
        S = np.asarray(S, np.int64)
        Dj = np.ascontiguousarray(D[np.ix_(S, S)])
        Mb, _, _ = build_init(Dj, k)
        r = swap_run(Dj, Mb, FASTPAM1) if variant == "fastpam1" else fasterpam_run(Dj, Mb)
        M = S[r.medoids].astype(np.int32)
        t = td(D, M)
        if best is None or t < best[0]:
            best = (t, j, M)
    return best


def td_points(X: np.ndarray, metric: str, M):
    """TD over all objects from the points (Eq. eqn:td; reading C2): metric
    "l2" (float32 X, d = f32 Euclidean, fp64 sum) or "l1" (int32 X, int64).
    Returns (TD, per-object minimum, assignment slot)."""
    M = _i32(M)
    n, d = X.shape
    asg = np.zeros(n, np.int32)
    if metric == "l2":
        Xc = np.ascontiguousarray(X, dtype=np.float32)
        mins = np.zeros(n, np.float64)
        f = _load().oracle_td_points_l2
        f.restype = ctypes.c_double
    else:
        Xc = np.ascontiguousarray(X, dtype=np.int32)
        mins = np.zeros(n, np.int64)
        f = _load().oracle_td_points_l1
        f.restype = ctypes.c_int64
    t = f(_ptr(Xc), ctypes.c_int32(n), ctypes.c_int32(d), _ptr(M), ctypes.c_int32(len(M)), _ptr(mins), _ptr(asg))
    return t, mins, asg


def sub_dissimilarity(X: np.ndarray, metric: str, S) -> np.ndarray:
    """The sample's dissimilarity matrix from its points by the definitions:
    l2 -> float32 of the fp64 Euclidean distance (oracle.dist_l2), l1 ->
    uint32 of the int64 Manhattan distance (oracle.dist_l1)."""
    S = np.asarray(S, np.int64)
    if metric == "l2":
        return dist_l2(np.ascontiguousarray(X[S], dtype=np.float32)).astype(np.float32)
    D = dist_l1(np.ascontiguousarray(X[S], dtype=np.int32))
    if D.size and D.max() > np.iinfo(np.uint32).max:
        raise ValueError("L1 distances exceed uint32")
    return D.astype(np.uint32)


def clara_points(X: np.ndarray, metric: str, k: int, samples, variant: str = "fastpam1"):
    """FastCLARA without the n x n matrix (
    reading C2): for every caller-drawn sample S, PAM (BUILD, Alg.1, then
    FastPAM1 Alg.3 or FasterPAM Alg.4) on the sample's dissimilarity matrix
    computed from its points, medoids mapped back to point indices, TD over
    ALL n objects from the points (td_points); the smallest (TD, sample index)
    wins.  Returns (TD, best sample index, medoids, assignment of all n)."""
    best = None
    for j, S in enumerate(samples):
        S = np.asarray(S, np.int64)
        Dj = sub_dissimilarity(X, metric, S)
        Mb, _, _ = build_init(Dj, k)
        r = swap_run(Dj, Mb, FASTPAM1) if variant == "fastpam1" else fasterpam_run(Dj, Mb)
        M = S[r.medoids].astype(np.int32)
        t, _, asg = td_points(X, metric, M)
        if best is None or t < best[0]:
            best = (t, j, M, asg)
    return best
