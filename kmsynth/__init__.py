"""Seeded synthetic inputs for the FastPAM SWAP workloads (BASELINE.json configs).

INPUT GENERATOR: shared by the CUDA path's tests/bench and the oracle.  It
holds none of the method's arithmetic -- only point sets, dissimilarity
matrices (the method's *input*) and random initial medoids.

The paper's datasets (ORLib, 100plants, optdigits, MNIST)
are not available; these seeded mixtures stand in for them with the shapes of
BASELINE.json (SURVEY.md 8(d) recipe):

  C1 n=500    2-D  5 centres ~U([0,100]^2), sigma 5, equal weights      -> uint32 L1 x100
  C2 n=5000  10-D 20 centres ~N(0,10^2 I), sigma 1, weights ~Dir(1)     -> float32 Euclidean
  C3 n=20000 27-D 100 prototypes ~Dir(0.3); rows ~Dir(200 P_j + 1e-3)
                  + N(0, 0.002^2), clipped at 0, renormalised           -> float32 Euclidean
  C4 n=50000 32-D 200 centres ~N(0,8^2 I), sigma 1, Dir(1) weights     -> float32 Euclidean
  C5 n=1e5   64-D 95000 inliers from 500 centres ~N(0,6^2 I), sigma 1,
                  Dir(1) weights + 5000 uniform outliers in the inliers'
                  bounding box                                          -> uint32 L1 x100

RNG: numpy Generator(PCG64(20080517 + cfg#)); random initial medoids use
seed + 1000 (k distinct indices, uniform without replacement).

Distances: L1 on integer coordinates round(100 x) is exact integer
arithmetic; Euclidean is f32(sqrt(sum_t (x_ot - x_ct)^2)) with each fp64
operation rounded in t order, so the numpy and CUDA materialisations agree
bit for bit (tests/test_synth.py for the CPU pair, test_gpu_parity.py::
test_synth_cuda_matches_numpy for CUDA).  Both are exactly symmetric with a zero
diagonal.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

L1_INT, L2_F32 = 0, 1

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libkmsynth.so")
_SRC = os.path.join(_HERE, "csrc", "synth_dist.cu")


@dataclass(frozen=True)
class Config:
    cid: int
    name: str
    n: int
    k: int
    dim: int
    metric: int
    init: str            # "build" or "random"
    variants: tuple      # SWAP variants run on this config
    gpus: tuple          # GPU counts BASELINE.json names

    @property
    def seed(self) -> int:
        return 20080517 + self.cid

    @property
    def dtype(self):
        return np.uint32 if self.metric == L1_INT else np.float32


CONFIGS = {
    1: Config(1, "C1", 500, 5, 2, L1_INT, "build", ("fastpam1",), (1,)),
    2: Config(2, "C2", 5000, 20, 10, L2_F32, "build", ("fastpam1",), (1,)),
    3: Config(3, "C3", 20000, 100, 27, L2_F32, "random", ("fastpam1", "fastpam2"), (1,)),
    4: Config(4, "C4", 50000, 200, 32, L2_F32, "build", ("fastpam1",), (1, 2, 4, 8)),
    5: Config(5, "C5", 100000, 500, 64, L1_INT, "random", ("fastpam2",), (1, 2, 4, 8)),
}


def _quantise(X: np.ndarray) -> np.ndarray:
    return np.rint(X * 100.0).astype(np.int32)


def make_points(cfg: Config | int, n: int | None = None) -> np.ndarray:
    """Seeded point set of a config (optionally only its first n points).

    Returns int32 coordinates (L1 configs, already x100-quantised) or float64
    coordinates (Euclidean configs)."""
    if isinstance(cfg, int):
        cfg = CONFIGS[cfg]
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    N = cfg.n
    if cfg.cid == 1:
        centres = rng.uniform(0.0, 100.0, size=(5, 2))
        labels = rng.integers(0, 5, size=N)
        X = centres[labels] + 5.0 * rng.standard_normal((N, 2))
    elif cfg.cid == 2:
        centres = 10.0 * rng.standard_normal((20, 10))
        wts = rng.dirichlet(np.ones(20))
        labels = rng.choice(20, size=N, p=wts)
        X = centres[labels] + rng.standard_normal((N, 10))
    elif cfg.cid == 3:
        protos = rng.dirichlet(0.3 * np.ones(27), size=100)
        labels = rng.integers(0, 100, size=N)
        X = np.empty((N, 27))
        for i in range(N):
            X[i] = rng.dirichlet(200.0 * protos[labels[i]] + 1e-3)
        X = np.maximum(0.0, X + 0.002 * rng.standard_normal((N, 27)))
        X = X / X.sum(axis=1, keepdims=True)
    elif cfg.cid == 4:
        centres = 8.0 * rng.standard_normal((200, 32))
        wts = rng.dirichlet(np.ones(200))
        labels = rng.choice(200, size=N, p=wts)
        X = centres[labels] + rng.standard_normal((N, 32))
    elif cfg.cid == 5:
        n_in = 95000
        centres = 6.0 * rng.standard_normal((500, 64))
        wts = rng.dirichlet(np.ones(500))
        labels = rng.choice(500, size=n_in, p=wts)
        Xin = centres[labels] + rng.standard_normal((n_in, 64))
        lo, hi = Xin.min(axis=0), Xin.max(axis=0)
        Xout = rng.uniform(lo, hi, size=(N - n_in, 64))
        X = np.concatenate([Xin, Xout], axis=0)
        X = X[rng.permutation(N)]
    else:
        raise KeyError(cfg.cid)
    if n is not None:
        X = X[:n]
    if cfg.metric == L1_INT:
        return _quantise(X)
    return np.ascontiguousarray(X, dtype=np.float64)


def random_medoids(cfg: Config | int, k: int | None = None, n: int | None = None) -> np.ndarray:
    """k distinct uniform indices (seed + 1000), slot order as drawn."""
    if isinstance(cfg, int):
        cfg = CONFIGS[cfg]
    rng = np.random.Generator(np.random.PCG64(cfg.seed + 1000))
    return rng.choice(n or cfg.n, size=k or cfg.k, replace=False).astype(np.int32)


def round_ld(w: int) -> int:
    """Row stride (elements) for a slab of width w: multiple of 4 (16-byte rows)."""
    return (w + 3) // 4 * 4


def dist_numpy(X: np.ndarray, metric: int, c0: int = 0, c1: int | None = None, ld: int | None = None) -> np.ndarray:
    """Exact CPU materialisation of columns [c0, c1) of D (rows padded to ld).

    Returns an (n, ld) array; the slab is [:, :c1-c0]."""
    n = X.shape[0]
    c1 = n if c1 is None else c1
    w = c1 - c0
    ld = round_ld(w) if ld is None else ld
    out = np.zeros((n, ld), dtype=np.uint32 if metric == L1_INT else np.float32)
    Y = X[c0:c1]
    step = max(1, (1 << 24) // max(1, w * X.shape[1]))
    for a in range(0, n, step):
        Xa = X[a:a + step]
        if metric == L1_INT:
            acc = np.zeros((Xa.shape[0], w), np.int64)
            for t in range(X.shape[1]):
                acc += np.abs(Xa[:, t].astype(np.int64)[:, None] - Y[:, t].astype(np.int64)[None, :])
            out[a:a + step, :w] = acc.astype(np.uint32)
        else:
            acc = np.zeros((Xa.shape[0], w), np.float64)
            for t in range(X.shape[1]):
                diff = Xa[:, t][:, None] - Y[:, t][None, :]
                acc = acc + diff * diff
            out[a:a + step, :w] = np.sqrt(acc).astype(np.float32)
    return out


_CPU_SO = os.path.join(_HERE, "libkmsynth_cpu.so")
_CPU_SRC = os.path.join(_HERE, "csrc", "synth_cpu.c")
_cpu_lib = None


def build_cpu_lib(force: bool = False) -> str:
    """gcc -O2 -fopenmp, no fast-math, no FMA contraction (bit-identical to dist_numpy)."""
    if force or not os.path.exists(_CPU_SO) or os.path.getmtime(_CPU_SO) < os.path.getmtime(_CPU_SRC):
        tmp = _CPU_SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fopenmp", "-ffp-contract=off", "-shared", "-fPIC",
                               "-o", tmp, _CPU_SRC, "-lm"])
        os.replace(tmp, _CPU_SO)
    return _CPU_SO


def dist_cpu(X: np.ndarray, metric: int, c0: int = 0, c1: int | None = None, ld: int | None = None,
             out: np.ndarray | None = None) -> np.ndarray:
    """Multi-threaded CPU materialisation of columns [c0, c1) of D, bit-identical
    to dist_numpy (an (n, ld) array; the slab is [:, :c1-c0])."""
    global _cpu_lib
    if _cpu_lib is None:
        _cpu_lib = ctypes.CDLL(build_cpu_lib())
    n, d = X.shape
    c1 = n if c1 is None else c1
    ld = round_ld(c1 - c0) if ld is None else ld
    dt = np.uint32 if metric == L1_INT else np.float32
    if out is None:
        out = np.zeros((n, ld), dtype=dt)
    assert out.shape == (n, ld) and out.dtype == dt and out.flags.c_contiguous
    if metric == L1_INT:
        Xc = np.ascontiguousarray(X, dtype=np.int32)
        f = _cpu_lib.kmsynth_cpu_dist_l1
    else:
        Xc = np.ascontiguousarray(X, dtype=np.float64)
        f = _cpu_lib.kmsynth_cpu_dist_l2
    f(ctypes.c_void_p(Xc.ctypes.data), ctypes.c_int64(n), ctypes.c_int32(d), ctypes.c_int64(c0),
      ctypes.c_int64(c1), ctypes.c_int64(ld), ctypes.c_void_p(out.ctypes.data))
    return out


def build_lib(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
                               "-Xcompiler", "-fPIC", "-shared", "-o", tmp, _SRC])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def dist_cuda(X: np.ndarray, metric: int, c0: int = 0, c1: int | None = None, ld: int | None = None,
              device="cuda"):
    """GPU materialisation of columns [c0, c1) of D as an (n, ld) torch tensor."""
    global _lib
    import torch
    if _lib is None:
        _lib = ctypes.CDLL(build_lib())
    n, d = X.shape
    c1 = n if c1 is None else c1
    ld = round_ld(c1 - c0) if ld is None else ld
    if metric == L1_INT:
        pts = torch.from_numpy(np.ascontiguousarray(X, dtype=np.int32)).to(device)
        out = torch.zeros((n, ld), dtype=torch.int32, device=device)   # uint32 bits
    else:
        pts = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float64)).to(device)
        out = torch.zeros((n, ld), dtype=torch.float32, device=device)
    stream = torch.cuda.current_stream(out.device).cuda_stream
    rc = _lib.kmsynth_dist(ctypes.c_void_p(pts.data_ptr()), ctypes.c_int(metric), ctypes.c_int(n), ctypes.c_int(d),
                           ctypes.c_int64(c0), ctypes.c_int64(c1), ctypes.c_int64(ld),
                           ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"kmsynth_dist failed with cudaError {rc}")
    return out


def as_numpy_D(t) -> np.ndarray:
    """Host numpy view of a dist_cuda tensor with the right element type."""
    a = t.cpu().numpy()
    return a.view(np.uint32) if a.dtype == np.int32 else a


def read_peak_gbs(t, reps: int = 5, stream=None) -> float:
    """Read-only HBM bandwidth (GB/s, best of reps) over the bytes of the CUDA tensor t
    (measurement helper for bench.py's roofline; not part of the method)."""
    import torch
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_lib())
    f = _lib.kmsynth_read_peak
    f.restype = ctypes.c_double
    f.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
    st = stream if stream is not None else torch.cuda.current_stream(t.device)
    return float(f(ctypes.c_void_p(t.data_ptr()), int(t.numel() * t.element_size()) // 16 * 16, int(reps),
                   ctypes.c_void_p(st.cuda_stream)))


def read_peak_bulk_gbs(t, reps: int = 5, stream=None) -> float:
    """Read-only HBM bandwidth (GB/s) through TMA bulk copies into shared
    memory (measurement helper; the SWAP stream's load path without compute)."""
    import torch
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_lib())
    f = _lib.kmsynth_read_peak_bulk
    f.restype = ctypes.c_double
    f.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
    st = stream if stream is not None else torch.cuda.current_stream(t.device)
    return float(f(ctypes.c_void_p(t.data_ptr()), int(t.numel() * t.element_size()), int(reps),
                   ctypes.c_void_p(st.cuda_stream)))


def write_peak_gbs(t, reps: int = 5, stream=None) -> float:
    """Write-only HBM bandwidth (GB/s, best of reps) over the bytes of the CUDA
    tensor t, whose contents are OVERWRITTEN (measurement helper for bench.py's
    dissimilarity roofline; not part of the method)."""
    import torch
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_lib())
    f = _lib.kmsynth_write_peak
    f.restype = ctypes.c_double
    f.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
    st = stream if stream is not None else torch.cuda.current_stream(t.device)
    return float(f(ctypes.c_void_p(t.data_ptr()), int(t.numel() * t.element_size()) // 16 * 16, int(reps),
                   ctypes.c_void_p(st.cuda_stream)))
