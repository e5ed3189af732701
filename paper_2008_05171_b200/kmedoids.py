"""Thin Python binding of libkmedoids.so (include/kmedoids.h).

Argument marshalling only: every step of BUILD / SWAP runs in the library's
sm_100a kernels.  There is no CPU fallback -- importing this module on a
machine without the built library raises, and every call checks the status
code the C ABI returns.

Function names follow the C ABI (``kmedoids_create``, ``kmedoids_init_build``,
``kmedoids_swap_iter``, ``kmedoids_run``, ...).  ``KMedoids`` wraps a handle
for convenience.  Device buffers are torch CUDA tensors (PyTorch supplies
device memory and streams only).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# KM_LIBRARY=checked selects the build with device-side index asserts
# (libkmedoids_checked.so, test runs); the default is the product build
LIB_PATH = os.path.join(_HERE, "libkmedoids_checked.so" if os.environ.get("KM_LIBRARY") == "checked"
                        else "libkmedoids.so")

KM_OK, KM_CONVERGED, KM_NOT_CONVERGED = 0, 1, 2
KM_EINVAL, KM_ENOMEM, KM_ECUDA, KM_ECOMM = 10, 11, 12, 13
KM_U32, KM_F32 = 0, 1
KM_FASTPAM1, KM_FASTPAM2, KM_FASTERPAM, KM_FASTPAM1_INC = 0, 1, 2, 3
VARIANTS = {"fastpam1": KM_FASTPAM1, "fastpam2": KM_FASTPAM2, "fasterpam": KM_FASTERPAM,
            "fastpam1_inc": KM_FASTPAM1_INC}


class KMError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"kmedoids status {status}: {msg}")
        self.status = status


class _Exchange(ctypes.Structure):
    _fields_ = [("record_send", ctypes.c_void_p), ("record_recv", ctypes.c_void_p),
                ("record_bytes", ctypes.c_size_t), ("column", ctypes.c_void_p),
                ("column_bytes", ctypes.c_size_t)]


class _Fp2Exchange(ctypes.Structure):
    _fields_ = [("record_send", ctypes.c_void_p), ("record_recv", ctypes.c_void_p),
                ("record_bytes", ctypes.c_size_t), ("col_send", ctypes.c_void_p),
                ("col_recv", ctypes.c_void_p), ("col_bytes_per_column", ctypes.c_size_t),
                ("col_capacity", ctypes.c_int32)]


_lib = None


def load_library() -> ctypes.CDLL:
    """Load libkmedoids.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    sig = {
        "kmedoids_create": [ctypes.POINTER(vp), vp, ctypes.c_int, i64, i64, i64, i64, i32, vp],
        "kmedoids_destroy": [vp],
        "kmedoids_set_medoids": [vp, vp],
        "kmedoids_init_build": [vp, vp, vp],
        "kmedoids_swap_iter": [vp, ctypes.c_int, vp, vp],
        "kmedoids_swap_iters": [vp, i32, vp, vp, vp],
        "kmedoids_swap_iters_variant": [vp, ctypes.c_int, i32, vp, vp, vp],
        "kmedoids_run": [vp, i32, ctypes.c_int, i32, vp, vp, vp, vp, vp],
        "kmedoids_run_host": [vp, ctypes.c_int, i64, i64, i32, i32, vp, ctypes.c_int, i32, vp, vp, vp, vp, vp, vp],
        "kmedoids_get_state": [vp, vp, vp, vp, vp, vp],
        "kmedoids_release_host_cache": [],
        "kmedoids_get_cache": [vp, vp, vp, vp, vp],
        "kmedoids_eval_candidates": [vp, vp, vp],
        "kmedoids_set_profiling": [vp, i32],
        "kmedoids_set_symmetric": [vp, i32],
        "kmedoids_last_swaps": [vp, vp, vp, vp, i32, vp],
        "kmedoids_fp2_last_plan": [vp, vp, vp, vp, vp],
        "kmedoids_stream_time": [vp, vp, vp, i32],
        "kmedoids_launch_count": [vp, vp],
        "kmedoids_stream_kernel": [vp, ctypes.POINTER(ctypes.c_char_p)],
        "kmedoids_shard_exchange": [vp, i32, ctypes.POINTER(_Exchange)],
        "kmedoids_shard_set_medoids": [vp, vp, vp],
        "kmedoids_shard_eval": [vp],
        "kmedoids_shard_select": [vp, vp, vp, vp, vp, vp, vp],
        "kmedoids_shard_pack_column": [vp, i32],
        "kmedoids_shard_apply": [vp],
        "kmedoids_shard_decide": [vp],
        "kmedoids_build_decide": [vp, i32],
        "kmedoids_build_apply_async": [vp, i32],
        "kmedoids_shard_apply_async": [vp],
        "kmedoids_shard_status": [vp, i32, vp, vp, vp, vp],
        "kmedoids_shard_resync": [vp, vp],
        "kmedoids_shard_trace": [vp, vp, vp, vp, i32, vp],
        "kmedoids_fp2_shard_exchange": [vp, i32, ctypes.POINTER(_Fp2Exchange)],
        "kmedoids_fp2_shard_eval": [vp],
        "kmedoids_fp2_shard_plan": [vp, vp, vp, vp],
        "kmedoids_fp2_shard_apply": [vp, vp, vp],
        "kmedoids_fp2_round_buffers": [vp, vp, vp, vp],
        "kmedoids_fp2_round_eval": [vp],
        "kmedoids_fp2_round_apply": [vp, vp, vp, vp],
        "kmedoids_build_eval": [vp, i32],
        "kmedoids_build_select": [vp, vp, vp, vp, vp],
        "kmedoids_build_apply": [vp, i32],
        "kmedoids_dissimilarity": [vp, ctypes.c_int, i64, i32, vp, i64, i64, i64, vp],
        "kmedoids_init_weighted": [vp, vp, vp, vp],
        "kmedoids_init_lab": [vp, i32, vp, vp, vp],
        "kmedoids_clara": [vp, i32, i32, vp, ctypes.c_int, vp, vp, vp],
        "kmedoids_clara_points": [vp, ctypes.c_int, i64, i32, i32, i32, i32, vp, ctypes.c_int, vp, vp, vp, vp, vp],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.kmedoids_last_error.restype = ctypes.c_char_p
    lib.kmedoids_last_error.argtypes = []
    _lib = lib
    return lib


def _check(status: int, ok=(KM_OK,)) -> int:
    if status not in ok:
        raise KMError(status, load_library().kmedoids_last_error().decode())
    return status


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _dtype_code(t) -> int:
    import torch
    if t.dtype in (torch.int32, getattr(torch, "uint32", torch.int32)):
        return KM_U32
    if t.dtype == torch.float32:
        return KM_F32
    raise TypeError(f"D must be int32/uint32 (u32 bits) or float32, got {t.dtype}")


@dataclass
class Result:
    medoids: np.ndarray
    assignment: np.ndarray
    td: int | float
    n_iter: int
    n_swaps: int
    converged: bool


class KMedoids:
    """A handle over a borrowed device slab D (see include/kmedoids.h)."""

    def __init__(self, D, n: int, k: int, col_begin: int = 0, col_end: int | None = None, stream=None):
        import torch
        lib = load_library()
        if not D.is_cuda:
            raise ValueError("D must be a CUDA tensor (use kmedoids_run_host for host data)")
        if D.dim() != 2 or D.stride(1) != 1:
            raise ValueError("D must be a 2-D row-major tensor")
        self.D = D                       # keep the borrowed slab alive
        self.n, self.k = int(n), int(k)
        self.col_begin = int(col_begin)
        self.col_end = int(n if col_end is None else col_end)
        self.dtype = _dtype_code(D)
        if D.shape[0] < self.n or D.shape[1] < self.col_end - self.col_begin:
            raise ValueError(f"D of shape {tuple(D.shape)} cannot hold {self.n} rows x "
                             f"{self.col_end - self.col_begin} columns")
        self.acc = np.int64 if self.dtype == KM_U32 else np.float64
        self.stream = stream if stream is not None else torch.cuda.current_stream(D.device)
        h = ctypes.c_void_p()
        _check(lib.kmedoids_create(ctypes.byref(h), ctypes.c_void_p(D.data_ptr()), self.dtype, self.n,
                                   int(D.stride(0)), self.col_begin, self.col_end, self.k,
                                   ctypes.c_void_p(self.stream.cuda_stream)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            load_library().kmedoids_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- single-GPU API -------------------------------------------------------
    def set_medoids(self, medoids):
        M = np.ascontiguousarray(np.asarray(medoids, dtype=np.int32))
        if M.shape != (self.k,):
            raise ValueError(f"expected {self.k} medoids")
        _check(load_library().kmedoids_set_medoids(self.h, _p(M)))

    def set_symmetric(self, on=True):
        """Declare D exactly symmetric (verified on the device; kmedoids.h)."""
        _check(load_library().kmedoids_set_symmetric(self.h, int(on)))

    def init_build(self):
        M = np.zeros(self.k, np.int32)
        td = np.zeros(1, self.acc)
        _check(load_library().kmedoids_init_build(self.h, _p(M), _p(td)))
        return M, td[0].item()

    def init_weighted(self, u):
        """Distance-weighted seeding with the caller's uniforms u[k] (NEXT-4)."""
        uu = np.ascontiguousarray(np.asarray(u, np.float64))
        if uu.shape != (self.k,):
            raise ValueError(f"expected {self.k} uniforms")
        M = np.zeros(self.k, np.int32)
        td = np.zeros(1, self.acc)
        _check(load_library().kmedoids_init_weighted(self.h, _p(uu), _p(M), _p(td)))
        return M, td[0].item()

    def init_lab(self, s: int, seq):
        """LAB with the caller's per-step index rows seq[k][s+k] (NEXT-4)."""
        q = np.ascontiguousarray(np.asarray(seq, np.int32))
        if q.shape != (self.k, s + self.k):
            raise ValueError(f"expected seq of shape ({self.k}, {s + self.k})")
        M = np.zeros(self.k, np.int32)
        td = np.zeros(1, self.acc)
        _check(load_library().kmedoids_init_lab(self.h, int(s), _p(q), _p(M), _p(td)))
        return M, td[0].item()

    def clara(self, samples, variant="fastpam1"):
        """FastCLARA over the caller's samples[nsamples][s] (NEXT-3): (medoids, TD, best sample)."""
        q = np.ascontiguousarray(np.asarray(samples, np.int32))
        if q.ndim != 2:
            raise ValueError("samples must be (nsamples, s)")
        M = np.zeros(self.k, np.int32)
        td = np.zeros(1, self.acc)
        b = np.zeros(1, np.int32)
        _check(load_library().kmedoids_clara(self.h, q.shape[0], q.shape[1], _p(q), VARIANTS[variant], _p(M), _p(td),
                                             _p(b)))
        return M, td[0].item(), int(b[0])

    def swap_iter(self, variant="fastpam1"):
        if getattr(self, "_it_bufs", None) is None:        # reused: keeps the per-call host work small
            sw = np.zeros(1, np.int32)
            td = np.zeros(1, self.acc)
            self._it_bufs = (sw, td, _p(sw), _p(td))
        sw, td, psw, ptd = self._it_bufs
        s = _check(load_library().kmedoids_swap_iter(self.h, VARIANTS[variant], psw, ptd), ok=(KM_OK, KM_CONVERGED))
        return s == KM_CONVERGED, int(sw[0]), td[0].item()

    def swap_iters(self, count: int, variant: str = "fastpam1"):
        """Up to `count` FastPAM1 or FastPAM2 iterations queued back to back (no
        host round trip between them); returns (converged, iterations, swaps, td)."""
        it = np.zeros(1, np.int32); sw = np.zeros(1, np.int32); td = np.zeros(1, self.acc)
        if variant == "fastpam1":
            s = _check(load_library().kmedoids_swap_iters(self.h, int(count), _p(it), _p(sw), _p(td)),
                       ok=(KM_OK, KM_CONVERGED))
        else:
            s = _check(load_library().kmedoids_swap_iters_variant(self.h, VARIANTS[variant], int(count), _p(it),
                                                                  _p(sw), _p(td)), ok=(KM_OK, KM_CONVERGED))
        return s == KM_CONVERGED, int(it[0]), int(sw[0]), td[0].item()

    def run(self, use_build=True, variant="fastpam1", max_iter=2000) -> Result:
        M = np.zeros(self.k, np.int32)
        asg = np.zeros(self.n, np.int32)
        td = np.zeros(1, self.acc)
        it = np.zeros(1, np.int32)
        sw = np.zeros(1, np.int32)
        s = _check(load_library().kmedoids_run(self.h, int(use_build), VARIANTS[variant], int(max_iter), _p(M),
                                               _p(asg), _p(td), _p(it), _p(sw)), ok=(KM_OK, KM_NOT_CONVERGED))
        return Result(M, asg, td[0].item(), int(it[0]), int(sw[0]), s == KM_OK)

    def get_state(self) -> Result:
        M = np.zeros(self.k, np.int32)
        asg = np.zeros(self.n, np.int32)
        td = np.zeros(1, self.acc)
        it = np.zeros(1, np.int32)
        sw = np.zeros(1, np.int32)
        _check(load_library().kmedoids_get_state(self.h, _p(M), _p(asg), _p(td), _p(it), _p(sw)))
        return Result(M, asg, td[0].item(), int(it[0]), int(sw[0]), True)

    def get_cache(self):
        dt = np.uint32 if self.dtype == KM_U32 else np.float32
        near = np.zeros(self.n, np.int32); sec = np.zeros(self.n, np.int32)
        dn = np.zeros(self.n, dt); ds = np.zeros(self.n, dt)
        _check(load_library().kmedoids_get_cache(self.h, _p(near), _p(sec), _p(dn), _p(ds)))
        return near, sec, dn, ds

    def eval_candidates(self):
        w = self.col_end - self.col_begin
        v = np.zeros(w, self.acc); s = np.zeros(w, np.int32)
        _check(load_library().kmedoids_eval_candidates(self.h, _p(v), _p(s)))
        return v, s

    def last_swaps(self):
        """[(slot, candidate, dTD)] applied by the last swap_iter call."""
        cnt = np.zeros(1, np.int32)
        _check(load_library().kmedoids_last_swaps(self.h, None, None, None, 0, _p(cnt)))
        m = int(cnt[0])
        sl = np.zeros(max(m, 1), np.int32); cd = np.zeros(max(m, 1), np.int32); dv = np.zeros(max(m, 1), self.acc)
        _check(load_library().kmedoids_last_swaps(self.h, _p(sl), _p(cd), _p(dv), m, _p(cnt)))
        return [(int(sl[j]), int(cd[j]), dv[j].item()) for j in range(m)]

    def fp2_last_plan(self):
        """Per-slot best (v[k], c[k]) and the improving slots in plan order of
        the last FastPAM2 iteration (reading R6 steps 2-5)."""
        v = np.zeros(self.k, self.acc); c = np.zeros(self.k, np.int32)
        order = np.zeros(self.k, np.int32); m = np.zeros(1, np.int32)
        _check(load_library().kmedoids_fp2_last_plan(self.h, _p(v), _p(c), _p(order), _p(m)))
        return v, c, order[:int(m[0])].copy()

    def set_profiling(self, on=True):
        _check(load_library().kmedoids_set_profiling(self.h, int(on)))

    def stream_time(self, reset=False):
        ms = ctypes.c_double(); cnt = ctypes.c_int64()
        _check(load_library().kmedoids_stream_time(self.h, ctypes.byref(ms), ctypes.byref(cnt), int(reset)))
        return ms.value, cnt.value

    def launch_count(self) -> int:
        c = ctypes.c_int64()
        _check(load_library().kmedoids_launch_count(self.h, ctypes.byref(c)))
        return c.value

    def stream_kernel(self) -> str:
        """Name of the SWAP-delta stream kernel this handle launches."""
        name = ctypes.c_char_p()
        _check(load_library().kmedoids_stream_kernel(self.h, ctypes.byref(name)))
        return name.value.decode()

    # ---- sharded phase API ------------------------------------------------------
    def shard_exchange(self, nranks: int) -> _Exchange:
        x = _Exchange()
        _check(load_library().kmedoids_shard_exchange(self.h, int(nranks), ctypes.byref(x)))
        return x

    def shard_set_medoids(self, medoids, columns):
        M = np.ascontiguousarray(np.asarray(medoids, dtype=np.int32))
        if M.shape != (self.k,):
            raise ValueError(f"expected {self.k} medoids")
        if (not columns.is_cuda or columns.device != self.D.device or not columns.is_contiguous()
                or columns.numel() * columns.element_size() < 4 * self.k * self.n):
            raise ValueError(f"columns must be a contiguous CUDA tensor on {self.D.device} holding "
                             f"k*n = {self.k * self.n} 4-byte dissimilarities")
        _check(load_library().kmedoids_shard_set_medoids(self.h, _p(M), ctypes.c_void_p(columns.data_ptr())))

    def shard_eval(self):
        _check(load_library().kmedoids_shard_eval(self.h))

    def shard_select(self, rank_col_begin):
        rcb = np.ascontiguousarray(np.asarray(rank_col_begin, dtype=np.int64))
        f = np.zeros(1, np.int32); sl = np.zeros(1, np.int32); c = np.zeros(1, np.int32)
        ow = np.zeros(1, np.int32); d = np.zeros(1, self.acc)
        _check(load_library().kmedoids_shard_select(self.h, _p(rcb), _p(f), _p(sl), _p(c), _p(ow), _p(d)),
               ok=(KM_OK, KM_CONVERGED))
        return bool(f[0]), int(sl[0]), int(c[0]), int(ow[0]), d[0].item()

    def shard_pack_column(self, cand: int):
        _check(load_library().kmedoids_shard_pack_column(self.h, int(cand)))

    def shard_apply(self):
        _check(load_library().kmedoids_shard_apply(self.h))

    # device-decided iteration (kmedoids.h: no host round trip inside an iteration)
    def shard_decide(self):
        _check(load_library().kmedoids_shard_decide(self.h))

    def build_decide(self, step: int):
        _check(load_library().kmedoids_build_decide(self.h, int(step)))

    def build_apply_async(self, step: int):
        _check(load_library().kmedoids_build_apply_async(self.h, int(step)))

    def shard_apply_async(self):
        _check(load_library().kmedoids_shard_apply_async(self.h))

    def shard_status(self, wait: int = 1):
        """(converged, n_iter, n_swaps, td) of the sharded run; wait: 0 as is,
        1 after all enqueued work, 2 after the iteration before the last one."""
        cv = np.zeros(1, np.int32); it = np.zeros(1, np.int32); sw = np.zeros(1, np.int32)
        td = np.zeros(1, self.acc)
        _check(load_library().kmedoids_shard_status(self.h, int(wait), _p(cv), _p(it), _p(sw), _p(td)))
        return bool(cv[0]), int(it[0]), int(sw[0]), td[0].item()

    def shard_resync(self) -> int:
        """Host bookkeeping after CUDA-graph replays of the sharded iteration
        (kmedoids_shard_resync); returns the decide steps since the reset."""
        c = np.zeros(1, np.int32)
        _check(load_library().kmedoids_shard_resync(self.h, _p(c)))
        return int(c[0])

    def shard_trace(self, cap: int = 4096):
        """Applied swaps of the sharded run: [(slot, cand, dTD)]."""
        sl = np.zeros(cap, np.int32); c = np.zeros(cap, np.int32); d = np.zeros(cap, self.acc)
        cnt = np.zeros(1, np.int32)
        _check(load_library().kmedoids_shard_trace(self.h, _p(sl), _p(c), _p(d), int(cap), _p(cnt)))
        m = min(int(cnt[0]), cap)
        return [(int(sl[i]), int(c[i]), d[i].item()) for i in range(m)]

    def fp2_shard_exchange(self, nranks: int) -> _Fp2Exchange:
        x = _Fp2Exchange()
        _check(load_library().kmedoids_fp2_shard_exchange(self.h, int(nranks), ctypes.byref(x)))
        return x

    def fp2_shard_eval(self):
        _check(load_library().kmedoids_fp2_shard_eval(self.h))

    def fp2_shard_plan(self, rank_col_begin):
        rcb = np.ascontiguousarray(np.asarray(rank_col_begin, dtype=np.int64))
        m = np.zeros(1, np.int32); mx = np.zeros(1, np.int32)
        _check(load_library().kmedoids_fp2_shard_plan(self.h, _p(rcb), _p(m), _p(mx)))
        return int(m[0]), int(mx[0])

    def fp2_shard_apply(self):
        sw = np.zeros(1, np.int32); td = np.zeros(1, self.acc)
        s = _check(load_library().kmedoids_fp2_shard_apply(self.h, _p(sw), _p(td)), ok=(KM_OK, KM_CONVERGED))
        return s == KM_CONVERGED, int(sw[0]), td[0].item()

    def fp2_round_buffers(self):
        """(send pointer, recv pointer, stride bytes) of the owner-side round buffers."""
        sp, rp, st = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_size_t()
        _check(load_library().kmedoids_fp2_round_buffers(self.h, ctypes.byref(sp), ctypes.byref(rp), ctypes.byref(st)))
        return int(sp.value), int(rp.value), int(st.value)

    def fp2_round_eval(self):
        _check(load_library().kmedoids_fp2_round_eval(self.h))

    def fp2_round_apply(self):
        """-> (more rounds, swaps of the iteration, TD) (the last two once more is False)."""
        mo = np.zeros(1, np.int32); sw = np.zeros(1, np.int32); td = np.zeros(1, self.acc)
        _check(load_library().kmedoids_fp2_round_apply(self.h, _p(mo), _p(sw), _p(td)))
        return bool(mo[0]), int(sw[0]), td[0].item()

    def build_eval(self, step: int):
        _check(load_library().kmedoids_build_eval(self.h, int(step)))

    def build_select(self, rank_col_begin):
        rcb = np.ascontiguousarray(np.asarray(rank_col_begin, dtype=np.int64))
        c = np.zeros(1, np.int32); ow = np.zeros(1, np.int32); g = np.zeros(1, self.acc)
        _check(load_library().kmedoids_build_select(self.h, _p(rcb), _p(c), _p(ow), _p(g)))
        return int(c[0]), int(ow[0]), g[0].item()

    def build_apply(self, step: int):
        _check(load_library().kmedoids_build_apply(self.h, int(step)))


# ---- C-ABI-named module functions ----------------------------------------------
def kmedoids_create(D, n, k, col_begin=0, col_end=None, stream=None) -> KMedoids:
    return KMedoids(D, n, k, col_begin, col_end, stream)


def kmedoids_destroy(h: KMedoids):
    h.close()


def kmedoids_set_medoids(h: KMedoids, medoids):
    h.set_medoids(medoids)


def kmedoids_init_build(h: KMedoids):
    return h.init_build()


def kmedoids_swap_iter(h: KMedoids, variant="fastpam1"):
    return h.swap_iter(variant)


def kmedoids_run(h: KMedoids, use_build=True, variant="fastpam1", max_iter=2000) -> Result:
    return h.run(use_build, variant, max_iter)


def kmedoids_run_host(D_host: np.ndarray, k: int, use_build=True, medoids=None, variant="fastpam1",
                      max_iter=2000, stream=None) -> Result:
    """Whole job from host memory (H2D of D, BUILD/SWAP, D2H of the result).

    D_host: (n, ld) uint32 or float32 numpy array (pin it for full PCIe speed,
    e.g. with ``pinned_empty``)."""
    import torch
    lib = load_library()
    if D_host.dtype == np.uint32 or D_host.dtype == np.int32:
        dt, acc = KM_U32, np.int64
    elif D_host.dtype == np.float32:
        dt, acc = KM_F32, np.float64
    else:
        raise TypeError(D_host.dtype)
    if not D_host.flags.c_contiguous:
        raise ValueError("D_host must be C-contiguous (n, ld)")
    n, ld = D_host.shape
    M = np.zeros(k, np.int32)
    asg = np.zeros(n, np.int32)
    td = np.zeros(1, acc)
    it = np.zeros(1, np.int32)
    sw = np.zeros(1, np.int32)
    init = np.ascontiguousarray(np.asarray(medoids, np.int32)) if medoids is not None else None
    st = stream if stream is not None else torch.cuda.current_stream()
    s = _check(lib.kmedoids_run_host(_p(D_host), dt, n, ld, int(k), int(use_build),
                                     _p(init) if init is not None else None, VARIANTS[variant], int(max_iter),
                                     ctypes.c_void_p(st.cuda_stream), _p(M), _p(asg), _p(td), _p(it), _p(sw)),
               ok=(KM_OK, KM_NOT_CONVERGED))
    return Result(M, asg, td[0].item(), int(it[0]), int(sw[0]), s == KM_OK)


def kmedoids_release_host_cache():
    """Free the device copy of D that kmedoids_run_host keeps between calls."""
    _check(load_library().kmedoids_release_host_cache())


def pinned_empty(shape, dtype):
    """Page-locked host numpy array (via torch's pinned allocator)."""
    import torch
    tdt = {np.dtype(np.uint32): torch.int32, np.dtype(np.int32): torch.int32,
           np.dtype(np.float32): torch.float32}[np.dtype(dtype)]
    t = torch.empty(shape, dtype=tdt, pin_memory=True)
    a = t.numpy()
    a = a.view(np.uint32) if np.dtype(dtype) == np.uint32 else a
    return a, t


KM_METRIC_L2_F32, KM_METRIC_L1_U32, KM_METRIC_L2_F32_EXACT = 0, 1, 2


def kmedoids_dissimilarity(X, metric="l2", D=None, col_begin=0, col_end=None, stream=None):
    """Materialise the column slab [col_begin, col_end) of the dissimilarity
    matrix of the points X (torch CUDA tensor, n x d) into D (n x ld; allocated
    if None): "l2" float32 X -> float32 Euclidean on the tensor cores,
    "l2exact" the same with the cancelling (within-cluster) pairs recomputed
    from the points (KM_METRIC_L2_F32_EXACT), "l1" int32 X -> uint32 (int32
    storage) Manhattan.  Returns D."""
    import torch
    lib = load_library()
    if not X.is_cuda or X.dim() != 2:
        raise ValueError("X must be a 2-D CUDA tensor")
    X = X.contiguous()
    n, d = X.shape
    col_end = n if col_end is None else int(col_end)
    code = {"l2": KM_METRIC_L2_F32, "l1": KM_METRIC_L1_U32, "l2exact": KM_METRIC_L2_F32_EXACT}[metric]
    want = torch.int32 if code == KM_METRIC_L1_U32 else torch.float32
    if X.dtype != want:
        raise TypeError(f"metric {metric} needs X of dtype {want}")
    w = col_end - col_begin
    if D is None:
        D = torch.empty((n, (w + 3) // 4 * 4), dtype=want, device=X.device)
    elif (D.dtype != want or not D.is_cuda or D.device != X.device or D.dim() != 2 or D.stride(1) != 1
          or D.shape[0] < n or D.shape[1] < w):
        raise ValueError(f"D must be a row-major {want} CUDA tensor on {X.device} of at least ({n}, {w}); "
                         f"got {D.dtype} {tuple(D.shape)} strides {D.stride()} on {D.device}")
    st = stream if stream is not None else torch.cuda.current_stream(X.device)
    _check(lib.kmedoids_dissimilarity(ctypes.c_void_p(X.data_ptr()), code, n, d, ctypes.c_void_p(D.data_ptr()),
                                      int(D.stride(0)), int(col_begin), int(col_end), ctypes.c_void_p(st.cuda_stream)))
    return D


def kmedoids_clara_points(X, metric, k: int, samples, variant="fastpam1", stream=None, assignment=False):
    """FastCLARA from points without the n x n matrix (kmedoids.h): X is a
    (n, d) CUDA tensor (float32 for "l2", int32 for "l1"), samples an
    (nsamples, s) array of distinct point indices.  Returns (medoids, TD,
    best sample index, assignment or None)."""
    import torch
    lib = load_library()
    if not X.is_cuda or X.dim() != 2:
        raise ValueError("X must be a 2-D CUDA tensor")
    code = {"l2": KM_METRIC_L2_F32, "l1": KM_METRIC_L1_U32}[metric]
    want = torch.float32 if code == KM_METRIC_L2_F32 else torch.int32
    if X.dtype != want:
        raise TypeError(f"metric {metric} needs X of dtype {want}")
    X = X.contiguous()
    n, d = X.shape
    q = np.ascontiguousarray(np.asarray(samples, np.int32))
    if q.ndim != 2:
        raise ValueError("samples must be (nsamples, s)")
    M = np.zeros(k, np.int32)
    td = np.zeros(1, np.float64 if code == KM_METRIC_L2_F32 else np.int64)
    b = np.zeros(1, np.int32)
    asg = np.zeros(n, np.int32) if assignment else None
    st = stream if stream is not None else torch.cuda.current_stream(X.device)
    _check(lib.kmedoids_clara_points(ctypes.c_void_p(X.data_ptr()), code, n, d, int(k), q.shape[0], q.shape[1],
                                     _p(q), VARIANTS[variant], ctypes.c_void_p(st.cuda_stream), _p(M), _p(td),
                                     _p(b), _p(asg) if asg is not None else None))
    return M, td[0].item(), int(b[0]), asg
