"""The C-ABI library loads and exports every symbol include/*.h declares
(no compute calls: this runs on the CPU-only box too)."""
import ctypes
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(kmedoids_[a-z_0-9]+)\s*\(", src))
    return sorted(names)


@pytest.fixture(scope="module")
def lib():
    from paper_2008_05171_b200 import kmedoids
    if not os.path.exists(kmedoids.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return kmedoids.load_library()


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for required in ("kmedoids_init_build", "kmedoids_swap_iter", "kmedoids_run", "kmedoids_create",
                     "kmedoids_destroy", "kmedoids_last_error"):
        assert required in names
    assert len(names) >= 20


def test_every_declared_symbol_is_exported(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_argument_validation_without_gpu(lib):
    from paper_2008_05171_b200 import kmedoids as K
    h = ctypes.c_void_p()
    # NULL D, bad k, misaligned ld: rejected before any CUDA call
    assert lib.kmedoids_create(ctypes.byref(h), None, K.KM_U32, 10, 12, 0, 10, 3, None) == K.KM_EINVAL
    assert b"NULL" in lib.kmedoids_last_error()
    fake = ctypes.c_void_p(1 << 20)
    assert lib.kmedoids_create(ctypes.byref(h), fake, K.KM_U32, 10, 12, 0, 10, 10, None) == K.KM_EINVAL
    assert lib.kmedoids_create(ctypes.byref(h), fake, K.KM_U32, 10, 10, 0, 10, 3, None) == K.KM_EINVAL
    assert lib.kmedoids_create(ctypes.byref(h), fake, K.KM_F32, 2, 4, 0, 2, 1, None) == K.KM_EINVAL
    assert lib.kmedoids_create(ctypes.byref(h), fake, K.KM_F32, 10, 12, 5, 3, 2, None) == K.KM_EINVAL
    assert lib.kmedoids_set_medoids(None, None) == K.KM_EINVAL


def test_product_path_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_2008_05171_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace("oracle_", ""), f
