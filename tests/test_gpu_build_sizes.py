"""BUILD (Alg.1) on CLARA-sized and degenerate problems against the
oracle's Alg.1: bit-exact on uint32 (ties from small value ranges,
asymmetric matrices, k = n - 1, k = 1), on every call of a handle (direct
launch, graph capture, graph replay), and the cache BUILD leaves behind
equals the from-scratch assignment (reading R2); float within R9."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from test_gpu_parity import KM, rand_int, to_dev  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("n,k,hi,sym", [(9, 3, 4, True), (100, 7, 4, False), (777, 40, 1000, True),
                                         (2000, 64, 3, True), (4096, 30, 1000, False), (50, 49, 5, True),
                                         (300, 1, 1000, True)])
def test_build_int_bit_exact_sizes(n, k, hi, sym):
    rng = np.random.default_rng(n * 31 + k)
    D = rand_int(rng, n, hi, symmetric=sym)
    Mb, tdb, _ = oracle.build_init(D, k)
    km = KM(to_dev(D), n, k)
    for _ in range(3):                       # direct launch, graph capture, graph replay
        Mg, tdg = km.init_build()
        assert Mg.tolist() == Mb.tolist()
        assert tdg == (oracle.td(D, Mb) if k >= 2 else tdb)
    if k >= 2:
        near, sec = km.get_cache()[:2]
        ref = oracle.assign(D, Mb)
        assert near.tolist() == np.asarray(ref.nearest).tolist() and sec.tolist() == np.asarray(ref.second).tolist()


def test_build_float_clara_sized():
    rng = np.random.default_rng(77)
    n, k, d = 1500, 40, 8
    X = (6 * rng.standard_normal((12, d)))[rng.integers(0, 12, size=n)] + rng.standard_normal((n, d))
    D = oracle.dist_l2(X.astype(np.float32)).astype(np.float32)
    km = KM(to_dev(D), n, k)
    Ms, tds = km.init_build()
    Mb, tdb, _ = oracle.build_init(D, k)
    assert Ms.tolist() == Mb.tolist()
    assert tds == pytest.approx(oracle.td(D, Mb), rel=1e-12)
