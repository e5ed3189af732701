"""FastPAM2 iterations queued one ahead (kmedoids_swap_iters_variant /
kmedoids_run; the sticky Decision::done of a pass without an improving slot)
against one kmedoids_swap_iter(KM_FASTPAM2) per call: the same swaps, the same
iteration and swap counts (the converging pass counted once),
the same state; int path also against the oracle's reading R6."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import kmsynth  # noqa: E402
import oracle  # noqa: E402
from test_gpu_parity import KM  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def per_call(Dt, n, k, M0):
    km = KM(Dt, n, k)
    km.set_medoids(M0)
    it = sw = 0
    while True:
        conv, s, td = km.swap_iter("fastpam2")
        it += 1
        sw += s
        if conv:
            break
    st = km.get_state()
    km.close()
    return st, it, sw


@pytest.mark.parametrize("cid,n,k,chunks", [(5, 1500, 12, (3, 2000)), (1, 500, 5, (1, 1, 2000)),
                                           (3, 2500, 30, (2000,)), (4, 3000, 40, (4, 4, 2000))])
def test_fastpam2_queued_equals_per_call(cid, n, k, chunks):
    cfg = kmsynth.CONFIGS[cid]
    X = kmsynth.make_points(cfg, n=n)
    Dt = kmsynth.dist_cuda(X, cfg.metric)
    M0 = kmsynth.random_medoids(cfg, k=k, n=n)
    st1, it1, sw1 = per_call(Dt, n, k, M0)
    km = KM(Dt, n, k)
    km.set_medoids(M0)
    it = sw = 0
    conv = False
    for c in chunks:                               # queued in chunks: the state carries over
        conv, i2, s2, td2 = km.swap_iters(c, "fastpam2")
        it += i2
        sw += s2
        if conv:
            break
    assert conv and it == it1 and sw == sw1
    st = km.get_state()
    assert st.medoids.tolist() == st1.medoids.tolist()
    assert st.assignment.tolist() == st1.assignment.tolist()
    assert st.td == st1.td and st.n_iter == st1.n_iter == it1 and st.n_swaps == st1.n_swaps == sw1
    # a further queued call: one more (non-improving) pass counted, nothing changes
    conv, i3, s3, _ = km.swap_iters(3, "fastpam2")
    assert conv and i3 == 1 and s3 == 0
    assert km.get_state().medoids.tolist() == st1.medoids.tolist()
    # kmedoids_run takes the queued path too
    km2 = KM(Dt, n, k)
    km2.set_medoids(M0)
    r = km2.run(use_build=False, variant="fastpam2")
    assert r.converged and r.medoids.tolist() == st1.medoids.tolist() and r.td == st1.td
    assert (r.n_iter, r.n_swaps) == (it1, sw1)
    if cfg.metric == kmsynth.L1_INT:
        D = kmsynth.as_numpy_D(Dt)[:, :n]
        ref = oracle.swap_run(D, M0, oracle.FASTPAM2)
        assert r.medoids.tolist() == ref.medoids.tolist() and r.td == ref.td
        assert (r.n_iter, r.n_swaps) == (ref.n_iter, ref.n_swaps)
    # FastPAM1 after a converged FastPAM2 run on the same handle still works
    km.set_medoids(M0)
    r1 = km.run(use_build=False, variant="fastpam1")
    assert r1.converged and r1.n_iter >= 1
