"""The seeded input generators agree with each other (CPU, no GPU needed):
kmsynth.dist_cpu (OpenMP C, used by scripts/make_goldens.py for the
full-size oracle inputs) is bit-identical to kmsynth.dist_numpy on every
config's recipe, on full squares and on ragged column slabs.  (The CUDA
materialiser is checked against dist_numpy in
tests/test_gpu_parity.py::test_synth_cuda_matches_numpy.)"""
import numpy as np
import pytest

import kmsynth


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("c0,c1", [(0, None), (5, 123), (96, 97)])
def test_dist_cpu_matches_numpy(cid, c0, c1):
    cfg = kmsynth.CONFIGS[cid]
    X = kmsynth.make_points(cfg, n=300 if cid == 3 else 400)
    a = kmsynth.dist_numpy(X, cfg.metric, c0, c1)
    b = kmsynth.dist_cpu(X, cfg.metric, c0, c1)
    assert a.dtype == b.dtype and a.shape == b.shape
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_generated_D_is_a_dissimilarity():
    """Zero diagonal, exact symmetry, non-negative (the library's input contract)."""
    for cid in (1, 2):
        cfg = kmsynth.CONFIGS[cid]
        X = kmsynth.make_points(cfg, n=256)
        D = kmsynth.dist_cpu(X, cfg.metric)
        assert (np.diag(D) == 0).all() and np.array_equal(D, D.T) and (D >= 0).all()
