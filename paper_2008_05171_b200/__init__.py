"""B200-native FastPAM SWAP (Schubert & Rousseeuw, arXiv 2008.05171).

The product is ``libkmedoids.so`` (C ABI in ``include/kmedoids.h``, sm_100a
kernels in ``csrc/``).  ``kmedoids`` is its thin ctypes binding and
``parallel`` drives the column-sharded multi-GPU phases over
``torch.distributed``.
"""
from .kmedoids import (KMedoids, KMError, Result, kmedoids_create, kmedoids_destroy, kmedoids_init_build,  # noqa: F401
                       kmedoids_clara_points, kmedoids_dissimilarity, kmedoids_run, kmedoids_run_host, kmedoids_set_medoids, kmedoids_swap_iter,
                       kmedoids_release_host_cache,
                       load_library)
