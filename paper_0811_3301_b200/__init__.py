"""B200-native two-pass DTW k-NN search (Lemire, arXiv:0811.3301).

The method -- query envelope, [piecewise-sum pre-filter,] LB_Keogh over the database, LB_Improved on the
survivors, banded DTW on what remains -- runs in hand-written sm_100a CUDA
kernels behind the C ABI of ``include/dtwlb.h`` (``libdtwlb.so``).  This package
is the thin Python binding (``binding``) plus the database-sharded multi-GPU
driver (``sharded``).  Importing it does not require a GPU; calling it does.
"""
from .binding import (Communicator, DtwlbError, KEOGH_ONLY, MAX_K, NO_PREFILTER, dtw_band, get_unique_id,
                      lb_envelope, lb_improved, lb_keogh, lb_piecewise, lb_piecewise_sym, load, nn_merge, nn_search,
                      release_workspace)

__all__ = ["Communicator", "DtwlbError", "KEOGH_ONLY", "MAX_K", "NO_PREFILTER", "dtw_band", "get_unique_id",
           "lb_envelope", "lb_improved", "lb_keogh", "lb_piecewise", "lb_piecewise_sym", "load", "nn_merge",
           "nn_search", "release_workspace"]
