"""fp64 CPU oracle for the two-pass DTW k-NN method (arXiv:0811.3301).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_0811_3301_b200`` never imports it, and
the two share no code (the seeded input generators in ``datagen.py`` are the
only common module, and they hold none of the method's arithmetic).

The arithmetic lives in ``dtwlb_oracle.c`` (plain C, fp64), compiled with gcc
into ``oracle/_build/liboracle.so``; this module only marshals numpy arrays.
Each wrapper names the paper passage its C function follows (``P:n`` = line n
of the paper's LaTeX source).  ``p == 0`` means p = infinity.

Parity pins: tests/test_oracle_pins.py, tests/test_oracle_search.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dtwlb_oracle.c")
_LIB = os.path.join(_HERE, "_build", "liboracle.so")
_lock = threading.Lock()
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_fp = ctypes.POINTER(ctypes.c_float)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no -ffast-math: IEEE fp64 throughout)."""
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            i, d, i64 = ctypes.c_int, ctypes.c_double, ctypes.c_int64
            lib.oracle_envelope_naive.argtypes = [_dp, i, i, _dp, _dp]
            lib.oracle_envelope_naive.restype = None
            lib.oracle_envelope_stream.argtypes = [_dp, i, i, _dp, _dp]
            lib.oracle_envelope_stream.restype = ctypes.c_long
            lib.oracle_projection.argtypes = [_dp, _dp, _dp, i, _dp]
            lib.oracle_projection.restype = None
            lib.oracle_lb_keogh.argtypes = [_dp, _dp, i, i, i]
            lib.oracle_lb_keogh.restype = d
            lib.oracle_lb_piecewise.argtypes = [_dp, _dp, i, i, i, i]
            lib.oracle_lb_piecewise.restype = d
            lib.oracle_lb_piecewise_paper.argtypes = [_dp, _dp, i, i, i, i]
            lib.oracle_lb_piecewise_paper.restype = d
            lib.oracle_lb_improved.argtypes = [_dp, _dp, i, i, i]
            lib.oracle_lb_improved.restype = d
            lib.oracle_dtw.argtypes = [_dp, _dp, i, i, i]
            lib.oracle_dtw.restype = d
            lib.oracle_dtw_pow.argtypes = [_dp, _dp, i, i, i]
            lib.oracle_dtw_pow.restype = d
            lib.oracle_nn_brute.argtypes = [_fp, i64, i64, _fp, i64, i, i, i, i, _i64p, _dp]
            lib.oracle_nn_brute.restype = None
            lib.oracle_nn_twopass.argtypes = [_fp, i64, i64, _fp, i64, i, i, i, i, i, _i64p, _dp,
                                              _i64p]
            lib.oracle_nn_twopass.restype = None
            lib.oracle_prune_counts.argtypes = [_fp, i64, i64, _fp, i64, i, i, i, _dp, _i64p,
                                                _i64p]
            lib.oracle_prune_counts.restype = None
            _lib = lib
    return _lib


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_dp)


def _f(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.ctypes.data_as(_fp)


def envelope(y, w):
    """Warping envelope U(y), L(y) by definition."""
    y, yp = _d(y)
    n = y.shape[-1]
    U = np.empty(n)
    L = np.empty(n)
    _load().oracle_envelope_naive(yp, n, int(w), U.ctypes.data_as(_dp), L.ctypes.data_as(_dp))
    return U, L


def envelope_stream(y, w):
    """Algorithm 1, corrected per reading c1; returns (U, L, comparisons)."""
    y, yp = _d(y)
    n = y.shape[-1]
    U = np.empty(n)
    L = np.empty(n)
    c = _load().oracle_envelope_stream(yp, n, int(w), U.ctypes.data_as(_dp),
                                       L.ctypes.data_as(_dp))
    return U, L, int(c)


def projection(x, U, L):
    """H(x, y), Eq. (1), given the query envelope U, L."""
    x, xp = _d(x)
    U, up = _d(U)
    L, lp = _d(L)
    H = np.empty(x.shape[-1])
    _load().oracle_projection(xp, up, lp, x.shape[-1], H.ctypes.data_as(_dp))
    return H


def lb_keogh(x, y, w, p):
    """LB_Keogh_p(x, y) = ||x - H(x,y)||_p, rooted."""
    x, xp = _d(x)
    y, yp = _d(y)
    return _load().oracle_lb_keogh(xp, yp, x.shape[-1], int(w), int(p))


def lb_piecewise(x, y, w, p, s=8):
    """Piecewise-sum bound (p = 2 per reading c18), rooted, over the builder's
    fixed-length cover (intervals of s samples, the last one shorter; reading c18)
    that the GPU pre-filter uses."""
    x, xp = _d(x)
    y, yp = _d(y)
    return _load().oracle_lb_piecewise(xp, yp, x.shape[-1], int(w), int(s), int(p))


def lb_piecewise_paper(x, y, w, p, d=8):
    """Piecewise-sum bound over the paper's own cover (d intervals of floor(n/d),
    the last one longer; d = 8 in the experiments), rooted; p = 2 divides each
    interval's squared distance by its length (reading c18)."""
    x, xp = _d(x)
    y, yp = _d(y)
    return _load().oracle_lb_piecewise_paper(xp, yp, x.shape[-1], int(w), int(d), int(p))


def lb_improved(x, y, w, p):
    """LB_Improved_p(x, y), rooted; NaN for p = infinity."""
    x, xp = _d(x)
    y, yp = _d(y)
    return _load().oracle_lb_improved(xp, yp, x.shape[-1], int(w), int(p))


def dtw(x, y, w, p):
    """Banded monotone DTW_p(x, y) by the suffix recursion, rooted."""
    x, xp = _d(x)
    y, yp = _d(y)
    return _load().oracle_dtw(xp, yp, x.shape[-1], int(w), int(p))


def dtw_pow(x, y, w, p):
    """q_{1,1} = DTW_p(x, y)^p."""
    x, xp = _d(x)
    y, yp = _d(y)
    return _load().oracle_dtw_pow(xp, yp, x.shape[-1], int(w), int(p))


def _chunks(Q, threads):
    threads = max(1, min(int(threads), Q)) if Q > 0 else 1
    step = (Q + threads - 1) // threads if Q > 0 else 0
    return [(s, min(Q, s + step)) for s in range(0, Q, step)] if Q > 0 else []


def nn_brute(queries, db, w, p, k, threads=1):
    """Brute-force k-NN under DTW_p (ground truth): k smallest (DTW_p, index), rooted."""
    queries, qp = _f(queries)
    db, dbp = _f(db)
    Q, n = queries.shape
    N = db.shape[0]
    idx = np.full((Q, k), -1, dtype=np.int64)
    dist = np.full((Q, k), np.inf)
    lib = _load()

    def run(r):
        lib.oracle_nn_brute(qp, r[0], r[1], dbp, N, n, int(w), int(p), int(k),
                            idx.ctypes.data_as(_i64p), dist.ctypes.data_as(_dp))

    with ThreadPoolExecutor(max_workers=max(1, threads)) as ex:
        list(ex.map(run, _chunks(Q, threads)))
    return idx, dist


def nn_twopass(queries, db, w, p, k, keogh_only=False, threads=1):
    """Sequential Algorithm 3, k-generalised; returns (idx, dist, counters).

    counters = [seen, pruned_by_keogh, pruned_by_improved, dtw_evaluations].
    ``keogh_only`` runs Algorithm 2.
    """
    queries, qp = _f(queries)
    db, dbp = _f(db)
    Q, n = queries.shape
    N = db.shape[0]
    idx = np.full((Q, k), -1, dtype=np.int64)
    dist = np.full((Q, k), np.inf)
    parts = _chunks(Q, threads)
    cnts = np.zeros((max(1, len(parts)), 4), dtype=np.int64)
    lib = _load()

    def run(a):
        j, r = a
        c = cnts[j]
        lib.oracle_nn_twopass(qp, r[0], r[1], dbp, N, n, int(w), int(p), int(k),
                              int(bool(keogh_only)), idx.ctypes.data_as(_i64p),
                              dist.ctypes.data_as(_dp), c.ctypes.data_as(_i64p))

    with ThreadPoolExecutor(max_workers=max(1, threads)) as ex:
        list(ex.map(run, list(enumerate(parts))))
    return idx, dist, cnts.sum(axis=0)


def prune_counts(queries, db, w, p, tau, threads=1):
    """Order-independent counts vs the final k-th distance tau[q]: (#{LB_Keogh^p > tau^p},
    #{LB_Keogh^p <= tau^p < LB_Improved^p}) per query (pinned: test_prune_counts_pinned)."""
    queries, qp = _f(queries)
    db, dbp = _f(db)
    Q, n = queries.shape
    tau, tp = _d(tau)
    ck = np.zeros(Q, dtype=np.int64)
    ci = np.zeros(Q, dtype=np.int64)
    lib = _load()

    def run(r):
        lib.oracle_prune_counts(qp, r[0], r[1], dbp, db.shape[0], n, int(w), int(p), tp,
                                ck.ctypes.data_as(_i64p), ci.ctypes.data_as(_i64p))

    with ThreadPoolExecutor(max_workers=max(1, threads)) as ex:
        list(ex.map(run, _chunks(Q, threads)))
    return ck, ci
