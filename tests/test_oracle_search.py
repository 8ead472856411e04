"""Pins of the oracle's two k-NN procedures (brute force and Algorithm 3).

The method is exact: Algorithm 3 must return exactly the
brute-force k smallest by (DTW_p, index).  Brute force itself is pinned against
an independent path-enumeration DTW on tiny inputs.
"""
import numpy as np
import pytest

import datagen
import oracle
from test_oracle_pins import dtw_by_paths


def _ref_knn_by_paths(qs, db, w, p, k):
    idx = np.empty((len(qs), k), dtype=np.int64)
    dist = np.empty((len(qs), k))
    for q, y in enumerate(qs.astype(float)):
        costs = [dtw_by_paths(x, y, w, p) for x in db.astype(float)]
        order = sorted(range(len(db)), key=lambda c: (costs[c], c))[:k]
        idx[q] = order
        dist[q] = [costs[c] ** (1.0 / p) for c in order]
    return idx, dist


def test_brute_matches_path_enumeration():
    rng = np.random.default_rng(7)
    for p in (1, 2):
        qs = rng.integers(-2, 3, size=(3, 5)).astype(np.float32)
        db = rng.integers(-2, 3, size=(25, 5)).astype(np.float32)  # many exact ties
        for w in (0, 1, 4):
            for k in (1, 4, 25):
                i1, d1 = oracle.nn_brute(qs, db, w, p, k)
                i2, d2 = _ref_knn_by_paths(qs, db, w, p, k)
                assert np.array_equal(i1, i2)
                assert np.allclose(d1, d2, rtol=1e-12, atol=0)


@pytest.mark.parametrize("p", [1, 2])
@pytest.mark.parametrize("k", [1, 3])
def test_twopass_equals_brute_random_walks(p, k):
    qs, db = datagen.make("C2p1", Q=6, N=600)
    db[17] = qs[2]            # self-match => distance 0
    db[40] = db[39]           # duplicate rows => smaller index first
    db[300] = qs[4] + 0.25    # translated copy
    w = 25
    ib, dbst = oracle.nn_brute(qs, db, w, p, k, threads=4)
    it, dt, cnt = oracle.nn_twopass(qs, db, w, p, k, threads=3)
    ik, dk, cntk = oracle.nn_twopass(qs, db, w, p, k, keogh_only=True, threads=2)
    assert np.array_equal(ib, it) and np.array_equal(ib, ik)
    assert np.array_equal(dbst, dt) and np.array_equal(dbst, dk)
    assert ib[2, 0] == 17 and dbst[2, 0] == 0.0
    seen, pk, pi, nd = cnt
    assert seen == 6 * 600 and pk + pi + nd == seen                 # S:452 counter invariant
    assert cntk[2] == 0 and cntk[1] + cntk[3] == seen
    assert nd <= cntk[3]                                             # LB_Improved prunes at least as much


def test_twopass_equals_brute_C1_full():
    qs, db = datagen.make("C1")
    c = datagen.CONFIGS["C1"]
    ib, dbst = oracle.nn_brute(qs, db, c.w, c.p, c.k)
    it, dt, cnt = oracle.nn_twopass(qs, db, c.w, c.p, c.k)
    assert np.array_equal(ib, it) and np.array_equal(dbst, dt)
    assert cnt[3] < c.N  # something was pruned


def test_strict_fixture_as_database():
    """Query (3,4,1,4), DB {(4,0,3,2), (3,4,1,4)}, w=1, p=1: index 1 at 0;
    with k=2 row 0 follows at DTW_1 = 5 (hand-derived fixture)."""
    qs = np.array([[3, 4, 1, 4]], np.float32)
    db = np.array([[4, 0, 3, 2], [3, 4, 1, 4]], np.float32)
    i, d = oracle.nn_brute(qs, db, 1, 1, 2)
    assert i.tolist() == [[1, 0]] and d.tolist() == [[0.0, 5.0]]
    i2, d2, cnt = oracle.nn_twopass(qs, db, 1, 1, 1)
    assert i2.tolist() == [[1]] and d2.tolist() == [[0.0]]


def test_k_equals_N_and_padding():
    qs, db = datagen.make("C1", Q=2, N=12)
    i, d = oracle.nn_brute(qs, db, 12, 1, 12)
    assert sorted(i[0].tolist()) == list(range(12)) and np.all(np.diff(d[0]) >= 0)
    i2, d2, _ = oracle.nn_twopass(qs, db, 12, 1, 12)
    assert np.array_equal(i, i2)
    i3, d3 = oracle.nn_brute(qs, db, 12, 1, 15)   # k > N pads with (-1, inf) in the oracle
    assert np.all(i3[:, 12:] == -1) and np.all(np.isinf(d3[:, 12:]))
