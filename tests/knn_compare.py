"""Tie-class comparison of a k-NN result against the oracle (reading c14).

fp32 (GPU) and fp64 (oracle) may order near-ties differently.  Rank r of the GPU
result must name a member of the oracle's tie class of rank r -- every oracle
candidate whose distance is within relative `rel` of the oracle's r-th distance
(the class may extend beyond rank k) -- with no duplicate indices, and its
distance must be within relative `rel` of the oracle's r-th distance.  Where the
oracle's neighbouring distances differ by more than `rel`, this is exact index
equality.
"""
import numpy as np


def assert_knn_match(g_idx, g_dist, o_idx, o_dist, k, rel=1e-4, abs_tol=1e-6):
    g_idx = np.asarray(g_idx)
    g_dist = np.asarray(g_dist, dtype=np.float64)
    o_idx = np.asarray(o_idx)
    o_dist = np.asarray(o_dist, dtype=np.float64)
    Q = g_idx.shape[0]
    assert g_idx.shape[1] == k
    for q in range(Q):
        assert len(set(g_idx[q].tolist())) == k, f"query {q}: duplicate indices {g_idx[q]}"
        for r in range(k):
            d_r = o_dist[q, r]
            tol = rel * abs(d_r) + abs_tol
            cls = {int(c) for c, d in zip(o_idx[q], o_dist[q]) if abs(d - d_r) <= tol}
            # the class must be fully visible in the oracle's extended list
            assert abs(o_dist[q, -1] - d_r) > tol or o_idx.shape[1] == k or np.isinf(o_dist[q, -1]), \
                f"query {q} rank {r}: oracle list too short to see the whole tie class"
            assert int(g_idx[q, r]) in cls, (
                f"query {q} rank {r}: gpu idx {g_idx[q, r]} (d={g_dist[q, r]!r}) not in oracle tie class "
                f"{sorted(cls)} (d={d_r!r}); oracle head {o_idx[q, :k]} / {o_dist[q, :k]}")
            assert abs(g_dist[q, r] - d_r) <= tol, f"query {q} rank {r}: dist {g_dist[q, r]} vs {d_r}"
