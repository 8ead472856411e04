"""Pin of DESIGN.md reading c22 (the DTW walk's abandon schedule), brute force on tiny inputs.

The walk abandons a pair after 8k rows when  rowmin_k + R[k] > tau^p (1 + eps) (the row part
from the pair's +-beta1 gate word minus the computed rows' terms, the column part from the
schedule the survivor kernel wrote), where
rowmin_k is the minimum of the banded DTW table's row 8k-1 and

    R[k] = sum_{r >= 8k} d(x_r, [L(y)_r, U(y)_r])^p + sum_{c >= 8k + 4 ceil(w/4)} d(y_c, [L(H)_c, U(H)_c])^p

(row terms: LB_Keogh's; column terms: LB_Improved's second sum, H the
projection of x on the envelope of y).  Exactness needs  rowmin_k + R[k] <= DTW_p^p(x, y)  for
every k; at k = 0 the column sum starts at 4 ceil(w/4) and R[0] <= LB_Improved^p.  Checked
here by brute force: the full banded DP (written out below) on random walks,
plus the oracle's LB_Keogh / LB_Improved as an independent cross-check of the two sums.
"""
import numpy as np
import pytest

import oracle


def _banded_table(x, y, w, p):
    n = len(x)
    D = np.full((n, n), np.inf)
    for i in range(n):
        for j in range(max(0, i - w), min(n, i + w + 1)):
            c = abs(x[i] - y[j]) ** p
            if i == 0 and j == 0:
                D[i, j] = c
                continue
            best = np.inf
            if i > 0:
                best = min(best, D[i - 1, j])
                if j > 0:
                    best = min(best, D[i - 1, j - 1])
            if j > 0:
                best = min(best, D[i, j - 1])
            D[i, j] = c + best
    return D


def _env(a, w):
    n = len(a)
    U = np.array([a[max(0, i - w):min(n, i + w + 1)].max() for i in range(n)])
    L = np.array([a[max(0, i - w):min(n, i + w + 1)].min() for i in range(n)])
    return U, L


def _terms(x, y, w, p):
    U, L = _env(y, w)
    row = np.maximum(np.maximum(x - U, L - x), 0.0) ** p
    H = np.minimum(np.maximum(x, L), U)
    UH, LH = _env(H, w)
    col = np.maximum(np.maximum(y - UH, LH - y), 0.0) ** p
    return row, col


@pytest.mark.parametrize("n,w,p", [(32, 3, 2), (48, 5, 1), (64, 8, 2), (40, 13, 2), (24, 0, 2)])
def test_schedule_bounds_every_completion(n, w, p):
    rng = np.random.default_rng(1000 * n + w + p)
    c0 = 4 * ((w + 3) // 4)
    tight = 0
    for trial in range(60):
        x = np.cumsum(rng.standard_normal(n))
        y = x + rng.standard_normal(n) * (0.3 if trial % 2 else 1.5) if trial % 3 else np.cumsum(rng.standard_normal(n))
        D = _banded_table(x, y, w, p)
        dtw_p = D[n - 1, n - 1]
        row, col = _terms(x, y, w, p)
        # the two sums are LB_Keogh^p and LB_Improved^p - LB_Keogh^p (oracle, fp64)
        assert row.sum() == pytest.approx(oracle.lb_keogh(x, y, w, p) ** p, rel=1e-9, abs=1e-12)
        assert row.sum() + col.sum() == pytest.approx(oracle.lb_improved(x, y, w, p) ** p, rel=1e-9, abs=1e-12)
        assert dtw_p == pytest.approx(oracle.dtw(x, y, w, p) ** p, rel=1e-9)
        for k in range(1, (n - 1) // 8 + 1):
            i = 8 * k
            R = row[i:].sum() + col[min(n, i + c0):].sum()
            rowmin = D[i - 1].min()
            assert rowmin + R <= dtw_p * (1 + 1e-12) + 1e-12, (trial, k)
            tight += rowmin + R > 0.9 * dtw_p
        # the walk's start value: LB_Improved^p minus the column head (reading c22)
        assert row.sum() + col[c0:].sum() <= dtw_p * (1 + 1e-12) + 1e-12
    assert tight > 0  # the bound is not vacuous on these inputs


def test_schedule_column_offset_is_needed():
    """Without the w offset (columns from 8k instead of 8k + w) the bound can exceed DTW:
    a computed row may already have paid a column's term -- the offset is load-bearing."""
    rng = np.random.default_rng(7)
    n, w, p = 32, 6, 2
    bad = 0
    for _ in range(200):
        x = np.cumsum(rng.standard_normal(n))
        y = np.cumsum(rng.standard_normal(n))
        D = _banded_table(x, y, w, p)
        row, col = _terms(x, y, w, p)
        for k in range(1, (n - 1) // 8 + 1):
            i = 8 * k
            bad += D[i - 1].min() + row[i:].sum() + col[i:].sum() > D[n - 1, n - 1] * (1 + 1e-9)
    assert bad > 0
