"""Pins of the fp64 oracle against what the paper and mathematics fix.

Every check here is independent of the oracle's own code path: printed paper
values (tests/golden/paper_values.json, each with its citation), brute force
from the *definition* (enumeration of warping paths / matchings), library
routines for special cases, closed forms and the paper's inequalities.
Integer-valued samples keep fp64 arithmetic exact where equality is asserted.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
RNG = np.random.default_rng(20260101)


def lp(a, b, p):
    d = np.abs(np.asarray(a, float) - np.asarray(b, float))
    return d.max() if p == 0 else (d ** p).sum() ** (1.0 / p)


# ---------------------------------------------------------------- brute force
def dtw_by_matchings(x, y, w, p):
    """DTW from the definition: the minimum over all
    monotone many-to-many matchings Gamma inside the band |i-j| <= w that cover
    every index of x and of y, of the l_p norm of {x_i - y_j}.  Enumerates every
    subset of band cells (tiny n only)."""
    n = len(x)
    cells = [(i, j) for i in range(n) for j in range(n) if abs(i - j) <= w]
    best = math.inf
    for r in range(1, len(cells) + 1):
        for gamma in itertools.combinations(cells, r):
            if {i for i, _ in gamma} != set(range(n)) or {j for _, j in gamma} != set(range(n)):
                continue
            mono = all(not (a[0] < b[0] and a[1] > b[1]) and not (a[0] > b[0] and a[1] < b[1])
                       for a in gamma for b in gamma)
            if not mono:
                continue
            d = [abs(x[i] - y[j]) for i, j in gamma]
            cost = max(d) if p == 0 else sum(v ** p for v in d)
            best = min(best, cost)
    return best  # p-th power (or max for p = inf)


def dtw_by_paths(x, y, w, p):
    """DTW as the minimum over explicit monotone lattice paths (0,0)->(n-1,n-1)
    with unit steps, inside the band; enumerated path by path (no DP)."""
    n = len(x)
    best = [math.inf]

    def rec(i, j, acc):
        c = abs(x[i] - y[j])
        acc = max(acc, c) if p == 0 else acc + c ** p
        if acc >= best[0]:
            return
        if i == n - 1 and j == n - 1:
            best[0] = acc
            return
        for di, dj in ((1, 0), (0, 1), (1, 1)):
            a, b = i + di, j + dj
            if a < n and b < n and abs(a - b) <= w:
                rec(a, b, acc)

    rec(0, 0, 0.0)
    return best[0]


def rand_int_series(n):
    return RNG.integers(-2, 3, size=n).astype(float)


# ---------------------------------------------------------------- envelope
@pytest.mark.parametrize("case", GOLDEN["envelope"], ids=lambda c: c["cite"][:30])
def test_envelope_golden(case):
    U, L = oracle.envelope(case["y"], case["w"])
    assert U.tolist() == case["U"] and L.tolist() == case["L"]
    U2, L2, _ = oracle.envelope_stream(case["y"], case["w"])
    assert U2.tolist() == case["U"] and L2.tolist() == case["L"]


def _env_numpy(y, w):
    from numpy.lib.stride_tricks import sliding_window_view
    n = len(y)
    w = min(w, n - 1)
    pad_hi = np.concatenate([np.full(w, -np.inf), y, np.full(w, -np.inf)])
    pad_lo = np.concatenate([np.full(w, np.inf), y, np.full(w, np.inf)])
    return (sliding_window_view(pad_hi, 2 * w + 1).max(axis=1),
            sliding_window_view(pad_lo, 2 * w + 1).min(axis=1))


def test_envelope_vs_library_and_streaming():
    """Definition == numpy sliding-window max/min; corrected Alg. 1 == definition
    with <= 3n comparisons; w = 0 gives y; w >= n-1 gives global max/min."""
    for _ in range(3000):
        n = int(RNG.integers(1, 40))
        w = int(RNG.integers(0, n + 3))
        kind = RNG.integers(0, 4)
        if kind == 0:
            y = RNG.standard_normal(n)
        elif kind == 1:
            y = RNG.integers(-2, 3, size=n).astype(float)  # many ties
        elif kind == 2:
            y = np.arange(n, dtype=float) * (1 if RNG.random() < 0.5 else -1)  # monotone
        else:
            y = np.full(n, 1.5)
        U, L = oracle.envelope(y, w)
        Un, Ln = _env_numpy(y, w)
        assert np.array_equal(U, Un) and np.array_equal(L, Ln)
        Us, Ls, cmp = oracle.envelope_stream(y, w)
        assert np.array_equal(U, Us) and np.array_equal(L, Ls)
        assert cmp <= 3 * n
        if w == 0:
            assert np.array_equal(U, y) and np.array_equal(L, y)
        if w >= n - 1:
            assert np.all(U == y.max()) and np.all(L == y.min())


def test_envelope_monotone_in_w():
    for _ in range(300):
        n = int(RNG.integers(2, 30))
        y = RNG.standard_normal(n)
        w1 = int(RNG.integers(0, n))
        w2 = int(RNG.integers(w1, n + 2))
        U1, L1 = oracle.envelope(y, w1)
        U2, L2 = oracle.envelope(y, w2)
        assert np.all(U1 <= U2) and np.all(L1 >= L2) and np.all(L1 <= y) and np.all(y <= U1)


# ---------------------------------------------------------------- DTW
@pytest.mark.parametrize("case", GOLDEN["dtw"], ids=lambda c: c["cite"][:30])
def test_dtw_golden(case):
    if "rooted" in case:
        assert oracle.dtw(case["x"], case["y"], case["w"], case["p"]) == pytest.approx(case["rooted"], abs=1e-12)
    else:
        assert oracle.dtw_pow(case["x"], case["y"], case["w"], case["p"]) == pytest.approx(case["value_pow"], abs=1e-12)


def test_dtw_equals_definition_by_matchings():
    """Exhaustive over all band matchings for n <= 3 (every w), several n = 4."""
    for n in (1, 2, 3):
        for _ in range(60):
            x, y = rand_int_series(n), rand_int_series(n)
            for w in range(0, n + 1):
                for p in (1, 2, 0):
                    assert oracle.dtw_pow(x, y, w, p) == dtw_by_matchings(x, y, w, p)
    for _ in range(6):
        x, y = rand_int_series(4), rand_int_series(4)
        for w in (1, 3):
            for p in (1, 2):
                assert oracle.dtw_pow(x, y, w, p) == dtw_by_matchings(x, y, w, p)


def test_dtw_equals_path_enumeration():
    """All monotone lattice paths in the band, n <= 7, integer samples (exact)."""
    for _ in range(400):
        n = int(RNG.integers(1, 8))
        x, y = rand_int_series(n), rand_int_series(n)
        w = int(RNG.integers(0, n + 1))
        for p in (1, 2, 0):
            assert oracle.dtw_pow(x, y, w, p) == dtw_by_paths(x, y, w, p)


def test_dtw_properties():
    for _ in range(500):
        n = int(RNG.integers(1, 24))
        x, y = RNG.standard_normal(n), RNG.standard_normal(n)
        for p in (1, 2):
            d0 = oracle.dtw(x, y, 0, p)
            assert d0 == pytest.approx(lp(x, y, p), rel=1e-12)                 # w=0 => l_p
            prev = d0
            for w in range(1, min(n, 6) + 1):
                d = oracle.dtw(x, y, w, p)
                assert d <= prev * (1 + 1e-12)                                 # non-increasing in w
                assert d == pytest.approx(oracle.dtw(y, x, w, p), rel=1e-12)   # symmetric
                b = RNG.standard_normal()
                assert d == pytest.approx(oracle.dtw(x + b, y + b, w, p), rel=1e-9, abs=1e-12)
                prev = d
            assert oracle.dtw(x, y, n, p) <= lp(x, y, p) * (1 + 1e-12)         # DTW <= l_p
            c = RNG.standard_normal()
            w = int(RNG.integers(0, n + 1))
            assert oracle.dtw(x, np.full(n, c), w, p) == pytest.approx(lp(x, np.full(n, c), p), rel=1e-12)
        if n > 1:                                                              # P:1027-1029, p=1,q=2
            w = int(RNG.integers(0, n + 1))
            assert math.sqrt(2 * n - 2) * oracle.dtw(x, y, w, 2) >= oracle.dtw(x, y, w, 1) * (1 - 1e-12)


def test_prop1_value_separation():
    """x >= c >= y => DTW_1 = ||x - y||_1 (Prop. 1)."""
    for _ in range(300):
        n = int(RNG.integers(1, 20))
        c = RNG.standard_normal()
        x = c + np.abs(RNG.standard_normal(n))
        y = c - np.abs(RNG.standard_normal(n))
        w = int(RNG.integers(0, n + 1))
        assert oracle.dtw(x, y, w, 1) == pytest.approx(np.abs(x - y).sum(), rel=1e-12)
        assert oracle.dtw(y, x, w, 1) == pytest.approx(np.abs(x - y).sum(), rel=1e-12)


def test_weak_triangle_inequality():
    """DTW(x,y) + DTW(y,z) >= DTW(x,z) / min(2w+1, n)^(1/p)."""
    for _ in range(300):
        n = int(RNG.integers(1, 16))
        x, y, z = (RNG.standard_normal(n) for _ in range(3))
        w = int(RNG.integers(0, n + 1))
        for p in (1, 2):
            lhs = oracle.dtw(x, y, w, p) + oracle.dtw(y, z, w, p)
            assert lhs >= oracle.dtw(x, z, w, p) / min(2 * w + 1, n) ** (1.0 / p) * (1 - 1e-12)


# ---------------------------------------------------------------- bounds
@pytest.mark.parametrize("case", GOLDEN["bounds"], ids=lambda c: c["cite"][:30])
def test_bounds_golden(case):
    x, y, w, p = case["x"], case["y"], case["w"], case["p"]
    assert oracle.lb_keogh(x, y, w, p) ** p == pytest.approx(case["keogh_pow"], abs=1e-12)
    assert oracle.lb_improved(x, y, w, p) ** p == pytest.approx(case["improved_pow"], abs=1e-12)
    if "dtw_pow" in case:
        assert oracle.dtw_pow(x, y, w, p) == pytest.approx(case["dtw_pow"], abs=1e-12)
        assert dtw_by_paths(np.array(x, float), np.array(y, float), w, p) == case["dtw_pow"]
    if "H" in case:
        U, L = oracle.envelope(y, w)
        assert oracle.projection(x, U, L).tolist() == case["H"]


def test_bound_chain_and_paper_inequalities():
    """LB_Keogh <= LB_Improved <= DTW;
    LB_Keogh^p + DTW(H,y)^p <= DTW^p (Theorem 1, P:292-299 with h = H);
    DTW - LB_Keogh <= ||H - y||_p (Prop. 2);
    DTW - LB_Keogh <= ||max(U - y, y - L)||_p (corollary);
    x inside the envelope => LB_Keogh = 0; w = 0 => LB_Keogh = l_p."""
    for _ in range(1500):
        n = int(RNG.integers(1, 12))
        integer = RNG.random() < 0.5
        x = rand_int_series(n) if integer else RNG.standard_normal(n)
        y = rand_int_series(n) if integer else RNG.standard_normal(n)
        w = int(RNG.integers(0, n + 1))
        U, L = oracle.envelope(y, w)
        H = oracle.projection(x, U, L)
        for p in (1, 2):
            kb = oracle.lb_keogh(x, y, w, p)
            ib = oracle.lb_improved(x, y, w, p)
            d = oracle.dtw(x, y, w, p)
            tol = 1e-12 * (1 + d)
            assert kb <= ib + tol and ib <= d + tol
            if integer:
                assert dtw_by_paths(x, y, w, p) == pytest.approx(d ** p, abs=1e-9)
            assert kb ** p + oracle.dtw_pow(H, y, w, p) <= d ** p + 1e-9 * (1 + d ** p)
            assert d - kb <= lp(H, y, p) + tol
            assert d - kb <= lp(np.maximum(U - y, y - L), 0, p) + tol
            if w == 0:
                assert kb == pytest.approx(lp(x, y, p), rel=1e-12, abs=1e-12)
        inside = np.clip(RNG.standard_normal(n), L, U)
        assert oracle.lb_keogh(inside, y, w, 1) == 0.0
        assert oracle.lb_keogh(y, y, w, 2) == 0.0 and oracle.lb_improved(y, y, w, 2) == 0.0


def test_value_separated_error_is_exact():
    """x >= c >= y: DTW_1 = ||x-H||_1 + ||H-y||_1 exactly."""
    for _ in range(200):
        n = int(RNG.integers(1, 15))
        c = float(RNG.integers(-3, 4))
        x = c + RNG.integers(0, 4, size=n).astype(float)
        y = c - RNG.integers(0, 4, size=n).astype(float)
        w = n  # full-width window
        U, L = oracle.envelope(y, w)
        H = oracle.projection(x, U, L)
        d = oracle.dtw(x, y, w, 1)
        assert d == np.abs(x - y).sum()
        assert d == np.abs(x - H).sum() + np.abs(H - y).sum()


def test_lb_improved_rejects_infinity():
    assert math.isnan(oracle.lb_improved([1, 2], [2, 1], 1, 0))


# ---------------------------------------------------------------- piecewise-sum pre-filter
def test_reverse_piecewise_symmetric_gate():
    """Reading c20: the piecewise-sum bound with query and candidate exchanged,
    lb_piecewise(y | envelope of x), is a lower bound of LB_Keogh_p(y, x) <= DTW_p(y, x)
    = DTW_p(x, y) (symmetry), so max(forward, reverse) <= DTW_p(x, y).  Pinned by:
    s = 1 reverse == sum_i d(y_i, [L(x)_i, U(x)_i])^p with numpy's sliding-window envelope
    of x; the chain on random cases; and the hand-checked fixture x = (0,0,0), y = (0,5,0),
    w = 1: forward 0 (x inside the envelope of y), reverse 5 = DTW_1 (p = 1),
    and with one interval (s = 3) reverse^2 = 5^2 / 3 for p = 2."""
    from numpy.lib.stride_tricks import sliding_window_view as swv
    x, y = np.zeros(3), np.array([0.0, 5.0, 0.0])
    assert oracle.lb_piecewise(x, y, 1, 1, 1) == 0.0
    assert oracle.lb_piecewise(y, x, 1, 1, 1) == 5.0 == oracle.dtw(x, y, 1, 1)
    assert oracle.lb_piecewise(y, x, 1, 2, 3) ** 2 == pytest.approx(25.0 / 3, rel=1e-12)
    for _ in range(1000):
        n = int(RNG.integers(1, 14))
        integer = RNG.random() < 0.5
        x = rand_int_series(n) if integer else RNG.standard_normal(n)
        y = rand_int_series(n) if integer else RNG.standard_normal(n)
        w = int(RNG.integers(0, n + 1))
        we = min(w, n - 1)
        xp = np.pad(np.asarray(x, float), (we, we), mode="edge")
        Ux, Lx = swv(xp, 2 * we + 1).max(axis=1), swv(xp, 2 * we + 1).min(axis=1)
        yv = np.asarray(y, float)
        for p in (1, 2):
            rev_keogh = float(np.sum(np.maximum(np.maximum(yv - Ux, Lx - yv), 0.0) ** p))
            assert oracle.lb_piecewise(y, x, w, p, 1) ** p == pytest.approx(rev_keogh, rel=1e-12, abs=1e-12)
            d = oracle.dtw(x, y, w, p)
            tol = 1e-12 * (1 + d)
            for s in (1, 2, 4, 8):
                sym = max(oracle.lb_piecewise(x, y, w, p, s), oracle.lb_piecewise(y, x, w, p, s))
                assert sym <= d + tol


@pytest.mark.parametrize("case", GOLDEN["piecewise"], ids=lambda c: c["cite"][:30])
def test_piecewise_golden(case):
    """Hand-derived values of the piecewise-sum bound (p = 2 reading c18)."""
    v = oracle.lb_piecewise(case["x"], case["y"], case["w"], case["p"], case["s"]) ** case["p"]
    assert v == pytest.approx(case["value_pow"], abs=1e-12)


def test_piecewise_chain_and_special_cases():
    """piecewise <= LB_Keogh <= DTW (P:656-660 chain; p = 2 by Cauchy-Schwarz per interval);
    s = 1 reduces to LB_Keogh; one interval (s >= n) is d(sum x, [sum L, sum U]) with the
    envelope from numpy's sliding window (library routine); larger s never tightens when s
    divides evenly (coarser cover of a refinement)."""
    from numpy.lib.stride_tricks import sliding_window_view as swv
    for _ in range(1500):
        n = int(RNG.integers(1, 14))
        integer = RNG.random() < 0.5
        x = rand_int_series(n) if integer else RNG.standard_normal(n)
        y = rand_int_series(n) if integer else RNG.standard_normal(n)
        w = int(RNG.integers(0, n + 1))
        for p in (1, 2):
            kb = oracle.lb_keogh(x, y, w, p)
            d = oracle.dtw(x, y, w, p)
            tol = 1e-12 * (1 + d)
            assert oracle.lb_piecewise(x, y, w, p, 1) == pytest.approx(kb, rel=1e-12, abs=1e-12)
            for s in (2, 3, 4, 8):
                pw = oracle.lb_piecewise(x, y, w, p, s)
                assert pw <= kb + tol and pw <= d + tol
            if n % 4 == 0:
                assert oracle.lb_piecewise(x, y, w, p, 4) <= oracle.lb_piecewise(x, y, w, p, 2) + tol
            we = min(w, n - 1)
            yp = np.pad(np.asarray(y, float), (we, we), mode="edge")
            U = swv(yp, 2 * we + 1).max(axis=1)
            L = swv(yp, 2 * we + 1).min(axis=1)
            sx, su, sl = float(np.sum(x)), float(U.sum()), float(L.sum())
            one = max(sx - su, sl - sx, 0.0)
            expect = one if p == 1 else one * one / n
            assert oracle.lb_piecewise(x, y, w, p, n) ** p == pytest.approx(expect, rel=1e-9, abs=1e-9)


# ---------------------------------------------------------------- the paper's own cover
@pytest.mark.parametrize("case", GOLDEN["piecewise_paper_cover"], ids=lambda c: c["cite"][:30])
def test_piecewise_paper_cover_golden(case):
    """Hand-derived values over the paper's cover P:661-665 (d intervals of floor(n/d), the
    last one longer)."""
    v = oracle.lb_piecewise_paper(case["x"], case["y"], case["w"], case["p"], case["d"]) ** case["p"]
    assert v == pytest.approx(case["value_pow"], abs=1e-12)


def test_piecewise_paper_cover_special_cases():
    """The paper's cover: d = n is LB_Keogh (one sample per interval); d = 1 is one
    interval, d(sum x, [sum L, sum U]) with numpy's sliding-window envelope (library routine);
    when d divides n it equals the builder's fixed-length cover with s = n/d; always
    <= LB_Keogh <= DTW; d outside [1, n] is rejected (NaN)."""
    from numpy.lib.stride_tricks import sliding_window_view as swv
    for _ in range(800):
        n = int(RNG.integers(1, 16))
        integer = RNG.random() < 0.5
        x = rand_int_series(n) if integer else RNG.standard_normal(n)
        y = rand_int_series(n) if integer else RNG.standard_normal(n)
        w = int(RNG.integers(0, n + 1))
        for p in (1, 2):
            kb = oracle.lb_keogh(x, y, w, p)
            dd = oracle.dtw(x, y, w, p)
            tol = 1e-12 * (1 + dd)
            assert oracle.lb_piecewise_paper(x, y, w, p, n) == pytest.approx(kb, rel=1e-12, abs=1e-12)
            for d in range(1, n + 1):
                v = oracle.lb_piecewise_paper(x, y, w, p, d)
                assert v <= kb + tol and v <= dd + tol
                if n % d == 0:
                    assert v == pytest.approx(oracle.lb_piecewise(x, y, w, p, n // d), rel=1e-12, abs=1e-12)
            we = min(w, n - 1)
            yp = np.pad(np.asarray(y, float), (we, we), mode="edge")
            U, L = swv(yp, 2 * we + 1).max(axis=1), swv(yp, 2 * we + 1).min(axis=1)
            sx = float(np.sum(x))
            one = max(sx - float(U.sum()), float(L.sum()) - sx, 0.0)
            expect = one if p == 1 else one * one / n
            assert oracle.lb_piecewise_paper(x, y, w, p, 1) ** p == pytest.approx(expect, rel=1e-9, abs=1e-9)
    assert math.isnan(oracle.lb_piecewise_paper([1.0, 2.0], [0.0, 0.0], 1, 1, 3))
    assert math.isnan(oracle.lb_piecewise_paper([1.0, 2.0], [0.0, 0.0], 1, 1, 0))


# ---------------------------------------------------------------- order-independent prune counts
def _numpy_bounds_pow(x, y, w, p):
    """LB_Keogh^p and LB_Improved^p by numpy (independent of the oracle's C code): sliding-window
    envelopes (library routine), the projection H = clip(x, L, U) of Eq. (1), the
    envelope of H, and the point-to-interval distances."""
    from numpy.lib.stride_tricks import sliding_window_view as swv
    n = len(y)
    we = min(w, n - 1)

    def env(v):
        vp = np.pad(np.asarray(v, float), (we, we), mode="edge")
        return swv(vp, 2 * we + 1).max(axis=1), swv(vp, 2 * we + 1).min(axis=1)

    x, y = np.asarray(x, float), np.asarray(y, float)
    U, L = env(y)
    H = np.clip(x, L, U)
    b1 = float(np.sum(np.abs(x - H) ** p))
    U2, L2 = env(H)
    b2 = float(np.sum(np.maximum(np.maximum(y - U2, L2 - y), 0.0) ** p))
    return b1, b1 + b2


@pytest.mark.parametrize("p,k", [(1, 1), (2, 1), (2, 3)])
def test_prune_counts_pinned(p, k):
    """oracle_prune_counts (SURVEY 8(c) "Prune rates" row), pinned against (1) the same counts
    from numpy bounds (independent code; candidates whose bound is within 1e-9 relative of tau
    may fall either way) and (2) the invariants that tie them to the paper's Alg. 3
    (P:578-620): Alg. 3 compares each bound with its CURRENT k-th best, which is never below the
    final tau, so the sequential scan evaluates LB_Improved on >= N - #keogh and DTW on
    >= N - #keogh - #improved candidates; and every candidate with DTW <= tau survives both
    bounds, so N - #keogh - #improved >= #{DTW <= tau} >= k."""
    rng = np.random.default_rng(77 + p + k)
    Q, N, n, w = 6, 60, 24, 3
    walk = lambda m: np.cumsum(rng.standard_normal((m, n)), axis=1).astype(np.float32)
    qs, db = walk(Q), walk(N)
    idx, dist = oracle.nn_brute(qs, db, w, p, k)
    tau = dist[:, k - 1]
    ck, ci = oracle.prune_counts(qs, db, w, p, tau)
    seen_keogh_evals = 0
    for q in range(Q):
        tp = float(tau[q]) ** p
        lo, hi = tp * (1 - 1e-9), tp * (1 + 1e-9)
        nk_lo = nk_hi = ni_lo = ni_hi = 0
        n_le = 0
        for c in range(N):
            b1, bi = _numpy_bounds_pow(db[c].astype(float), qs[q].astype(float), w, p)
            if b1 > hi:
                nk_lo += 1; nk_hi += 1
                continue
            if b1 > lo:  # ambiguous at the tolerance: may be counted by either
                nk_hi += 1
            if bi > hi:
                ni_lo += 1; ni_hi += 1
            elif bi > lo:
                ni_hi += 1
            if oracle.dtw_pow(db[c], qs[q], w, p) <= hi:
                n_le += 1
        assert nk_lo <= ck[q] <= nk_hi
        assert ni_lo - (nk_hi - nk_lo) <= ci[q] <= ni_hi + (nk_hi - nk_lo)
        assert N - ck[q] - ci[q] >= n_le >= k
        # sequential Alg. 3 on this query alone
        _, _, cnt = oracle.nn_twopass(qs[q:q + 1], db, w, p, k)
        seen, pk, pi, ndtw = (int(v) for v in cnt)
        assert seen == N and pk + pi + ndtw == N
        assert seen - pk >= N - ck[q]
        assert ndtw >= N - ck[q] - ci[q]
        seen_keogh_evals += seen - pk
    assert seen_keogh_evals > 0
