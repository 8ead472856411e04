"""Parity of each C-ABI kernel entry point against the fp64 oracle (GPU only).

Tolerances: envelope bit-exact (min/max do not round);
LB_Keogh / LB_Improved relative 1e-5; DTW relative 1e-4 (BASELINE north_star).
Shapes span several CTA tiles plus ragged tails (n not a multiple of 4 or 32,
N not a multiple of the 128-candidate tile), w = 0, w >= n, w > 64 (generic DTW).
"""
import os

import numpy as np
import pytest
import torch

import datagen
import oracle

pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(11)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def series(rows, n, kind="rw"):
    if kind == "rw":
        return datagen.random_walks(rows, n, seed=int(RNG.integers(1 << 30)), znorm=True)
    if kind == "ties":
        return RNG.integers(-2, 3, size=(rows, n)).astype(np.float32)
    if kind == "raw":
        return datagen.random_walks(rows, n, seed=int(RNG.integers(1 << 30)), znorm=False) * 37.0
    raise ValueError(kind)


def paa_abs_tol(p, *rows):
    """Absolute slack of the outward-rounded piecewise-sum bound (readings c13, c18): each segment
    sum of s = 8 samples is held as an fp32 interval about one ulp of its magnitude wide (directed
    fp64 sum, then directed rounding to fp32), and the GPU bound is computed against those
    intervals, so each segment distance d_j may sit below the exact one by up to ~2 ulp(8 max|x|).
    Over D = ceil(n/8) segments: a sum for p = 1 (D times that), a rooted l2 norm for p = 2 (sqrt(D)
    times, by the triangle inequality); factor 2 for the accumulation's own rounding."""
    m = max(float(np.abs(r).max()) for r in rows)
    D = max(1, (rows[0].shape[1] + 7) // 8)
    ulp = float(np.spacing(np.float32(8.0 * m)))
    return 4.0 * ulp * (D if p == 1 else np.sqrt(D))


def close(g, o, rel, abs_=0.0):
    g = np.asarray(g, np.float64)
    o = np.asarray(o, np.float64)
    err = np.abs(g - o) - (rel * np.abs(o) + abs_)
    i = int(np.argmax(err))
    assert err.max() <= 0, f"max violation at {np.unravel_index(i, g.shape)}: gpu {g.flat[i]!r} oracle {o.flat[i]!r}"


ENV_CASES = [(1, 0), (1, 5), (2, 1), (3, 1), (4, 2), (7, 3), (128, 12), (256, 25), (257, 25), (512, 51),
             (1000, 50), (100, 99), (64, 200), (33, 0), (4000, 1500)]


@pytest.mark.parametrize("n,w", ENV_CASES)
@pytest.mark.parametrize("kind", ["rw", "ties"])
def test_envelope_bitwise(cuda_ok, n, w, kind):
    from paper_0811_3301_b200 import lb_envelope
    rows = 37
    x = series(rows, n, kind)
    x[0] = np.arange(n, dtype=np.float32)  # strictly monotone row
    x[1] = 1.25                            # constant row
    U, L = lb_envelope(dev(x), w)
    U, L = U.cpu().numpy(), L.cpu().numpy()
    for r in range(rows):
        Uo, Lo = oracle.envelope(x[r].astype(np.float64), w)
        assert np.array_equal(U[r], Uo.astype(np.float32)) and np.array_equal(L[r], Lo.astype(np.float32)), r


BOUND_CASES = [(4, 1), (7, 3), (128, 12), (256, 25), (257, 25), (512, 51), (1000, 50), (64, 100), (33, 0)]


def _env_dev(q, w):
    from paper_0811_3301_b200 import lb_envelope
    U, L = lb_envelope(dev(q), w)
    return torch.stack([U, L]).contiguous()


@pytest.mark.parametrize("n,w", BOUND_CASES)
@pytest.mark.parametrize("p", [1, 2])
def test_lb_keogh_and_improved(cuda_ok, n, w, p):
    from paper_0811_3301_b200 import lb_improved, lb_keogh
    Q, N = 67, 300  # > one 64-query tile, > two 128-candidate tiles, ragged
    if n >= 512:
        Q, N = 9, 140
    kind = "raw" if n == 128 else "rw"
    qs, db = series(Q, n, kind), series(N, n, kind)
    db[5] = qs[3]                      # identical row => both bounds 0
    q_env = _env_dev(qs, w)
    kb = lb_keogh(q_env, dev(db), p).cpu().numpy()
    ib = lb_improved(dev(qs), q_env, dev(db), w, p).cpu().numpy()
    ok = np.empty((Q, N))
    oi = np.empty((Q, N))
    for q in range(Q):
        for c in range(N):
            ok[q, c] = oracle.lb_keogh(db[c], qs[q], w, p)
            oi[q, c] = oracle.lb_improved(db[c], qs[q], w, p)
    close(kb, ok, 1e-5, 1e-6)
    close(ib, oi, 1e-5, 1e-6)
    assert kb[3, 5] == 0.0 and ib[3, 5] == 0.0
    assert np.all(ib >= kb * (1 - 1e-6))


@pytest.mark.parametrize("n,w", BOUND_CASES + [(1, 0), (9, 2), (1001, 50)])
@pytest.mark.parametrize("p", [1, 2])
def test_lb_piecewise(cuda_ok, n, w, p):
    """Pre-filter bound (s = 8): outward rounding keeps the GPU value at or
    below the exact (fp64) bound, within relative 1e-5 of it; never above LB_Keogh."""
    from paper_0811_3301_b200 import lb_keogh, lb_piecewise
    Q, N = 67, 300
    if n >= 512:
        Q, N = 9, 140
    kind = "raw" if n == 128 else "rw"
    qs, db = series(Q, n, kind), series(N, n, kind)
    db[5] = qs[3]
    q_env = _env_dev(qs, w)
    pw = lb_piecewise(q_env, dev(db), p).cpu().numpy().astype(np.float64)
    kb = lb_keogh(q_env, dev(db), p).cpu().numpy().astype(np.float64)
    op = np.array([[oracle.lb_piecewise(db[c], qs[q], w, p, 8) for c in range(N)] for q in range(Q)])
    assert np.all(pw <= op * (1 + 1e-7) + 1e-30), "outward rounding violated"
    close(pw, op, 1e-5, max(1e-5, paa_abs_tol(p, qs, db)))
    assert np.all(pw <= kb * (1 + 1e-5) + 1e-6)
    assert pw[3, 5] == 0.0


@pytest.mark.parametrize("n,w", BOUND_CASES + [(1, 0), (9, 2), (1001, 50)])
@pytest.mark.parametrize("p", [1, 2])
def test_lb_piecewise_sym(cuda_ok, n, w, p):
    """Symmetric gate (reading c20): max of the forward and the reverse piecewise-sum
    bounds, at or below the exact fp64 value (outward rounding), within relative 1e-5 of
    it, never above DTW_p."""
    from paper_0811_3301_b200 import dtw_band, lb_piecewise_sym
    Q, N = 37, 200
    if n >= 512:
        Q, N = 7, 90
    kind = "raw" if n == 128 else "rw"
    qs, db = series(Q, n, kind), series(N, n, kind)
    db[5] = qs[3]
    ps = lb_piecewise_sym(dev(qs), _env_dev(qs, w), dev(db), w, p).cpu().numpy().astype(np.float64)
    op = np.array([[max(oracle.lb_piecewise(db[c], qs[q], w, p, 8), oracle.lb_piecewise(qs[q], db[c], w, p, 8))
                    for c in range(N)] for q in range(Q)])
    assert np.all(ps <= op * (1 + 1e-7) + 1e-30), "outward rounding violated"
    close(ps, op, 1e-5, max(1e-5, paa_abs_tol(p, qs, db)))
    assert ps[3, 5] == 0.0
    d = dtw_band(dev(np.repeat(db[:16], 1, 0)), dev(np.repeat(qs[:1], 16, 0)), w, p).cpu().numpy()
    assert np.all(ps[0, :16] <= d * (1 + 1e-5) + 1e-6)


def test_lb_piecewise_golden(cuda_ok):
    from paper_0811_3301_b200 import lb_piecewise
    x = np.array([[2, 3, 0, 0, 5, 0, 0, 0, 0]], np.float32)
    y = np.array([[3, 2, 3, 4, 1, 1, 1, 1, 1]], np.float32)
    for p in (1, 2):
        got = lb_piecewise(_env_dev(y, 1), dev(x), p).item() ** p
        assert got == pytest.approx(oracle.lb_piecewise(x[0], y[0], 1, p, 8) ** p, rel=1e-6)


@pytest.mark.parametrize("n,w", [(1, 0), (2, 1), (3, 2), (4, 1), (7, 3), (128, 12), (256, 25), (257, 25),
                                 (256, 8), (256, 17), (200, 40), (512, 51), (1000, 50), (300, 64), (128, 100),
                                 (64, 200), (33, 0)])
@pytest.mark.parametrize("p", [1, 2])
def test_dtw_band(cuda_ok, n, w, p):
    from paper_0811_3301_b200 import dtw_band
    count = 150 if n <= 512 else 40
    x, y = series(count, n), series(count, n)
    x[0] = y[0]
    out = dtw_band(dev(x), dev(y), w, p).cpu().numpy()
    ref = np.array([oracle.dtw(x[r], y[r], w, p) for r in range(count)])
    close(out, ref, 1e-4, 1e-6)
    assert out[0] == 0.0


def test_dtw_band_paper_values(cuda_ok):
    """P:257-258 and P:1018-1019 worked values through the GPU."""
    from paper_0811_3301_b200 import dtw_band
    x = dev([[0, 0, 1, 0], [0, 0, 1, 0]])
    y = dev([[2, 3, 2, 2], [2, 3, 2, 2]])
    assert dtw_band(x, y, 3, 2).cpu().numpy().tolist() == pytest.approx([17 ** 0.5] * 2, rel=1e-6)
    assert dtw_band(x, y, 0, 2).cpu().numpy().tolist() == pytest.approx([18 ** 0.5] * 2, rel=1e-6)
    x = dev([[0, 1, 2]])
    y = dev([[1, 2, 3]])
    assert dtw_band(x, y, 1, 1).item() == pytest.approx(2.0)
    assert dtw_band(x, y, 0, 1).item() == pytest.approx(3.0)


# wide bands (w > 64, dtw_wide.cu): band coordinates (w = 100, 101: four lanes x S = 51 cells),
# column coordinates for unconstrained DTW (w >= n - 1, n <= 256: S = 25/32/48/64 columns per
# lane, ragged last lane), and the generic fallback (w = 150)
WIDE_CASES = [(102, 100), (150, 100), (333, 101), (1000, 100), (66, 65), (100, 99), (101, 150), (128, 127),
              (129, 128), (192, 191), (200, 199), (256, 255), (400, 150)]


@pytest.mark.parametrize("n,w", WIDE_CASES)
@pytest.mark.parametrize("p", [0, 1, 2])
def test_dtw_band_wide(cuda_ok, n, w, p):
    from paper_0811_3301_b200 import dtw_band
    count = 300 if n <= 256 else 60  # > one warp's 8 pairs x several chunks of 32 pairs
    x, y = series(count, n), series(count, n)
    x[0] = y[0]
    x[1] = y[1] + 5.0
    out = dtw_band(dev(x), dev(y), w, p).cpu().numpy()
    ref = np.array([oracle.dtw(x[r], y[r], w, p) for r in range(count)])
    if p == 0:  # DTW_inf: only |x_i - y_j| rounds, exactly once
        assert np.array_equal(out, ref.astype(np.float32))
    else:
        close(out, ref, 1e-4, 1e-6)
    assert out[0] == 0.0


@pytest.mark.parametrize("n,w", [(1, 0), (4, 3), (9, 2), (128, 12), (256, 25), (257, 25), (512, 51), (300, 64),
                                 (100, 99), (1000, 50)])
def test_dtw_band_inf(cuda_ok, n, w):
    """DTW_inf (p = 0 encodes p = infinity): a max of |x_i - y_j| along the best
    path; the GPU rounds only |x_i - y_j| (exactly once), so it equals the fp64 oracle
    rounded to fp32 bit for bit."""
    from paper_0811_3301_b200 import dtw_band
    count = 60
    x, y = series(count, n), series(count, n)
    x[0] = y[0]
    out = dtw_band(dev(x), dev(y), w, 0).cpu().numpy()
    ref = np.array([oracle.dtw(x[r], y[r], w, 0) for r in range(count)]).astype(np.float32)
    assert np.array_equal(out, ref)
    assert out[0] == 0.0


def test_dtw_inf_paper_values(cuda_ok):
    """P:983-984 (Appendix A): z = (7,7,7,0), y = (7,0,5,0), x = (7,0,1,0):
    DTW_inf(z, y) = 5 and DTW_inf(z, x) = 1 (w >= 2)."""
    from paper_0811_3301_b200 import dtw_band
    z = dev([[7, 7, 7, 0], [7, 7, 7, 0]])
    yx = dev([[7, 0, 5, 0], [7, 0, 1, 0]])
    assert dtw_band(z, yx, 3, 0).cpu().numpy().tolist() == [5.0, 1.0]


def test_bounds_strict_fixture(cuda_ok):
    """x=(4,0,3,2), y=(3,4,1,4), w=1: LB_Keogh^p 1, LB_Improved^p 2, DTW^p 5 (p=1) / 7 (p=2)."""
    from paper_0811_3301_b200 import dtw_band, lb_improved, lb_keogh
    x = np.array([[4, 0, 3, 2]], np.float32)
    y = np.array([[3, 4, 1, 4]], np.float32)
    env = _env_dev(y, 1)
    for p, d in ((1, 5.0), (2, 7.0)):
        assert lb_keogh(env, dev(x), p).item() ** p == pytest.approx(1.0)
        assert lb_improved(dev(y), env, dev(x), 1, p).item() ** p == pytest.approx(2.0)
        assert dtw_band(dev(x), dev(y), 1, p).item() ** p == pytest.approx(d)


def test_error_model_on_gpu(cuda_ok):
    from paper_0811_3301_b200 import DtwlbError, dtw_band, lb_keogh
    with pytest.raises(DtwlbError) as e:
        dtw_band(dev(np.zeros((2, 4))), dev(np.zeros((2, 4))), 1, 3)
    assert e.value.name == "EUNSUPPORTED"
    with pytest.raises(DtwlbError) as e:
        dtw_band(dev(np.zeros((2, 4))), dev(np.zeros((2, 4))), -1, 1)
    assert e.value.name == "EINVAL"


@pytest.mark.parametrize("n,w", [(4, 1), (128, 12), (256, 25), (300, 64), (150, 100), (100, 99), (400, 150)])
def test_dtw_band_p4(cuda_ok, n, w):
    """DTW_4 (Appendix C compares DTW_1, DTW_2, DTW_4 and DTW_inf) through dtw_band:
    the register-band kernel (w <= 64), the four-lanes-per-pair kernels (w = 100; unconstrained
    n = 100) and the generic one (w = 150) against the fp64 oracle (generic p)."""
    from paper_0811_3301_b200 import dtw_band
    count = 120
    x, y = series(count, n), series(count, n)
    x[0] = y[0]
    out = dtw_band(dev(x), dev(y), w, 4).cpu().numpy()
    ref = np.array([oracle.dtw(x[r], y[r], w, 4) for r in range(count)])
    close(out, ref, 1e-4, 1e-6)
    assert out[0] == 0.0


def test_dtw_band_wide_eight_lanes(cuda_ok):
    """The eight-lanes-per-pair variant of the wide kernel (DTWLB_WIDE_KW=8, read once per
    process -> a subprocess): band (w = 100) and column (w = n - 1) coordinates, p = 1, 2,
    against the oracle."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, %r)\n"
        "import oracle\n"
        "from paper_0811_3301_b200 import dtw_band\n"
        "rng = np.random.default_rng(11)\n"
        "for n, w in ((150, 100), (333, 101), (100, 99), (128, 127), (256, 255)):\n"
        "    for p in (1, 2):\n"
        "        x = np.cumsum(rng.standard_normal((70, n)), axis=1).astype(np.float32)\n"
        "        y = np.cumsum(rng.standard_normal((70, n)), axis=1).astype(np.float32)\n"
        "        out = dtw_band(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), w, p).cpu().numpy()\n"
        "        ref = np.array([oracle.dtw(x[r], y[r], w, p) for r in range(70)])\n"
        "        assert np.allclose(out, ref, rtol=1e-4, atol=1e-6), (n, w, p)\n"
        "print('ok')\n") % root
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, DTWLB_WIDE_KW="8"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
