"""nn_search parity against the fp64 oracle (GPU only).

Ground truth is the oracle's brute-force k-NN (or its Algorithm-3 scan, which
tests/test_oracle_search.py pins to brute force).  Comparison: tests/knn_compare.py
(tie classes at relative 1e-4, distances within relative 1e-4).
"""
import os

import numpy as np
import pytest
import torch

import datagen
import oracle
from knn_compare import assert_knn_match

pytestmark = pytest.mark.gpu
THREADS = max(1, os.cpu_count() or 1)
EXTRA = 8


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def run(qs, db, w, p, k, **kw):
    from paper_0811_3301_b200 import nn_search
    idx, dist = nn_search(dev(qs), dev(db), w, p, k, **kw)
    torch.cuda.synchronize()
    return idx.cpu().numpy(), dist.cpu().numpy()


def check(qs, db, w, p, k, brute=True, **kw):
    g_idx, g_dist = run(qs, db, w, p, k, **kw)
    ke = min(len(db), k + EXTRA)
    if brute:
        o_idx, o_dist = oracle.nn_brute(qs, db, w, p, ke, threads=THREADS)
    else:
        o_idx, o_dist, _ = oracle.nn_twopass(qs, db, w, p, ke, threads=THREADS)
    base = kw.get("index_base", 0)
    assert_knn_match(g_idx - base, g_dist, o_idx, o_dist, k)
    return g_idx, g_dist


def test_C1_full(cuda_ok):
    c = datagen.CONFIGS["C1"]
    qs, db = datagen.make(c)
    check(qs, db, c.w, c.p, c.k)


@pytest.mark.parametrize("name", ["C2p1", "C2p2"])
def test_C2_full(cuda_ok, name):
    c = datagen.CONFIGS[name]
    qs, db = datagen.make(c)
    check(qs, db, c.w, c.p, c.k, brute=False)


@pytest.mark.parametrize("prefilter", [True, False])
@pytest.mark.parametrize("name,Q,N", [("C3", 6, 20_000), ("C4", 8, 30_000), ("C5", 8, 60_000)])
def test_reduced_large_configs(cuda_ok, name, Q, N, prefilter):
    c = datagen.CONFIGS[name]
    qs, db = datagen.make(c, Q=Q, N=N)
    check(qs, db, c.w, c.p, c.k, brute=False, prefilter=prefilter)


@pytest.mark.parametrize("prefilter", [True, False])
@pytest.mark.parametrize("p", [1, 2])
@pytest.mark.parametrize("k", [1, 3, 10])
def test_duplicates_self_queries_ties(cuda_ok, p, k, prefilter):
    qs, db = datagen.make("C2p1", Q=20, N=3000)
    db[100] = qs[0]          # exact self-match -> distance 0
    db[2000] = qs[0]         # duplicate of the self-match: smaller index first
    db[7] = db[8]            # duplicate rows
    db[1500] = qs[5] + 1e-3  # near tie
    g_idx, g_dist = check(qs, db, 25, p, k, prefilter=prefilter)
    assert g_idx[0, 0] == 100 and g_dist[0, 0] == 0.0
    if k > 1:
        assert g_idx[0, 1] == 2000 and g_dist[0, 1] == 0.0


@pytest.mark.parametrize("n,w", [(7, 3), (7, 0), (50, 60), (128, 100), (130, 5), (1, 0), (300, 64), (96, 33)])
def test_odd_shapes_and_bands(cuda_ok, n, w):
    if n == 1:  # a length-1 random walk is the constant 0: use white noise instead
        g = np.random.default_rng(5)
        qs = g.standard_normal((9, 1)).astype(np.float32)
        db = g.standard_normal((700, 1)).astype(np.float32)
    else:
        qs = datagen.random_walks(9, n, seed=3, role=1)
        db = datagen.random_walks(700, n, seed=4)
    for p in (1, 2):
        check(qs, db, w, p, 2)
        check(qs, db, w, p, 2, prefilter=False)


def test_all_tied_database_returns_smallest_indices(cuda_ok):
    """Every candidate at distance 0: ties break to the smallest index (reading c4)."""
    qs = np.zeros((4, 16), np.float32)
    db = np.zeros((500, 16), np.float32)
    for p in (1, 2):
        for pf in (True, False):
            idx, dist = run(qs, db, 3, p, 7, prefilter=pf)
            assert np.all(idx == np.arange(7)) and np.all(dist == 0)


def test_k_equals_N_and_small_N(cuda_ok):
    qs, db = datagen.make("C1", Q=3, N=40)
    check(qs, db, 12, 1, 40)     # full sorted order
    check(qs, db, 12, 2, 1)
    check(qs, db[:1], 12, 1, 1)  # N = 1


def test_keogh_only_index_base_eps0(cuda_ok):
    qs, db = datagen.make("C2p2", Q=16, N=5000)
    check(qs, db, 25, 2, 5, keogh_only=True)
    check(qs, db, 25, 2, 5, keogh_only=True, prefilter=False)
    check(qs, db, 25, 1, 3, prefilter=False, query_block=5)
    check(qs, db, 25, 2, 5, index_base=1_000_000)
    check(qs, db, 25, 2, 5, eps=0.0)
    check(qs, db, 25, 2, 5, query_block=4)   # several query blocks


@pytest.mark.parametrize("name", ["C2p1", "C2p2"])
def test_cascade_and_prefilter_switches(cuda_ok, name):
    """Every combination of the pre-filter and the DTW cascading abandon
    (reading c19) returns the same exact k-NN; only the work done differs."""
    from paper_0811_3301_b200 import nn_search
    c = datagen.CONFIGS[name]
    qs, db = datagen.make(c, Q=24, N=6000)
    ref = None
    for pf in (True, False):
        for cas in (True, False):
            g_idx, g_dist = check(qs, db, c.w, c.p, 4, brute=False, prefilter=pf, cascade=cas)
            if ref is None:
                ref = (g_idx, g_dist)
            else:  # bit-identical across modes: DTW values do not depend on the pruning path
                assert np.array_equal(ref[0], g_idx) and np.array_equal(ref[1], g_dist)
    _, _, st = nn_search(dev(qs), dev(db), c.w, c.p, 4, return_stats=True)
    assert st["prefilter_evaluated"] == 24 * 6000 and st["prefilter_segment"] == 8
    assert st["dtw_evaluated"] <= st["improved_evaluated"] <= st["keogh_evaluated"] <= 24 * 6000


@pytest.mark.parametrize("name,w", [("C2p2", None), ("C2p1", None), ("C2p2", 100)])
def test_no_abandon_same_knn(cuda_ok, name, w):
    """DTWLB_NO_ABANDON: without early abandoning every DTW the bounds pass runs to
    its last row -- the k-NN is bit-identical (abandoning only skips pairs that cannot enter the
    top-k, reading c15), no pair is abandoned, and every started pair's cells are all computed.
    Covers the register-band kernel and (w = 100) the four-lanes-per-pair wide kernel."""
    from paper_0811_3301_b200 import nn_search
    c = datagen.CONFIGS[name]
    qs, db = datagen.make(c, Q=16, N=3000)
    w = c.w if w is None else w
    g_idx, g_dist = check(qs, db, w, c.p, 3, brute=False)
    i2, d2, st = nn_search(dev(qs), dev(db), w, c.p, 3, abandon=False, return_stats=True)
    assert np.array_equal(i2.cpu().numpy(), g_idx) and np.array_equal(d2.cpu().numpy(), g_dist)
    assert st["dtw_abandoned"] == 0
    assert st["dtw_cells_computed"] == st["dtw_cells_nominal"] > 0
    _, _, st1 = nn_search(dev(qs), dev(db), w, c.p, 3, return_stats=True)
    assert st1["dtw_cells_computed"] < st["dtw_cells_computed"]


def test_threshold_exchange_callback(cuda_ok):
    """The sharded path's exchange hook (a7): called once per query block after the first
    range with a CUDA view of the block's thresholds; lowering them to any value >= the
    true k-th best (here: the global k-th best from the oracle, times 1+eps) keeps the
    result exact, and an identity exchange changes nothing."""
    from paper_0811_3301_b200 import nn_search
    c = datagen.CONFIGS["C2p2"]
    qs, db = datagen.make(c, Q=20, N=5000)
    o_idx, o_dist, _ = oracle.nn_twopass(qs, db, c.w, c.p, 3 + EXTRA, threads=THREADS)
    calls = []

    def ident(thr):
        calls.append(thr.numel())

    a_idx, a_dist = nn_search(dev(qs), dev(db), c.w, c.p, 3, query_block=8, exchange=ident)
    assert calls == [8, 8, 4]
    tau = torch.tensor(o_dist[:, 2].astype(np.float64) ** c.p * (1 + 1e-3), dtype=torch.float32).cuda()
    pos = [0]

    def lower(thr):
        n = thr.numel()
        torch.minimum(thr, tau[pos[0]:pos[0] + n], out=thr)
        pos[0] += n

    b_idx, b_dist = nn_search(dev(qs), dev(db), c.w, c.p, 3, query_block=8, exchange=lower)
    assert pos[0] == 20
    assert_knn_match(a_idx.cpu().numpy(), a_dist.cpu().numpy(), o_idx, o_dist, 3)
    assert np.array_equal(a_idx.cpu().numpy(), b_idx.cpu().numpy())
    assert np.array_equal(a_dist.cpu().numpy(), b_dist.cpu().numpy())


def test_host_buffers(cuda_ok):
    """e2e path: host (numpy) inputs and outputs through the same C-ABI call."""
    from paper_0811_3301_b200 import nn_search
    qs, db = datagen.make("C2p1", Q=10, N=4000)
    h_idx, h_dist = nn_search(qs, db, 25, 1, 3)
    assert not h_idx.is_cuda
    d_idx, d_dist = run(qs, db, 25, 1, 3)
    assert np.array_equal(h_idx.numpy(), d_idx) and np.array_equal(h_dist.numpy(), d_dist)


def test_empty_query_set(cuda_ok):
    from paper_0811_3301_b200 import nn_search
    idx, dist = nn_search(dev(np.zeros((0, 16))), dev(np.zeros((5, 16))), 2, 1, 1)
    assert idx.shape == (0, 1)


def test_deterministic_repeat(cuda_ok):
    qs, db = datagen.make("C2p2", Q=32, N=8000)
    a = run(qs, db, 25, 2, 10)
    b = run(qs, db, 25, 2, 10)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("name,sample", [("C5", 3), ("C3", 3), ("C4", 3)])
def test_full_size_sampled(cuda_ok, name, sample):
    """Full BASELINE size in bench.py's launch configuration; the oracle checks a
    sample of queries one by one (its Algorithm-3 scan over the whole database)."""
    from paper_0811_3301_b200 import nn_search
    c = datagen.CONFIGS[name]
    qs, db = datagen.make(c)
    idx, dist = nn_search(dev(qs), dev(db), c.w, c.p, c.k)
    idx, dist = idx.cpu().numpy(), dist.cpu().numpy()
    rows = np.linspace(0, c.Q - 1, sample).astype(int)
    o_idx, o_dist, _ = oracle.nn_twopass(qs[rows], db, c.w, c.p, c.k + EXTRA, threads=THREADS)
    assert_knn_match(idx[rows], dist[rows], o_idx, o_dist, c.k)
    # properties at any size: ascending, finite, distinct, in range
    assert np.all(np.diff(dist, axis=1) >= 0) and np.all(np.isfinite(dist))
    assert idx.min() >= 0 and idx.max() < c.N


def test_output_aliasing_rejected(cuda_ok):
    """nn_search rejects outputs that overlap an input or each other (EINVAL, include/dtwlb.h)."""
    from paper_0811_3301_b200 import DtwlbError, nn_search
    qs, db = datagen.make("C2p1", Q=4, N=500)
    q_t, db_t = dev(qs), dev(db)
    idx = torch.empty((4, 2), dtype=torch.int64, device="cuda")
    dst = torch.empty((4, 2), dtype=torch.float32, device="cuda")
    with pytest.raises(DtwlbError, match="EINVAL"):
        nn_search(q_t, db_t, 25, 1, 2, out=(idx, q_t[0, :8]))            # dist over the queries
    with pytest.raises(DtwlbError, match="EINVAL"):
        nn_search(q_t, db_t, 25, 1, 2, out=(db_t.view(torch.int64)[:4, :2], dst))  # idx over the db
    buf = torch.empty(64, dtype=torch.int64, device="cuda")
    with pytest.raises(DtwlbError, match="EINVAL"):
        nn_search(q_t, db_t, 25, 1, 2, out=(buf[:8].view(4, 2), buf.view(torch.float32)[4:12].view(4, 2)))
    i2, d2 = nn_search(q_t, db_t, 25, 1, 2, out=(idx, dst))  # disjoint: fine
    assert i2.data_ptr() == idx.data_ptr()


@pytest.mark.parametrize("name,Q,N,w", [("C3", 12, 8000, 100), ("C3", 3, 8000, 101), ("C2p1", 40, 4000, 255),
                                        ("C2p2", 20, 4000, 300), ("C3", 6, 5000, 150)])
def test_wide_band_walk(cuda_ok, name, Q, N, w):
    """w > 64 through nn_search: the four-lanes-per-pair band kernel (w = 100, 101), the column
    kernel for unconstrained DTW (C2 n = 256 with w >= n - 1), and the generic kernel (w = 150);
    exact early abandon against the walk's thresholds, results equal to the oracle."""
    c = datagen.CONFIGS[name]
    qs, db = datagen.make(c, Q=Q, N=N)
    k = 3
    g_idx, g_dist = run(qs, db, w, c.p, k)
    o_idx, o_dist, _ = oracle.nn_twopass(qs, db, w, c.p, k + EXTRA, threads=THREADS)
    assert_knn_match(g_idx, g_dist, o_idx, o_dist, k)


@pytest.mark.parametrize("name", ["C5", "C3", "C4"])
def test_full_size_oracle_cache(cuda_ok, name):
    """Full BASELINE size, bench.py's launch configuration, against the oracle-result cache
    (tests/golden/oracle_knn_<cfg>.npz, written by scripts/oracle_cache.py from oracle/ only:
    Alg. 3 fp64 scan, 256 sampled queries); two cached queries are re-verified live."""
    from paper_0811_3301_b200 import nn_search
    path = os.path.join(os.path.dirname(__file__), "golden", f"oracle_knn_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"no oracle cache for {name} (python scripts/oracle_cache.py {name})")
    g = np.load(path)
    c = datagen.CONFIGS[name]
    assert (int(g["Q"]), int(g["N"]), int(g["n"]), int(g["w"]), int(g["p"]), int(g["seed"])) == \
        (c.Q, c.N, c.n, c.w, c.p, c.seed), "stale cache: config changed"
    qs, db = datagen.make(c)
    rows = g["rows"]
    live = rows[[1, len(rows) // 2]]  # re-verify a subset of the cache against the oracle itself
    l_idx, l_dist, _ = oracle.nn_twopass(qs[live], db, c.w, c.p, int(g["k"]), threads=THREADS)
    pos = [int(np.searchsorted(rows, r)) for r in live]
    assert np.array_equal(l_idx, g["idx"][pos]) and np.array_equal(l_dist, g["dist"][pos])
    idx, dist = nn_search(dev(qs), dev(db), c.w, c.p, c.k)
    idx, dist = idx.cpu().numpy(), dist.cpu().numpy()
    assert_knn_match(idx[rows], dist[rows], g["idx"], g["dist"], c.k)


def test_key_list_pool_redo(cuda_ok):
    """Exact-count key lists: a range whose lists exceed the pool (DTWLB_LIST_POOL_MAX, read once
    per process -> a subprocess) makes nn_search redo the query block as two half blocks, down to
    blocks that fit; the result is unchanged."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import datagen, oracle\n"
        "from knn_compare import assert_knn_match\n"
        "from paper_0811_3301_b200 import nn_search\n"
        "qs, db = datagen.make('C2p2', Q=40, N=6000)\n"
        "idx, dist = nn_search(torch.from_numpy(qs).cuda(), torch.from_numpy(db).cuda(), 25, 2, 5, query_block=40)\n"
        "o_idx, o_dist = oracle.nn_brute(qs, db, 25, 2, 13, threads=8)\n"
        "assert_knn_match(idx.cpu().numpy(), dist.cpu().numpy(), o_idx, o_dist, 5)\n"
        "print('ok')\n") % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.dirname(__file__))
    env = dict(os.environ, DTWLB_LIST_POOL_MAX="3000")  # ~40 queries x 6000 x a few % survive per range
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


@pytest.mark.parametrize("n,w,p", [(1100, 40, 2), (1500, 150, 1)])
def test_long_series_beyond_survivor_kernel(cuda_ok, n, w, p):
    """n > 1024 (beyond the survivor kernel's 32 samples per lane): nn_search runs Alg. 2
    (LB_Keogh over every pair, then the DTW walk; any n must work) and lb_improved
    the warp-per-pair kernel; both against the oracle."""
    from paper_0811_3301_b200 import lb_envelope, lb_improved
    rng = np.random.default_rng(n + w)
    qs = np.cumsum(rng.standard_normal((5, n)), axis=1).astype(np.float32)
    db = np.cumsum(rng.standard_normal((700, n)), axis=1).astype(np.float32)
    db[123] = qs[2] + np.float32(0.01)
    check(qs, db, w, p, 3)
    U, L = lb_envelope(dev(qs), w)
    env = torch.stack([U, L]).contiguous()
    got = lb_improved(dev(qs), env, dev(db[:40]), w, p).cpu().numpy()
    want = np.array([[oracle.lb_improved(db[c], qs[q], w, p) for c in range(40)] for q in range(5)])
    assert np.allclose(got, want, rtol=1e-5, atol=1e-6)
