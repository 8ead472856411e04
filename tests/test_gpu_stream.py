"""Few-query streaming mode (SURVEY 8(d) "C5-stream", Q <= 8): the LB_Keogh pass runs as one
streaming pass over the database (stream.cu, TMA bulk copies).  Parity of the streaming
kernel (through the lb_keogh C-ABI call) against the fp64 oracle, of nn_search
in stream mode against the oracle's Alg. 3 scan / brute force, and bit-identity with the
tiled path (DTWLB_NO_STREAM) and with a caller-provided database index (nn_opts.db_env)."""
import os

import numpy as np
import pytest
import torch

import datagen
import oracle
from knn_compare import assert_knn_match

pytestmark = pytest.mark.gpu
THREADS = max(1, os.cpu_count() or 1)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _env(qs, w):
    from paper_0811_3301_b200 import lb_envelope
    U, L = lb_envelope(dev(qs), w)
    return torch.stack([U, L]).contiguous()


@pytest.mark.parametrize("n,w,N", [(4, 1, 300), (128, 12, 40_000), (256, 25, 1_000), (1000, 50, 300),
                                   (96, 100, 777)])
@pytest.mark.parametrize("Q", [1, 3, 4, 6, 8])
@pytest.mark.parametrize("p", [1, 2])
def test_stream_lb_keogh_vs_oracle(cuda_ok, n, w, N, Q, p):
    """N = 40 000 rows of n = 128: 157 tiles of 256 rows over 148 persistent CTAs (several tiles
    per CTA, a ragged last tile); n = 1000: a partial last 32-float chunk; n = 4: one chunk."""
    from paper_0811_3301_b200 import lb_keogh
    rng = np.random.default_rng(n * 10 + Q + p)
    qs = np.cumsum(rng.standard_normal((Q, n)), axis=1).astype(np.float32)
    db = np.cumsum(rng.standard_normal((N, n)), axis=1).astype(np.float32)
    db[N // 2] = qs[0]  # identical row: bound 0
    got = lb_keogh(_env(qs, w), dev(db), p).cpu().numpy()
    rows = np.arange(N) if N <= 1000 else np.r_[np.arange(600), rng.choice(N, 1400, replace=False), N - 1 - np.arange(300)]
    want = np.array([[oracle.lb_keogh(db[c], qs[q], w, p) for c in rows] for q in range(Q)])
    assert np.allclose(got[:, rows], want, rtol=1e-5, atol=1e-6)
    assert got[0, N // 2] == 0.0
    # the tiled kernel (Q = 9 > 8) on the same pairs agrees to fp32 summation order
    qs9 = np.concatenate([qs, qs[:1].repeat(9 - Q, axis=0)])
    tiled = lb_keogh(_env(qs9, w), dev(db), p).cpu().numpy()[:Q]
    assert np.allclose(got, tiled, rtol=2e-6, atol=1e-6)


@pytest.mark.parametrize("name,N", [("C5", 60_000), ("C3", 20_000), ("C4", 30_000), ("C2p1", 10_000),
                                    ("C2p2", 10_000), ("C1", 256)])
@pytest.mark.parametrize("Q", [1, 2, 5, 8])
def test_stream_nn_search(cuda_ok, name, N, Q):
    from paper_0811_3301_b200 import nn_search
    c = datagen.CONFIGS[name]
    qs, db = datagen.make(c, Q=Q, N=N)
    k = c.k
    idx, dist, st = nn_search(dev(qs), dev(db), c.w, c.p, k, return_stats=True)
    assert st["prefilter_evaluated"] == 0 and st["keogh_evaluated"] == Q * N  # stream mode ran
    idx, dist = idx.cpu().numpy(), dist.cpu().numpy()
    o_idx, o_dist, _ = oracle.nn_twopass(qs, db, c.w, c.p, k + 8, threads=THREADS)
    assert_knn_match(idx, dist, o_idx, o_dist, k)
    t_idx, t_dist = nn_search(dev(qs), dev(db), c.w, c.p, k, stream=False)
    assert np.array_equal(idx, t_idx.cpu().numpy()) and np.array_equal(dist, t_dist.cpu().numpy())


@pytest.mark.parametrize("Q", [1, 8])
def test_stream_db_index_reused(cuda_ok, Q):
    """nn_opts.db_env: the caller's database envelope (lb_envelope of the rows, same w) gives
    the same result as the envelope computed inside the call, in stream and tiled modes."""
    from paper_0811_3301_b200 import lb_envelope, nn_search
    c = datagen.CONFIGS["C5"]
    qs, db = datagen.make(c, Q=Q, N=50_000)
    db_t = dev(db)
    U, L = lb_envelope(db_t, c.w)
    env = torch.stack([U, L]).contiguous()
    for stream in (True, False):
        a = nn_search(dev(qs), db_t, c.w, c.p, c.k, stream=stream)
        b = nn_search(dev(qs), db_t, c.w, c.p, c.k, stream=stream, db_env=env)
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def test_stream_full_size_C5s8_sampled(cuda_ok):
    """The C5-stream bench workload (8 queries x the 10^6-row C5 database, n = 256, w = 25,
    p = 2, k = 10) in bench.py's launch configuration; the oracle checks 2 queries one by one
    (its Alg. 3 scan over the whole database)."""
    from paper_0811_3301_b200 import nn_search
    c = datagen.CONFIGS["C5s8"]
    qs, db = datagen.make(c)
    idx, dist = nn_search(dev(qs), dev(db), c.w, c.p, c.k)
    idx, dist = idx.cpu().numpy(), dist.cpu().numpy()
    rows = np.array([0, 7])
    o_idx, o_dist, _ = oracle.nn_twopass(qs[rows], db, c.w, c.p, c.k + 8, threads=2)
    assert_knn_match(idx[rows], dist[rows], o_idx, o_dist, c.k)
    assert np.all(np.diff(dist, axis=1) >= 0) and np.all(np.isfinite(dist))
