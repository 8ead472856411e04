"""Row a7 on one GPU: the database-sharded protocol emulated with G logical shards.

Each shard runs the CUDA ``nn_search`` on its rows with ``index_base`` = its first
row and the threshold exchange; the exchange lowers the block's thresholds to the
minimum seen over the shards so far (every shard's k-th best is >= the global k-th
best, so any such value is safe); the [G][Q][k] lists are merged by
the CUDA ``nn_merge``.  The result must be the k-NN over the whole set S
(P:501-503): equal to the oracle's brute force (tie classes, reading c14) and
bit-identical to one ``nn_search`` over the unsharded database (every pair's DTW
is computed by the same per-pair arithmetic whatever the shard).
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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def emulate(qs, db, w, p, k, bounds, query_block=8, walk=0):
    """G logical shards [bounds[g], bounds[g+1]) searched one after the other; returns the
    merged (idx, dist) from nn_merge and the number of threshold entries the exchange lowered.
    walk = nn_opts.exchange_walk: each block makes 1 + walk exchange calls (phase = call index
    within the block), each phase with its own running minimum over the shards."""
    from paper_0811_3301_b200 import nn_merge, nn_search
    Q = qs.shape[0]
    G = len(bounds) - 1
    q_t = dev(qs)
    shared = torch.full((1 + walk, Q), float("inf"), dtype=torch.float32, device="cuda")
    lowered = [0]
    g_idx = torch.empty((G, Q, k), dtype=torch.int64, device="cuda")
    g_dst = torch.empty((G, Q, k), dtype=torch.float32, device="cuda")
    for g in range(G):
        lo, hi = bounds[g], bounds[g + 1]
        kk = min(k, hi - lo)
        pos = [0] * (1 + walk)
        calls = [0]

        def exchange(thr, kk=kk, pos=pos, calls=calls):
            n = thr.numel()
            ph = calls[0] % (1 + walk)
            calls[0] += 1
            view = shared[ph, pos[ph]:pos[ph] + n]
            before = thr.clone()
            if kk == k:  # a shard with fewer than k rows contributes +inf (sharded.py)
                torch.minimum(view, thr, out=view)
            torch.minimum(thr, view, out=thr)
            lowered[0] += int((thr < before).sum().item())
            pos[ph] += n

        if kk == 0:
            g_idx[g].fill_(-1)
            g_dst[g].fill_(float("inf"))
            continue
        idx, dst = nn_search(q_t, dev(db[lo:hi]), w, p, kk, index_base=lo, query_block=query_block,
                             exchange=exchange, shards=G, exchange_walk=walk)
        assert pos == [Q] * (1 + walk)  # 1 + walk exchanges per query block, covering every query
        g_idx[g, :, :kk] = idx
        g_dst[g, :, :kk] = dst
        if kk < k:
            g_idx[g, :, kk:] = -1
            g_dst[g, :, kk:] = float("inf")
    m_idx, m_dst = nn_merge(g_idx, g_dst)
    torch.cuda.synchronize()
    return m_idx.cpu().numpy(), m_dst.cpu().numpy(), lowered[0]


@pytest.mark.parametrize("walk", [0, 3])
@pytest.mark.parametrize("G", [2, 3, 8])
@pytest.mark.parametrize("name,Q,N", [("C5", 16, 24_000), ("C2p2", 24, 10_000), ("C2p1", 12, 10_000)])
def test_sharded_emulation_equals_global(cuda_ok, G, name, Q, N, walk):
    from paper_0811_3301_b200 import nn_search
    from paper_0811_3301_b200.sharded import shard_range
    c = datagen.CONFIGS[name]
    k = c.k if name == "C5" else 3
    qs, db = datagen.make(c, Q=Q, N=N)
    bounds = [shard_range(N, G, g)[0] for g in range(G)] + [N]
    m_idx, m_dst, lowered = emulate(qs, db, c.w, c.p, k, bounds, walk=walk)
    o_idx, o_dst, _ = oracle.nn_twopass(qs, db, c.w, c.p, k + 8, threads=THREADS)
    assert_knn_match(m_idx, m_dst, o_idx, o_dst, k)
    s_idx, s_dst = nn_search(dev(qs), dev(db), c.w, c.p, k, query_block=8)
    assert np.array_equal(m_idx, s_idx.cpu().numpy())
    assert np.array_equal(m_dst, s_dst.cpu().numpy())
    assert lowered > 0  # later shards start from the earlier shards' thresholds


def test_sharded_emulation_unbalanced_and_small_shards(cuda_ok):
    """Unbalanced shards, one smaller than k and one empty; the global nearest neighbours are
    planted in the small shard (exact copies / scaled copies of the queries)."""
    c = datagen.CONFIGS["C2p2"]
    k = 5
    qs, db = datagen.make(c, Q=10, N=3000)
    db[1] = qs[0]
    db[2] = qs[3] * np.float32(0.99)
    bounds = [0, 3, 3, 1700, 3000]  # shard sizes 3 (< k), 0, 1697, 1300
    m_idx, m_dst, _ = emulate(qs, db, c.w, c.p, k, bounds, query_block=4, walk=3)
    o_idx, o_dst = oracle.nn_brute(qs, db, c.w, c.p, k + 8, threads=THREADS)
    assert_knn_match(m_idx, m_dst, o_idx, o_dst, k)
    assert m_idx[0, 0] == 1 and m_dst[0, 0] == 0.0


def test_nn_merge_against_host_merge(cuda_ok):
    """nn_merge on random shard lists (ascending per shard, padded with (-1, +inf), equal
    distances across shards) equals the host merge: k smallest by (dist, idx)."""
    from paper_0811_3301_b200 import nn_merge
    from shard_ref import merge_reference
    rng = np.random.default_rng(5)
    for G, Q, k in [(1, 3, 4), (2, 17, 10), (5, 9, 3), (8, 33, 7), (64, 2, 2)]:
        d = np.sort(rng.integers(0, 6, size=(G, Q, k)).astype(np.float32), axis=2)  # many ties
        i = np.zeros((G, Q, k), dtype=np.int64)
        for g in range(G):
            for q in range(Q):
                ids = rng.choice(1000, size=k, replace=False) + 1000 * g
                order = np.lexsort((ids, d[g, q]))
                d[g, q] = d[g, q][order]
                i[g, q] = ids[order]
                pad = rng.integers(0, k + 1)
                if pad:
                    i[g, q, k - pad:] = -1
                    d[g, q, k - pad:] = np.inf
        gi, gd = nn_merge(torch.from_numpy(i).cuda(), torch.from_numpy(d).cuda())
        ri, rd = merge_reference(torch.from_numpy(i), torch.from_numpy(d))
        assert np.array_equal(gi.cpu().numpy(), ri.numpy())
        assert np.array_equal(gd.cpu().numpy(), rd.numpy())


def test_library_nccl_exchange_single_rank(cuda_ok):
    """nn_opts.nccl_comm: the library's own NCCL communicator (dtwlb_get_unique_id /
    dtwlb_comm_init, one rank on this GPU) min-reduces the thresholds at every exchange point
    (after the first range and 3 times inside the last walk) on the call's stream; with one
    rank the reduction is the identity, so the result equals the unsharded search bit for bit."""
    from paper_0811_3301_b200 import Communicator, get_unique_id, nn_search
    c = datagen.CONFIGS["C2p2"]
    qs, db = datagen.make(c, Q=24, N=10_000)
    comm = Communicator(get_unique_id(), 1, 0)
    try:
        a_idx, a_dst = nn_search(dev(qs), dev(db), c.w, c.p, 3, query_block=8, nccl_comm=comm, shards=1,
                                 exchange_walk=3)
        torch.cuda.synchronize()
    finally:
        comm.close()
    b_idx, b_dst = nn_search(dev(qs), dev(db), c.w, c.p, 3, query_block=8)
    assert np.array_equal(a_idx.cpu().numpy(), b_idx.cpu().numpy())
    assert np.array_equal(a_dst.cpu().numpy(), b_dst.cpu().numpy())
    o_idx, o_dst = oracle.nn_brute(qs, db, c.w, c.p, 3 + 8, threads=THREADS)
    assert_knn_match(a_idx.cpu().numpy(), a_dst.cpu().numpy(), o_idx, o_dst, 3)
