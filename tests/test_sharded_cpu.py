"""World-size-2 `gloo` tests of the database-sharded protocol on CPU.

The per-shard search is the oracle's brute force (CPU stand-in for the CUDA
`nn_search`, which needs a GPU); the exchange (all-gather of [Q][k] lists with
global indices) and the merge are the product's `sharded.py` code.  The result
must equal the oracle's k-NN over the whole database.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen
import oracle
from paper_0811_3301_b200.sharded import EXCHANGE_WALK


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_search(queries, db, w, p, k, index_base=0, out=None, **_):
    idx, dst = oracle.nn_brute(queries.numpy(), db.numpy(), w, p, k)
    return torch.from_numpy(idx + index_base), torch.from_numpy(dst.astype(np.float32))


def _cascade_search(queries, db, w, p, k, index_base=0, out=None, query_block=None, exchange=None, shards=0,
                    exchange_walk=0):
    """CPU stand-in of nn_search's two-range protocol built from oracle primitives: per
    query block, range 1 = the S candidates with the smallest LB_Keogh (exact DTW, local
    top-k, tau); exchange(tau) may lower tau; range 2 = the other candidates whose
    LB_Keogh <= tau (1+eps) with tau tightening as results arrive, walked in 1 + exchange_walk
    parts with an exchange after each of the first exchange_walk parts (nn_opts.exchange_walk)."""
    qs, dbn = queries.numpy().astype(np.float64), db.numpy().astype(np.float64)
    Q, N = qs.shape[0], dbn.shape[0]
    eps = 1e-3
    qb = query_block or Q
    idx = np.full((Q, k), -1, dtype=np.int64)
    dst = np.full((Q, k), np.inf)
    for b0 in range(0, Q, qb):
        rows = range(b0, min(Q, b0 + qb))
        lbs = {q: np.array([oracle.lb_keogh(dbn[c], qs[q], w, p) ** p for c in range(N)]) for q in rows}
        tops = {q: [] for q in rows}
        thr = torch.full((len(rows),), float("inf"), dtype=torch.float32)
        S = max(k, N // 4)

        def visit(q, cands):
            for c in cands:
                if lbs[q][c] > thr[q - b0].item() * (1 + 1e-6):
                    continue
                d = oracle.dtw_pow(dbn[c], qs[q], w, p)
                tops[q] = sorted(tops[q] + [(d, c)])[:k]
                if len(tops[q]) == k:
                    thr[q - b0] = min(thr[q - b0].item(), tops[q][-1][0] * (1 + eps))

        for q in rows:
            visit(q, np.argsort(lbs[q], kind="stable")[:S])
        if exchange is not None:
            exchange(thr)
        parts = 1 + (exchange_walk if exchange is not None else 0)
        rest = {q: np.argsort(lbs[q], kind="stable")[S:] for q in rows}
        for part in range(parts):
            for q in rows:
                r2 = rest[q]
                visit(q, r2[part * len(r2) // parts:(part + 1) * len(r2) // parts])
            if part + 1 < parts:
                exchange(thr)
        for q in rows:
            for r, (d, c) in enumerate(tops[q]):
                idx[q, r] = c + index_base
                dst[q, r] = d ** (1.0 / p)
    return torch.from_numpy(idx), torch.from_numpy(dst.astype(np.float32))


def _worker_exchange(rank, world, port, N, k, result_q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_0811_3301_b200.sharded import shard_range, sharded_nn_search
        from shard_ref import merge_reference
        cfg = datagen.CONFIGS["C2p2"]
        lo, hi = shard_range(N, world, rank)
        qs, _ = datagen.make(cfg, Q=4, N=0)
        qs = qs[:, :32].copy()
        shard = datagen.series(cfg.family, hi - lo, cfg.n, cfg.seed, datagen.ROLE_DB, cfg.znorm, start=lo)[:, :32]
        shard = np.ascontiguousarray(shard)
        seen = []

        def search(queries, db, w, p, kk, index_base=0, out=None, query_block=None, exchange=None, shards=0,
                   exchange_walk=0):
            # every shard is told the shard count (its best-first seed range is 1/world of the whole)
            assert shards == world, (shards, world)

            def ex(t):
                before = t.clone()
                exchange(t)
                seen.append((before.numpy().copy(), t.numpy().copy()))
            return _cascade_search(queries, db, w, p, kk, index_base, out, query_block, ex, exchange_walk=exchange_walk)

        idx, dst = sharded_nn_search(torch.from_numpy(qs), torch.from_numpy(shard), lo, 3, cfg.p, k,
                                     search=search, merge=merge_reference, query_block=3)
        result_q.put((rank, idx.numpy(), dst.numpy(), seen))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:
        result_q.put((rank, None, repr(e), None))
        raise


def test_threshold_exchange_is_exact_and_tightens():
    """After the first range each block's thresholds are min-reduced over the shards
    (SURVEY 8(e) item 1); the merged result still equals the brute-force k-NN of the
    whole database, and the exchange lowers at least one shard's thresholds."""
    world, N, k = 2, 120, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_exchange, args=(r, world, port, N, k, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort(key=lambda r: r[0])
    for r in res:
        assert r[1] is not None, r[2]
    cfg = datagen.CONFIGS["C2p2"]
    qs, db = datagen.make(cfg, Q=4, N=N)
    o_idx, o_dst = oracle.nn_brute(np.ascontiguousarray(qs[:, :32]), np.ascontiguousarray(db[:, :32]), 3, cfg.p, k)
    for rank, idx, dst, seen in res:
        assert np.array_equal(idx, o_idx)
        assert np.allclose(dst, o_dst, rtol=1e-6)
        # blocks of 3 queries: 4 queries -> 2 blocks x (1 + EXCHANGE_WALK) exchanges on every rank
        assert len(seen) == 2 * (1 + EXCHANGE_WALK)
        for before, after in seen:
            assert np.all(after <= before)
    lowered = sum(int(np.any(a < b)) for _, _, _, seen in res for b, a in seen)
    assert lowered >= 1


def _worker(rank, world, port, N, k, result_q):
    try:
        _worker_body(rank, world, port, N, k, result_q)
    except Exception as e:  # report instead of hanging the parent
        result_q.put((rank, None, repr(e), None))
        raise


def _worker_body(rank, world, port, N, k, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_0811_3301_b200.sharded import shard_range, sharded_nn_search
    from shard_ref import merge_reference
    cfg = datagen.CONFIGS["C2p2"]
    lo, hi = shard_range(N, world, rank)
    qs, _ = datagen.make(cfg, Q=5, N=0)
    shard = datagen.series(cfg.family, hi - lo, cfg.n, cfg.seed, datagen.ROLE_DB, cfg.znorm, start=lo)
    if rank == 1:
        shard[3] = qs[2]  # an exact match living on the second shard (global index lo+3)
    idx, dst = sharded_nn_search(torch.from_numpy(qs), torch.from_numpy(shard), lo, cfg.w, cfg.p, k,
                                 search=_oracle_search, merge=merge_reference)
    result_q.put((rank, idx.numpy(), dst.numpy(), lo))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("N,k", [(301, 3), (7, 5), (40, 10)])
def test_sharded_equals_global(N, k):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, k, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort(key=lambda r: r[0])
    for r in res:
        assert r[1] is not None, r[2]
    cfg = datagen.CONFIGS["C2p2"]
    qs, db = datagen.make(cfg, Q=5, N=N)
    lo1 = res[1][3]
    db[lo1 + 3] = qs[2]
    o_idx, o_dst = oracle.nn_brute(qs, db, cfg.w, cfg.p, min(k, N))
    for rank, idx, dst, _ in res:
        assert np.array_equal(idx[:, :min(k, N)], o_idx)          # identical on every rank
        assert np.allclose(dst[:, :min(k, N)], o_dst, rtol=1e-6)
    assert res[0][1][2, 0] == lo1 + 3 and res[0][2][2, 0] == 0.0


def test_shard_ranges_partition():
    from paper_0811_3301_b200.sharded import shard_range
    for N in (1, 7, 1000, 1_000_000):
        for G in (1, 2, 3, 4, 8):
            r = [shard_range(N, G, i) for i in range(G)]
            assert r[0][0] == 0 and r[-1][1] == N
            assert all(r[i][1] == r[i + 1][0] for i in range(G - 1))
            sizes = [b - a for a, b in r]
            assert max(sizes) - min(sizes) <= 1


def _worker_unbalanced(rank, world, port, bounds, k, result_q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_0811_3301_b200.sharded import sharded_nn_search
        from shard_ref import merge_reference
        cfg = datagen.CONFIGS["C2p2"]
        lo, hi = bounds[rank], bounds[rank + 1]
        qs, _ = datagen.make(cfg, Q=4, N=0)
        qs = np.ascontiguousarray(qs[:, :32])
        shard = np.ascontiguousarray(
            datagen.series(cfg.family, hi - lo, cfg.n, cfg.seed, datagen.ROLE_DB, cfg.znorm, start=lo)[:, :32])
        if rank == 0:  # rank 0's two rows are query 0's nearest: its 2nd best is far below the global 5th
            shard[0] = qs[0]
            shard[1] = qs[0] * np.float32(0.999)
        sent = []

        def search(queries, db, w, p, kk, index_base=0, out=None, query_block=None, exchange=None, shards=0,
                   exchange_walk=0):
            def ex(t):
                exchange(t)
                sent.append(t.numpy().copy())
            return _cascade_search(queries, db, w, p, kk, index_base, out, query_block, ex, exchange_walk=exchange_walk)

        idx, dst = sharded_nn_search(torch.from_numpy(qs), torch.from_numpy(shard), lo, 3, cfg.p, k,
                                     search=search, merge=merge_reference, query_block=4)
        result_q.put((rank, idx.numpy(), dst.numpy(), sent))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:
        result_q.put((rank, None, repr(e), None))
        raise


def test_unbalanced_shard_smaller_than_k():
    """a shard with fewer than k rows must not contribute its own kk-th best to the
    threshold exchange (it is no upper bound on the global k-th best).  Rank 0 holds 2 rows,
    rank 1 holds 38, k = 5: every rank must still return the brute-force k-NN of all 40 rows,
    and the threshold rank 1 receives is its own k-th best (rank 0 sends +inf)."""
    world, k = 2, 5
    bounds = [0, 2, 40]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_unbalanced, args=(r, world, port, bounds, k, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort(key=lambda r: r[0])
    for r in res:
        assert r[1] is not None, r[2]
    cfg = datagen.CONFIGS["C2p2"]
    qs, db = datagen.make(cfg, Q=4, N=40)
    qs, db = np.ascontiguousarray(qs[:, :32]), np.ascontiguousarray(db[:, :32])
    db[0] = qs[0]
    db[1] = qs[0] * np.float32(0.999)
    o_idx, o_dst = oracle.nn_brute(qs, db, 3, cfg.p, k)
    for rank, idx, dst, sent in res:
        assert np.array_equal(idx, o_idx)
        assert np.allclose(dst, o_dst, rtol=1e-6)
    # rank 1's thresholds after the exchange are bounded below by the global k-th best
    kth = (o_dst[:, k - 1].astype(np.float64) ** cfg.p)
    for t in res[1][3]:
        assert np.all(t >= kth * (1 - 1e-6))


def _worker_qshard(rank, world, port, Q, N, k, result_q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_0811_3301_b200.sharded import query_sharded_nn_search
        cfg = datagen.CONFIGS["C2p1"]
        qs, db = datagen.make(cfg, Q=Q, N=N)
        calls = []

        def search(queries, dbt, w, p, kk, **kw):
            calls.append(queries.shape[0])
            return _oracle_search(queries, dbt, w, p, kk)

        idx, dst = query_sharded_nn_search(torch.from_numpy(qs), torch.from_numpy(db), cfg.w, cfg.p, k,
                                           search=search)
        result_q.put((rank, idx.numpy(), dst.numpy(), calls))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:
        result_q.put((rank, None, repr(e), None))
        raise


@pytest.mark.parametrize("Q", [7, 2])
def test_query_sharded_equals_global(Q):
    """Query-sharded comparison mode: replicated database, queries split over the
    ranks (7 = 3 + 4; 2 = 1 + 1), results all-gathered: every rank returns the brute-force k-NN."""
    world, N, k = 2, 150, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_qshard, args=(r, world, port, Q, N, k, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort(key=lambda r: r[0])
    for r in res:
        assert r[1] is not None, r[2]
    cfg = datagen.CONFIGS["C2p1"]
    qs, db = datagen.make(cfg, Q=Q, N=N)
    o_idx, o_dst = oracle.nn_brute(qs, db, cfg.w, cfg.p, k)
    for rank, idx, dst, calls in res:
        assert np.array_equal(idx, o_idx)
        assert np.allclose(dst, o_dst, rtol=1e-6)
        assert calls == [Q // 2 if rank == 0 else Q - Q // 2]


def _worker_uid(rank, world, port, result_q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_0811_3301_b200.binding import DtwlbError
        from paper_0811_3301_b200.sharded import broadcast_unique_id
        try:
            uid = broadcast_unique_id()
        except DtwlbError as e:  # NCCL not loadable in this image: nothing to bootstrap
            uid = repr(e).encode()
        result_q.put((rank, uid))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:
        result_q.put((rank, repr(e).encode()))
        raise


def test_communicator_id_broadcast():
    """Bootstrap of the library's NCCL communicator (nn_opts.nccl_comm): rank 0's 128-byte
    dtwlb_get_unique_id reaches every rank unchanged (gloo here; the GPU ranks then call
    dtwlb_comm_init with it)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_uid, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert res[0] == res[1]
    assert len(res[0]) == 128
