"""Database-sharded multi-GPU k-NN: one process per GPU.

Rank r of G owns database rows [r*N//G, (r+1)*N//G); queries are replicated.
Each rank runs the full cascade on its shard (``nn_search`` with
``index_base`` = its first row).  After each query block's first (best-first)
range the ranks all-reduce (MIN) their per-query thresholds tau_q^p (1+eps)
(``exchange``): a shard's local k-th best is >= the global k-th best, so the
minimum over shards is a safe threshold for every shard and prunes each shard's
second range as if it saw the whole database.  Finally the ranks exchange their
[Q][k] (index, distance) lists with one NCCL all-gather and merge them
(``nn_merge``: the k smallest by (distance, index) of the G*k entries).  No
candidate of the global k-NN is ever pruned (its distance is <= every
threshold), and the union of the shard lists contains the global k-NN.

The search and merge callables are injectable so the protocol can be tested
with ``gloo`` on CPU (tests/test_sharded_cpu.py); the product path uses the
CUDA library (``binding.nn_search`` / ``binding.nn_merge``).
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist

# threshold exchanges inside the last range's DTW walk (nn_opts.exchange_walk: after its rounds
# 2, 4, 6) on top of the one after the best-first range: within the last range each shard's
# threshold otherwise tightens only from its own 1/G of the candidates
EXCHANGE_WALK = 3


def shard_range(N: int, world: int, rank: int):
    """Contiguous, balanced rows [lo, hi) of rank `rank` (sizes differ by at most 1)."""
    return rank * N // world, (rank + 1) * N // world


def common_query_block(N_shard: int, group: Optional[dist.ProcessGroup] = None, device=None) -> int:
    """Queries per pipeline block, identical on every rank (the threshold exchange is a
    collective called once per block): the minimum over ranks of what each rank's free
    device memory allows (~10 bytes per (query, candidate) pair, cf. nn_search)."""
    if device is not None and device.type == "cuda":
        free = torch.cuda.mem_get_info(device)[0]
        qb = max(64, int(free * 0.4 / (max(1, N_shard) * 10 + 4096)) // 64 * 64)
    else:
        qb = 1 << 20
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        t = torch.tensor([qb], dtype=torch.int64, device=device if device is not None else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        qb = int(t.item())
    return qb


def broadcast_unique_id(group: Optional[dist.ProcessGroup] = None, device=None) -> bytes:
    """Rank 0's 128-byte NCCL id (dtwlb_get_unique_id), broadcast to every rank of `group`."""
    from . import binding
    buf = torch.zeros(128, dtype=torch.uint8, device=device)
    if dist.get_rank(group) == 0:
        buf.copy_(torch.frombuffer(bytearray(binding.get_unique_id()), dtype=torch.uint8))
    dist.broadcast(buf, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return bytes(buf.cpu().numpy().tobytes())


def make_communicator(group: Optional[dist.ProcessGroup] = None, device=None):
    """The library's NCCL communicator over `group` (nn_opts.nccl_comm): rank 0 creates the
    128-byte id, torch.distributed broadcasts it, every rank joins on its current device."""
    from . import binding
    uid = broadcast_unique_id(group, device)
    return binding.Communicator(uid, dist.get_world_size(group), dist.get_rank(group))


def sharded_nn_search(queries: torch.Tensor, db_shard: torch.Tensor, shard_lo: int, w: int, p: int, k: int,
                      group: Optional[dist.ProcessGroup] = None,
                      search: Optional[Callable] = None, merge: Optional[Callable] = None,
                      out_local=None, gather_bufs=None, query_block: Optional[int] = None, comm=None):
    """Global k-NN over the union of all ranks' shards; every rank gets the result.

    Shards with fewer than k rows contribute their whole shard padded with
    (index -1, distance +inf), which the merge ignores.  ``comm`` (make_communicator) makes the
    library min-reduce the thresholds itself with NCCL (no Python in the search loop); it is used
    only when every shard holds >= k rows (checked collectively), else the Python exchange runs.
    """
    if search is None or merge is None:
        from . import binding
        search = search or binding.nn_search
        merge = merge or binding.nn_merge
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    Q = queries.shape[0]
    dev = queries.device
    kk = min(k, db_shard.shape[0])
    kw = {}
    if world > 1:
        # all ranks use the same blocking; thresholds are min-reduced after each block's first range
        kw["query_block"] = query_block or common_query_block(db_shard.shape[0], group, dev)
        kw["shards"] = world  # each shard seeds from 1/world of the best-first range
        kw["exchange_walk"] = EXCHANGE_WALK  # + exchanges inside the last range's walk
        use_comm = False
        if comm is not None:  # every rank must take the same path: min over the shards of kk
            t = torch.tensor([kk], dtype=torch.int64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
            use_comm = int(t.item()) >= k
        if use_comm:
            kw["nccl_comm"] = comm
        elif kk >= k:
            kw["exchange"] = lambda thr: dist.all_reduce(thr, op=dist.ReduceOp.MIN, group=group)
        else:
            # a shard with fewer than k rows: its kk-th best is NOT an upper bound on the global
            # k-th best, so it contributes +inf and only receives the other shards' minimum
            def _ex_small(thr):
                t = torch.full_like(thr, float("inf"))
                dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
                torch.minimum(thr, t, out=thr)
            kw["exchange"] = _ex_small
    if kk > 0:
        if out_local is not None and kk == k:
            idx, dst = search(queries, db_shard, w, p, k, index_base=shard_lo, out=out_local, **kw)
        else:
            idx, dst = search(queries, db_shard, w, p, kk, index_base=shard_lo, **kw)
    else:
        idx = torch.empty((Q, 0), dtype=torch.int64, device=dev)
        dst = torch.empty((Q, 0), dtype=torch.float32, device=dev)
        if world > 1:  # an empty shard still takes part in every block's threshold exchange
            qb = kw["query_block"]
            for b0 in range(0, Q, qb):
                for _ in range(1 + kw["exchange_walk"]):  # the calls every other shard makes per block
                    kw["exchange"](torch.full((min(qb, Q - b0),), float("inf"), dtype=torch.float32, device=dev))
    if kk < k:  # pad to k
        pad_i = torch.full((Q, k - kk), -1, dtype=torch.int64, device=dev)
        pad_d = torch.full((Q, k - kk), float("inf"), dtype=torch.float32, device=dev)
        idx = torch.cat([idx, pad_i], 1)
        dst = torch.cat([dst, pad_d], 1)
    if world == 1:
        return idx, dst
    if gather_bufs is None:
        g_idx = torch.empty((world * Q, k), dtype=torch.int64, device=dev)
        g_dst = torch.empty((world * Q, k), dtype=torch.float32, device=dev)
    else:
        g_idx, g_dst = gather_bufs
    # concatenated along dim 0 (the layout both NCCL and gloo accept), viewed as [G][Q][k]
    dist.all_gather_into_tensor(g_idx, idx.contiguous(), group=group)
    dist.all_gather_into_tensor(g_dst, dst.contiguous(), group=group)
    return merge(g_idx.view(world, Q, k), g_dst.view(world, Q, k))



def query_shard_range(Q: int, world: int, rank: int):
    """Contiguous, balanced queries [lo, hi) of rank `rank` in the query-sharded mode."""
    return rank * Q // world, (rank + 1) * Q // world


def query_sharded_nn_search(queries: torch.Tensor, db: torch.Tensor, w: int, p: int, k: int,
                            group: Optional[dist.ProcessGroup] = None, search: Optional[Callable] = None,
                            **kw):
    """The comparison mode of SURVEY 8(e): the whole database is replicated on every rank and the
    QUERIES are split; each rank searches its queries against all N rows with no collective during
    the search, then the [Q][k] results are all-gathered so that every rank holds the full answer.
    Exact for the same reason as the single-GPU search (every query sees the whole set S).
    Per-rank work is Q/G queries x N rows, the same as the database-sharded mode's Q x N/G, but each
    rank streams the full database (N n 4 bytes of HBM per query block) and needs it resident."""
    if search is None:
        from . import binding
        search = binding.nn_search
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    Q = queries.shape[0]
    lo, hi = query_shard_range(Q, world, rank)
    dev = queries.device
    idx, dst = search(queries[lo:hi], db, w, p, k, **kw)
    if world == 1:
        return idx, dst
    # ranks may hold different query counts: pad to the largest, gather, then drop the padding
    cnt = max(query_shard_range(Q, world, r)[1] - query_shard_range(Q, world, r)[0] for r in range(world))
    pi = torch.full((cnt, k), -1, dtype=torch.int64, device=dev)
    pd = torch.full((cnt, k), float("inf"), dtype=torch.float32, device=dev)
    pi[:hi - lo] = idx
    pd[:hi - lo] = dst
    gi = torch.empty((world * cnt, k), dtype=torch.int64, device=dev)
    gd = torch.empty((world * cnt, k), dtype=torch.float32, device=dev)
    dist.all_gather_into_tensor(gi, pi, group=group)
    dist.all_gather_into_tensor(gd, pd, group=group)
    parts_i, parts_d = [], []
    for r in range(world):
        a, b = query_shard_range(Q, world, r)
        parts_i.append(gi[r * cnt:r * cnt + (b - a)])
        parts_d.append(gd[r * cnt:r * cnt + (b - a)])
    return torch.cat(parts_i), torch.cat(parts_d)
