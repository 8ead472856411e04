"""Projected multi-GPU C5 step from single-GPU measurements.

Only one B200 is available to this build, so the G-GPU database-sharded step is projected from
its parts, each MEASURED on one GPU with CUDA events:

  * every shard's nn_search on its N/G rows (shard_range), with the threshold exchange fed what
    the NCCL all-reduce MIN would return: pass A runs every shard once and records its thresholds
    at every exchange call (after the first, best-first range -- these do not depend on the
    exchange -- and inside the last range's walk, nn_opts.exchange_walk); pass B replays the
    minima over the shards and records each shard's contribution again (tighter, once the earlier
    exchanges have lowered its thresholds); pass C (timed) replays the minima of both -- for the
    in-walk calls an upper bound of what the all-reduce returns (conservative: slower, never
    faster than the real exchange), every value >= the global k-th best, so exact;
  * nn_merge of the [G][Q][k] shard lists;
  * the all-gather of the lists is NOT measurable here: it is ESTIMATED as 30 us + bytes / 700 GB/s
    (the recipe's measured 8-rank NVLink bus bandwidth is 725 GB/s at 1 GiB).

projected(G) = max over shards of the shard time (median of 3 timed calls) + merge + all-gather estimate.  The query-sharded
comparison mode (replicated database, Q/G queries per GPU) is projected the same way (max over the
G query slices; its all-gather is the same size).  Also checks that the merged sharded result is
bit-identical to the single-GPU result.

usage: python scripts/shard_projection.py [--config C5] [--gpus 2,4,8] > profiles/<round>_shard_projection.json
"""
import argparse
import gc
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402
from paper_0811_3301_b200 import binding as B  # noqa: E402
from paper_0811_3301_b200.sharded import (EXCHANGE_WALK as WALK, common_query_block,  # noqa: E402
                                          query_shard_range, shard_range)


REP_MS = []  # per-repetition times of the last timed() call


def timed(fn, reps=5):
    """Median over reps of the per-call device time (CUDA events around each call), after a
    warm-up call that sizes the workspace; Python's garbage collector is off meanwhile (a
    collection inside an exchange callback stalls the host-driven walk by tens of ms)."""
    fn()
    torch.cuda.synchronize()
    gc.collect()
    gc.disable()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record()
    for r in range(reps):
        out = fn()
        ev[r + 1].record()
    torch.cuda.synchronize()
    gc.enable()
    REP_MS[:] = [ev[r].elapsed_time(ev[r + 1]) for r in range(reps)]
    return sorted(REP_MS)[reps // 2], out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--gpus", default="2,4,8")
    args = ap.parse_args()
    cfg = datagen.CONFIGS[args.config]
    qs_h, db_h = datagen.make(cfg)
    qs = torch.from_numpy(qs_h).cuda()
    db = torch.from_numpy(db_h).cuda()
    w, p, k = cfg.w, cfg.p, cfg.k
    t1, (i1, d1) = timed(lambda: B.nn_search(qs, db, w, p, k))
    _, _, st1 = B.nn_search(qs, db, w, p, k, return_stats=True)
    one_stats = {kk: (round(v, 3) if isinstance(v, float) else v) for kk, v in st1.items()
                 if kk.startswith("ms_") or kk in ("improved_evaluated", "dtw_evaluated", "dtw_cells_computed",
                                                   "walk_rounds", "range1_dtw")}
    res = {"config": cfg.name, "Q": cfg.Q, "N": cfg.N, "one_gpu_ms": t1, "one_gpu_stats": one_stats,
           "projections": []}
    for G in [int(g) for g in args.gpus.split(",")]:
        bounds = [shard_range(cfg.N, G, g) for g in range(G)]
        qb = common_query_block(bounds[0][1] - bounds[0][0], device=qs.device)
        # pass A: every shard's thresholds after its first range, per query block
        rec = []
        for lo, hi in bounds:
            blocks = []
            B.nn_search(qs, db[lo:hi], w, p, k, index_base=lo, query_block=qb, shards=G, exchange_walk=WALK,
                        exchange=lambda thr, b=blocks: b.append(thr.clone()))
            rec.append(torch.cat(blocks))
        thr_min = torch.stack(rec).min(dim=0).values
        # pass B: replay pass A's minima and record what each shard would contribute then (its
        # local thresholds, tighter than in pass A once the earlier exchanges have lowered them)
        rec = []
        for lo, hi in bounds:
            contrib, pos_b = [], [0]

            def ex_b(thr, contrib=contrib, pos_b=pos_b):
                n_ = thr.numel()
                contrib.append(thr.clone())
                torch.minimum(thr, thr_min[pos_b[0]:pos_b[0] + n_], out=thr)
                pos_b[0] += n_
            B.nn_search(qs, db[lo:hi], w, p, k, index_base=lo, query_block=qb, shards=G, exchange_walk=WALK,
                        exchange=ex_b)
            rec.append(torch.cat(contrib))
        thr_min = torch.minimum(thr_min, torch.stack(rec).min(dim=0).values)
        # pass C (timed): the exchange returns what the all-reduce MIN would
        shard_ms, lists, shard_reps = [], [], []
        for lo, hi in bounds:
            def run(lo=lo, hi=hi):
                pos = [0]

                def ex(thr):
                    n = thr.numel()
                    torch.minimum(thr, thr_min[pos[0]:pos[0] + n], out=thr)
                    pos[0] += n
                return B.nn_search(qs, db[lo:hi], w, p, k, index_base=lo, query_block=qb, exchange=ex, shards=G,
                                   exchange_walk=WALK)
            ms, out = timed(run)
            shard_ms.append(ms)
            shard_reps.append([round(x, 2) for x in REP_MS])
            lists.append(out)
        # stage times of shard 0 (a separate stats-enabled run of pass C)
        lo0, hi0 = bounds[0]
        pos0 = [0]

        def ex0(thr):
            n_ = thr.numel()
            torch.minimum(thr, thr_min[pos0[0]:pos0[0] + n_], out=thr)
            pos0[0] += n_
        _, _, st0 = B.nn_search(qs, db[lo0:hi0], w, p, k, index_base=lo0, query_block=qb, exchange=ex0, shards=G,
                                exchange_walk=WALK, return_stats=True)
        stages0 = {kk: round(v, 3) for kk, v in st0.items() if kk.startswith("ms_")}
        stages0.update({kk: st0[kk] for kk in ("improved_evaluated", "dtw_evaluated", "dtw_cells_computed",
                                                "walk_rounds", "range1_dtw")})
        g_idx = torch.stack([o[0] for o in lists])
        g_dst = torch.stack([o[1] for o in lists])
        merge_ms, (m_idx, m_dst) = timed(lambda: B.nn_merge(g_idx, g_dst), reps=10)
        exact = bool(torch.equal(m_idx, i1) and torch.equal(m_dst, d1))
        gather_bytes = G * cfg.Q * k * 12
        gather_est_ms = 0.030 + gather_bytes / 700e9 * 1e3
        proj = max(shard_ms) + merge_ms + gather_est_ms
        # query-sharded comparison: replicated database, Q/G queries per GPU
        q_ms = []
        for g in range(G):
            a, b = query_shard_range(cfg.Q, G, g)
            ms, _ = timed(lambda a=a, b=b: B.nn_search(qs[a:b], db, w, p, k), reps=1)
            q_ms.append(ms)
        qproj = max(q_ms) + gather_est_ms
        res["projections"].append({
            "gpus": G, "query_block": qb, "shard_ms": shard_ms, "max_shard_ms": max(shard_ms),
            "merge_ms": merge_ms, "allgather_est_ms": gather_est_ms, "projected_step_ms": proj,
            "projected_speedup": t1 / proj, "projected_efficiency": t1 / proj / G,
            "sharded_result_bit_identical": exact, "shard0_stats": stages0, "shard_rep_ms": shard_reps,
            "query_sharded": {"slice_ms": q_ms, "projected_step_ms": qproj, "projected_speedup": t1 / qproj}})
        print(f"G={G}: shards max {max(shard_ms):.1f} ms (min {min(shard_ms):.1f}), merge {merge_ms:.3f} ms, "
              f"projected {proj:.1f} ms -> {t1 / proj:.2f}x; query-sharded {qproj:.1f} ms -> {t1 / qproj:.2f}x; "
              f"exact={exact}", file=sys.stderr)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
