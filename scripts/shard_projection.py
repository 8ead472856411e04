"""Projected multi-GPU C5 step from single-GPU measurements.

Only one B200 is available to this build, so the G-GPU database-sharded step is projected from
its parts, each MEASURED on one GPU with CUDA events:

  * every shard's nn_search on its N/G rows (shard_range), with the threshold exchange fed
    exactly what the NCCL all-reduce MIN would return: pass A runs every shard once and records
    its per-block thresholds after the first (best-first) range; pass B (timed) runs every shard
    again with exchange(thr) = min(thr, min over shards of pass A) -- the same values the real
    all-reduce produces, since a shard's post-range-1 thresholds do not depend on the exchange;
  * nn_merge of the [G][Q][k] shard lists;
  * the all-gather of the lists is NOT measurable here: it is ESTIMATED as 30 us + bytes / 700 GB/s
    (the recipe's measured 8-rank NVLink bus bandwidth is 725 GB/s at 1 GiB).

projected(G) = max over shards of the shard time + merge + all-gather estimate.  The query-sharded
comparison mode (replicated database, Q/G queries per GPU) is projected the same way (max over the
G query slices; its all-gather is the same size).  Also checks that the merged sharded result is
bit-identical to the single-GPU result.

usage: python scripts/shard_projection.py [--config C5] [--gpus 2,4,8] > profiles/<round>_shard_projection.json
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402
from paper_0811_3301_b200 import binding as B  # noqa: E402
from paper_0811_3301_b200.sharded import common_query_block, query_shard_range, shard_range  # noqa: E402


def timed(fn, reps=2):
    fn()  # warm-up (workspace sized)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


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
    res = {"config": cfg.name, "Q": cfg.Q, "N": cfg.N, "one_gpu_ms": t1, "projections": []}
    for G in [int(g) for g in args.gpus.split(",")]:
        bounds = [shard_range(cfg.N, G, g) for g in range(G)]
        qb = common_query_block(bounds[0][1] - bounds[0][0], device=qs.device)
        # pass A: every shard's thresholds after its first range, per query block
        rec = []
        for lo, hi in bounds:
            blocks = []
            B.nn_search(qs, db[lo:hi], w, p, k, index_base=lo, query_block=qb, shards=G,
                        exchange=lambda thr, b=blocks: b.append(thr.clone()))
            rec.append(torch.cat(blocks))
        thr_min = torch.stack(rec).min(dim=0).values
        # pass B (timed): the exchange returns what the all-reduce MIN would
        shard_ms, lists = [], []
        for lo, hi in bounds:
            def run(lo=lo, hi=hi):
                pos = [0]

                def ex(thr):
                    n = thr.numel()
                    torch.minimum(thr, thr_min[pos[0]:pos[0] + n], out=thr)
                    pos[0] += n
                return B.nn_search(qs, db[lo:hi], w, p, k, index_base=lo, query_block=qb, exchange=ex, shards=G)
            ms, out = timed(run)
            shard_ms.append(ms)
            lists.append(out)
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
            "sharded_result_bit_identical": exact,
            "query_sharded": {"slice_ms": q_ms, "projected_step_ms": qproj, "projected_speedup": t1 / qproj}})
        print(f"G={G}: shards max {max(shard_ms):.1f} ms (min {min(shard_ms):.1f}), merge {merge_ms:.3f} ms, "
              f"projected {proj:.1f} ms -> {t1 / proj:.2f}x; query-sharded {qproj:.1f} ms -> {t1 / qproj:.2f}x; "
              f"exact={exact}", file=sys.stderr)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
