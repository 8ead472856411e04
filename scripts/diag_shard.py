"""Diagnostic: one C5 database shard (the first N/G rows) searched with the full query set, at several
query blocks, with the stage times -- why a 1/2 shard does not take half the 1-GPU time."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402
from paper_0811_3301_b200 import binding as B  # noqa: E402

cfg = datagen.CONFIGS["C5"]
qs_h, db_h = datagen.make(cfg)
qs = torch.from_numpy(qs_h).cuda()
db = torch.from_numpy(db_h).cuda()
for N, qb in [(1_000_000, 0), (1_000_000, 8192), (500_000, 0), (500_000, 4096), (500_000, 8192), (250_000, 0), (125_000, 0)]:
    d = db[:N]
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        i_, d_, st = B.nn_search(qs, d, cfg.w, cfg.p, cfg.k, query_block=qb, return_stats=True)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"N": N, "query_block": qb, "ms": round(ms, 2),
                      "stages": {k: round(v, 2) for k, v in st.items() if k.startswith("ms_")},
                      "improved_frac": st["improved_evaluated"] / st["pairs"], "dtw_frac": st["dtw_evaluated"] / st["pairs"],
                      "cells": st["dtw_cells_computed"], "rounds": st["walk_rounds"]}), flush=True)
