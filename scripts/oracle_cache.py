"""Oracle-result cache for the full-size configs ("compute once, cache, re-verify
subsets").  Calls ONLY oracle/ (fp64 Alg. 3 scan, pinned to brute force by
tests/test_oracle_search.py) on a sample of queries of each full-size BASELINE config and stores
the k + 8 nearest neighbours (indices and rooted distances) under tests/golden/, so the GPU test
can check far more than a handful of full-size queries without re-running the slow oracle.

usage: python scripts/oracle_cache.py [C5 C3 C4] [--sample 256]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402
import oracle  # noqa: E402

EXTRA = 8


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C5", "C3", "C4"])
    ap.add_argument("--sample", type=int, default=256)
    args = ap.parse_args()
    threads = os.cpu_count() or 1
    for name in args.configs:
        c = datagen.CONFIGS[name]
        qs, db = datagen.make(c)
        rows = np.unique(np.linspace(0, c.Q - 1, args.sample).astype(np.int64))
        t0 = time.time()
        o_idx, o_dist, _ = oracle.nn_twopass(qs[rows], db, c.w, c.p, c.k + EXTRA, threads=threads)
        out = os.path.join(ROOT, "tests", "golden", f"oracle_knn_{name}.npz")
        np.savez_compressed(out, rows=rows, idx=o_idx, dist=o_dist, w=c.w, p=c.p, k=c.k + EXTRA,
                            Q=c.Q, N=c.N, n=c.n, seed=c.seed)
        print(f"{name}: {len(rows)} queries in {time.time() - t0:.1f} s -> {out}", flush=True)


if __name__ == "__main__":
    main()
