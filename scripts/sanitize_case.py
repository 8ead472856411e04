"""Small workloads for compute-sanitizer (SURVEY 4 tier 4): every kernel family of the library on
small inputs -- nn_search (pre-filtered cascade, Alg. 3 as printed, Alg. 2, stream mode, wide band),
the dense bound entry points, dtw_band (register, wide, generic kernels) and nn_merge -- checked
against the oracle so a sanitizer run also proves the results are unchanged under instrumentation.
usage: compute-sanitizer --tool memcheck python scripts/sanitize_case.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import datagen  # noqa: E402
import oracle  # noqa: E402
from knn_compare import assert_knn_match  # noqa: E402
from paper_0811_3301_b200 import (dtw_band, lb_envelope, lb_improved, lb_keogh, lb_piecewise_sym,  # noqa: E402
                                  nn_merge, nn_search)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def main():
    checks = 0
    for name, Q, N, kw in [("C1", 1, 256, {}), ("C2p2", 40, 3000, {}), ("C2p1", 20, 3000, {"prefilter": False}),
                           ("C2p2", 20, 3000, {"keogh_only": True}), ("C5", 8, 5000, {}),
                           ("C5", 3, 5000, {"stream": False}), ("C3", 4, 2000, {})]:
        c = datagen.CONFIGS[name]
        qs, db = datagen.make(c, Q=Q, N=N)
        k = min(c.k, 5)
        idx, dist = nn_search(dev(qs), dev(db), c.w, c.p, k, **kw)
        o_idx, o_dist = oracle.nn_brute(qs, db, c.w, c.p, k + 6, threads=8)
        assert_knn_match(idx.cpu().numpy(), dist.cpu().numpy(), o_idx, o_dist, k)
        checks += 1
    # wide bands through the walk (band w = 100 and unconstrained column mode)
    for name, w in (("C3", 100), ("C2p1", 255)):
        c = datagen.CONFIGS[name]
        qs, db = datagen.make(c, Q=4, N=1500)
        idx, dist = nn_search(dev(qs), dev(db), w, c.p, 3)
        o_idx, o_dist = oracle.nn_brute(qs, db, w, c.p, 9, threads=8)
        assert_knn_match(idx.cpu().numpy(), dist.cpu().numpy(), o_idx, o_dist, 3)
        checks += 1
    # dense bounds and dtw_band
    rng = np.random.default_rng(3)
    qs = np.cumsum(rng.standard_normal((5, 96)), axis=1).astype(np.float32)
    db = np.cumsum(rng.standard_normal((300, 96)), axis=1).astype(np.float32)
    U, L = lb_envelope(dev(qs), 9)
    env = torch.stack([U, L]).contiguous()
    lb_keogh(env, dev(db), 2)
    lb_improved(dev(qs), env, dev(db), 9, 1)
    lb_piecewise_sym(dev(qs), env, dev(db), 9, 2)
    for n, w, p in ((96, 9, 2), (96, 40, 1), (150, 100, 2), (100, 99, 1), (400, 150, 2), (64, 63, 0)):
        x = np.cumsum(rng.standard_normal((40, n)), axis=1).astype(np.float32)
        y = np.cumsum(rng.standard_normal((40, n)), axis=1).astype(np.float32)
        d = dtw_band(dev(x), dev(y), w, p).cpu().numpy()
        ref = np.array([oracle.dtw(x[r], y[r], w, p) for r in range(40)])
        assert np.allclose(d, ref, rtol=1e-4), (n, w, p)
        checks += 1
    gi = torch.tensor([[[0, 2]], [[1, -1]]], dtype=torch.int64).cuda()
    gd = torch.tensor([[[0.5, 1.0]], [[0.5, float("inf")]]], dtype=torch.float32).cuda()
    mi, md = nn_merge(gi, gd)
    assert mi.cpu().tolist() == [[0, 1]]
    torch.cuda.synchronize()
    print(f"sanitize_case ok: {checks} oracle-checked calls")


if __name__ == "__main__":
    main()
