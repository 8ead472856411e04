"""The row+column cascade of the w <= 32 DTW kernel (reading c21; off by default,
DTWLB_COLCASC=1 switches it on -- read once per process, hence a child process here):
nn_search must return the oracle's k-NN with it on, bit-identical to the default path."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import datagen
import oracle
from knn_compare import assert_knn_match

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import datagen
from paper_0811_3301_b200 import nn_search
out = []
for name, Q, N, k in {cases!r}:
    c = datagen.CONFIGS[name]
    qs, db = datagen.make(c, Q=Q, N=N)
    idx, dist = nn_search(torch.from_numpy(qs).cuda(), torch.from_numpy(db).cuda(), c.w, c.p, k)
    out.append([idx.cpu().numpy().tolist(), dist.cpu().numpy().tolist()])
print(json.dumps(out))
"""
CASES = [("C2p2", 24, 10_000, 5), ("C2p1", 16, 10_000, 3), ("C5", 8, 60_000, 10), ("C1", 1, 256, 1)]


def _run(env_on):
    env = dict(os.environ)
    env.pop("DTWLB_COLCASC", None)
    if env_on:
        env["DTWLB_COLCASC"] = "1"
    r = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT, cases=CASES)], capture_output=True,
                       text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_row_column_cascade_matches_oracle_and_default(cuda_ok):
    on, off = _run(True), _run(False)
    for (name, Q, N, k), (gi, gd), (fi, fd) in zip(CASES, on, off):
        c = datagen.CONFIGS[name]
        qs, db = datagen.make(c, Q=Q, N=N)
        o_idx, o_dist, _ = oracle.nn_twopass(qs, db, c.w, c.p, min(N, k + 8), threads=os.cpu_count() or 1)
        assert_knn_match(np.array(gi), np.array(gd), o_idx, o_dist, k)
        assert gi == fi and np.array_equal(np.array(gd, np.float32), np.array(fd, np.float32)), name
