"""Appendix B workload through `dtw_band` with no time constraint (w = n - 1):
DTW_p on a sample equals the fp64 oracle (relative 1e-4), white-noise triples never
violate the triangle inequality (the paper found none in 10^5 triples), and random-walk
triples violate it at about the paper's rates (20 % for p = 1, 15 % for p = 2; our
generator gives 18.4 % / 17.4 % on 10^5 triples, profiles/r01f_appendix_b.json)."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))


def test_appendix_b_triangle_statistics(cuda_ok):
    import appendix_b
    res = appendix_b.run(3000, check_oracle=True)
    for key, r in res.items():
        assert r["oracle_max_rel_err"] < 1e-4, (key, r)
    assert res["white_noise_p1"]["violation_frac"] == 0.0
    assert res["white_noise_p2"]["violation_frac"] == 0.0
    assert 0.12 < res["random_walk_p1"]["violation_frac"] < 0.26
    assert 0.10 < res["random_walk_p2"]["violation_frac"] < 0.24
