"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no envelope, bound or DTW):
only the workload recipes of BASELINE.json ``configs`` and the random-number
plumbing.  Every series is generated in fp64 and rounded once to fp32; both
the oracle (which upcasts back to fp64) and the GPU read the same fp32 arrays.

Streams: ``numpy.random.Generator(PCG64(SeedSequence([seed, role, block])))``
with role 0 = database, 1 = queries, and blocks of ``BLOCK`` rows, so row r of
a family does not depend on how many rows are drawn (N can be sliced).

Families:
- ``rw``    random walk x_1 = 0, x_i = x_{i-1} + N(0,1) (paper P:744); optional
            z-normalisation (mean 0, population std 1) as BASELINE configs 2,3,5 add.
- ``shape`` radial distance of a closed contour,
            r(t) = 1 + sum_{h=1..8} (a_h cos h t + b_h sin h t), a_h, b_h ~ N(0, (0.3/h)^2),
            n uniform angles from a random cyclic start offset s ~ U{0..n-1},
            plus N(0, 0.01^2) noise, z-normalised (BASELINE config 4; stands in for the
            paper's shape datasets P:804-806, which are not available).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

BLOCK = 4096
ROLE_DB = 0
ROLE_QUERY = 1


@dataclass(frozen=True)
class Config:
    name: str
    Q: int
    N: int
    n: int
    w: int
    p: int
    k: int
    family: str
    znorm: bool
    seed: int

    @property
    def pairs(self) -> int:
        return self.Q * self.N

    @property
    def band_cells(self) -> int:
        """Cells of the Sakoe-Chiba band |i-j| <= w in an n x n table."""
        w = min(self.w, self.n - 1)
        return self.n * (2 * w + 1) - w * (w + 1)


# BASELINE.json "configs" (C1..C5); C2 runs at p = 1 and p = 2.
CONFIGS = {
    "C1": Config("C1", 1, 256, 128, 12, 1, 1, "rw", False, 0),
    "C2p1": Config("C2p1", 64, 10_000, 256, 25, 1, 1, "rw", True, 2),
    "C2p2": Config("C2p2", 64, 10_000, 256, 25, 2, 1, "rw", True, 2),
    "C3": Config("C3", 1_000, 100_000, 1_000, 50, 2, 1, "rw", True, 3),
    "C4": Config("C4", 4_096, 200_000, 512, 51, 1, 1, "shape", True, 4),
    "C5": Config("C5", 8_192, 1_000_000, 256, 25, 2, 10, "rw", True, 5),
    # C5-stream (SURVEY 8(d) added row): the first Q in {1, 2, 4, 8} C5 queries against the C5
    # database -- the memory-bound regime of the bound pass (BASELINE "bound passes >= 60% HBM")
    "C5s1": Config("C5s1", 1, 1_000_000, 256, 25, 2, 10, "rw", True, 5),
    "C5s2": Config("C5s2", 2, 1_000_000, 256, 25, 2, 10, "rw", True, 5),
    "C5s4": Config("C5s4", 4, 1_000_000, 256, 25, 2, 10, "rw", True, 5),
    "C5s8": Config("C5s8", 8, 1_000_000, 256, 25, 2, 10, "rw", True, 5),
}


def _rng(seed: int, role: int, block: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, role, block])))


def _znorm(x: np.ndarray) -> np.ndarray:
    mu = x.mean(axis=1, keepdims=True)
    sd = x.std(axis=1, keepdims=True)  # population std (ddof = 0), reading c9
    sd[sd == 0] = 1.0
    return (x - mu) / sd


def _rw_block(g: np.random.Generator, rows: int, n: int) -> np.ndarray:
    steps = g.standard_normal((rows, n))
    steps[:, 0] = 0.0  # x_1 = 0
    return np.cumsum(steps, axis=1)


def _shape_block(g: np.random.Generator, rows: int, n: int) -> np.ndarray:
    h = np.arange(1, 9, dtype=np.float64)
    a = g.standard_normal((rows, 8)) * (0.3 / h)
    b = g.standard_normal((rows, 8)) * (0.3 / h)
    s = g.integers(0, n, size=rows)
    t = np.arange(n, dtype=np.float64)
    theta = 2.0 * np.pi * (t[None, :] + s[:, None]) / n  # (rows, n)
    r = np.ones((rows, n))
    for j in range(8):
        r += a[:, j:j + 1] * np.cos(h[j] * theta) + b[:, j:j + 1] * np.sin(h[j] * theta)
    r += 0.01 * g.standard_normal((rows, n))
    return r


def series(family: str, rows: int, n: int, seed: int, role: int, znorm: bool,
           start: int = 0) -> np.ndarray:
    """Rows [start, start+rows) of a family as a C-contiguous float32 [rows][n] array."""
    out = np.empty((rows, n), dtype=np.float32)
    if rows == 0:
        return out
    gen = _rw_block if family == "rw" else _shape_block
    b0, b1 = start // BLOCK, (start + rows - 1) // BLOCK
    for b in range(b0, b1 + 1):
        blk = gen(_rng(seed, role, b), BLOCK, n)
        if znorm:
            blk = _znorm(blk)
        lo = max(start, b * BLOCK)
        hi = min(start + rows, (b + 1) * BLOCK)
        out[lo - start:hi - start] = blk[lo - b * BLOCK:hi - b * BLOCK].astype(np.float32)
    return out


def make(cfg: Config | str, Q: int | None = None, N: int | None = None, db_start: int = 0):
    """(queries [Q][n], db [N][n]) float32 for a config; Q/N may be reduced (prefix rows)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    Q = cfg.Q if Q is None else Q
    N = cfg.N if N is None else N
    qs = series(cfg.family, Q, cfg.n, cfg.seed, ROLE_QUERY, cfg.znorm)
    db = series(cfg.family, N, cfg.n, cfg.seed, ROLE_DB, cfg.znorm, start=db_start)
    return qs, db


def random_walks(rows: int, n: int, seed: int, znorm: bool = True, role: int = ROLE_DB):
    """Convenience: seeded random walks (tests with ad-hoc shapes)."""
    return series("rw", rows, n, seed, role, znorm)
