"""Seeded synthetic stand-in for the paper's unpublished rate-0.1, n=10^6 code.

The paper's QC-MET-LDPC matrix is not published (``SPEC.md:13,108``).  Its
published invariants are a 360x400 base grid, z = 2500 and 3,767,500 expanded
edges (``PAPER.md:345``), i.e. exactly 1507 circulants.  This module builds
the "v2" stand-in recipe of SURVEY.md Appendix A:

* 50 high-degree columns (0..49) shared by everything;
* rows 0..9 are type-1 checks of degree 11,11,11,11,11,11,11,10,10,10 on the
  high columns only;
* rows 10..359 take 3 high columns plus one private degree-1 column 50 + (i-10).

High columns are picked least-loaded-first with random tie-breaking.  The
result has row degrees {4, 10, 11}, 350 degree-1 columns and a greedy schedule
of 30 layers.  Support is drawn from the same stream as the shifts, and is
identical for z=100 and z=2500 at seed 0, which makes the
z=100 twin a cheap oracle-sized copy of the benchmark code.
"""

from __future__ import annotations

import numpy as np

from .qc_code import BaseMatrix

__all__ = ["standin_v2", "TYPE1_DEGREES"]

TYPE1_DEGREES = (11, 11, 11, 11, 11, 11, 11, 10, 10, 10)
N_ROWS, N_COLS, N_HIGH = 360, 400, 50


def standin_v2(z=2500, seed=0):
    """The v2 stand-in base matrix at expansion factor ``z``."""
    rng = np.random.default_rng(seed=seed)
    grid = np.full((N_ROWS, N_COLS), -1, dtype=np.int64)
    load = np.zeros(N_HIGH)

    def pick(k):
        order = np.lexsort((rng.random(N_HIGH), load))
        cols = order[:k]
        load[cols] += 1
        return cols

    # columns are picked before the row's shifts are drawn; this order
    # reproduces the 30-layer schedule quoted in SURVEY.md Appendix A
    for i, deg in enumerate(TYPE1_DEGREES):
        cols = pick(deg)
        grid[i, cols] = rng.integers(0, z, size=deg)
    for i in range(len(TYPE1_DEGREES), N_ROWS):
        cols = pick(3)
        grid[i, cols] = rng.integers(0, z, size=3)
        grid[i, N_HIGH + i - len(TYPE1_DEGREES)] = rng.integers(0, z)
    return BaseMatrix(N_ROWS, N_COLS, z, grid)
