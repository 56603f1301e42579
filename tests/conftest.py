"""Shared fixtures.  GPU tests carry @pytest.mark.gpu and call the CUDA path through
the C ABI; everything else runs on CPU (oracle vs golden fixtures, host logic, the
library's exported symbols, gloo multi-process sharding)."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
CODES = ROOT / "codes"
for p in (str(ROOT), str(ROOT / "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)

# the reference test suite's fixed matrices (pkg/tests/test_decoder.py:30-35, conftest.py:12-14)
TEST_BASE_4x8_Z3 = [
    [0, 1, -1, -1, 2, -1, 1, -1],
    [0, -1, 1, -1, -1, 2, 0, -1],
    [-1, 2, -1, 0, -1, 1, -1, 2],
    [-1, -1, 2, 1, 0, -1, -1, 2],
]
MERGE_EXAMPLE_FULL = [[1, 0, -1], [2, 1, 1], [0, 2, 0]]
MERGE_EXAMPLE_TOP_PAIR = [[1, -1, -1], [-1, 2, 1], [2, 0, 0]]
MERGE_EXAMPLE_OUTER_PAIR = [[1, -1, -1], [2, 0, 0], [-1, 2, 1]]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); calls the C ABI")


def make_code(shifts, z, merged=False):
    import paper_2004_09084_b200 as q

    base = q.BaseMatrix(len(shifts), len(shifts[0]), z, shifts)
    sched = q.greedy_schedule(base) if merged else q.single_row_schedule(base)
    return base, sched, q.build_compact_index(base, sched)


def load_code(name, merged=True):
    import paper_2004_09084_b200 as q

    base = q.load_base_matrix(CODES / f"{name}.txt")
    sched = q.greedy_schedule(base) if merged else q.single_row_schedule(base)
    return base, sched, q.build_compact_index(base, sched)


def channel_llrs(n, snr, seed, snr_idx, frames, start=0):
    import paper_2004_09084_b200 as q

    chan = q.ChannelConfig(snr=snr, seed=seed)
    return np.stack(
        [q.init_llr(q.transmit(np.zeros(n, np.uint8), chan, q.frame_rng(seed, snr_idx, start + i)), chan)
         for i in range(frames)]
    )


def random_base_matrix(rng, max_rows=6, max_cols=12, max_z=16):
    """Random valid shift grid (pkg/tests/conftest.py:22-32 semantics)."""
    n_rows = int(rng.integers(1, max_rows + 1))
    n_cols = int(rng.integers(n_rows, max_cols + 1))
    z = int(rng.integers(1, max_z + 1))
    shifts = np.full((n_rows, n_cols), -1, dtype=np.int64)
    for i in range(n_rows):
        degree = int(rng.integers(1, n_cols + 1))
        cols = rng.choice(n_cols, size=degree, replace=False)
        shifts[i, cols] = rng.integers(0, z, size=degree)
    return shifts.tolist(), z


@pytest.fixture(scope="session")
def gpu():
    """Skip-free GPU guard: a -m gpu run on a box without the library or a device fails loudly."""
    from paper_2004_09084_b200 import _native

    assert _native.device_count() >= 1
    return 0
