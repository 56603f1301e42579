"""Multi-process data-parallel path on CPU: world_size 2 over gloo.

Each rank takes its contiguous frame range (sharding.shard_range, the same helper
bench.py uses for its per-GPU slices), decodes it (CPU oracle stands in for the GPU
here), and the ranks all-gather bit-packed outcomes; the result must equal the
single-process decode of the whole batch, in order (bench.py:139-150 semantics).
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from conftest import channel_llrs, load_code
    from oracle import oracle
    from paper_2004_09084_b200.sharding import gather_outcomes, shard_range

    base, sched, index = load_code("demo_4x8_z100")
    n = base.n_cols * base.z
    total = 13
    a, b = shard_range(total, world, rank)
    llr = channel_llrs(n, 1.6, 20240901, 4, b - a, start=a)
    code = oracle.OracleCode(index, sched)
    w, c, it = oracle.decode(code, llr, None, 20, True, threads=1)
    gw, gc, gi = gather_outcomes(w, c, it)
    if rank == 0:
        np.savez(out_path, w=gw, c=gc, i=gi)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharding_matches_single_process(tmp_path):
    from conftest import channel_llrs, load_code
    from oracle import oracle

    out = tmp_path / "gathered.npz"
    mp.spawn(_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    g = np.load(out)
    base, sched, index = load_code("demo_4x8_z100")
    n = base.n_cols * base.z
    llr = channel_llrs(n, 1.6, 20240901, 4, 13)
    w, c, it = oracle.decode(oracle.OracleCode(index, sched), llr, None, 20, True)
    assert np.array_equal(g["w"], w) and np.array_equal(g["c"], c) and np.array_equal(g["i"], it)
