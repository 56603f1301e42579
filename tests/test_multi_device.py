"""Data-parallel paths (north-star item 5; /root/reference/pkg/src/qcldpc/bench.py:139-150).

The driver's boxes here have one GPU, so every multi-device path is exercised with
several slices (threads, ranks) sharing cuda:0: the splitting, the per-slice decode
and the order-preserving concatenation are what is under test, and results must be
bit-identical to one decoder decoding the whole batch.
"""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import CODES, ROOT, channel_llrs, load_code


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


# ------------------------------------------------------------------ CPU (no GPU)


def test_bench_relaunches_itself_under_torchrun():
    """`python bench.py --gpus N` outside torchrun becomes one rank per GPU."""
    sys.path.insert(0, str(ROOT))
    import bench

    args = type("A", (), dict(gpus=4, steps=7, warmup=3, batch=64, impl="b200", precision="fp32"))()
    cmd = bench.relaunch_cmd(args, 12345)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=12345" in cmd
    tail = cmd[cmd.index(str(ROOT / "bench.py")) + 1:]
    assert tail == ["--gpus", "4", "--steps", "7", "--warmup", "3", "--batch", "64", "--impl", "b200",
                    "--precision", "fp32"]


def test_campaign_roofline_fields():
    from paper_2004_09084_b200.campaign import CampaignCell, CampaignConfig, _device_metadata, _roofline

    cfg = CampaignConfig(matrix_path="x", snr_list=(0.2,), devices=(0, 1), precision="fp32")
    meta = _device_metadata(cfg, pool=False)
    assert meta["gpu_count"] == 2 and meta["bytes_per_edge_iteration"] == 16 and meta["host_cores"] >= 1
    cell = CampaignCell(0.2, 0.0, 10.0, 1e-3, 1.0, 0.5, 3767500, 0.5)
    r = _roofline(cell, iterations_total=640, wall=0.25, device_meta=meta)
    assert r["edge_iterations"] == 640 * 3767500
    assert r["achieved_gbs"] == pytest.approx(16 * 640 * 3767500 / 0.25 / 1e9)
    assert r["achieved_gbs_per_gpu"] == pytest.approx(r["achieved_gbs"] / 2)
    assert r["roofline_fraction"] == pytest.approx(r["achieved_gbs_per_gpu"] / meta["hbm_peak_gbs_per_gpu"])


# ------------------------------------------------------------------------ GPU


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_sharded_decoder_two_slices_on_one_gpu_bit_identical(gpu, precision):
    import paper_2004_09084_b200 as q

    base, sched, index = load_code("standin_v2_z100")
    n, m = base.n_cols * base.z, base.n_rows * base.z
    llr = channel_llrs(n, 0.2, 7, 0, 13)
    syn = np.zeros((13, m), np.uint8)
    cfg = q.DecoderConfig(max_iterations=30, early_termination=True)
    want = q.LayeredDecoder(index, sched, cfg, precision=precision).decode_batch_arrays(llr, syn)
    got = q.ShardedDecoder(index, sched, cfg, devices=[0, 0], precision=precision).decode_batch_arrays(llr, syn)
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
    assert got[0].shape == (13, n)


@pytest.mark.gpu
def test_campaign_two_devices_equal_one(gpu):
    from paper_2004_09084_b200.campaign import CampaignConfig, run_campaign

    common = dict(matrix_path=str(CODES / "standin_v2_z100.txt"), snr_list=(0.18, 0.2), max_iterations=20,
                  early_termination=True, batch_size=16, min_trials=64, seed=3)
    for channel in ("host", "device"):
        one = run_campaign(CampaignConfig(channel=channel, devices=(0,), **common))
        two = run_campaign(CampaignConfig(channel=channel, devices=(0, 0), **common))
        for a, b in zip(one.cells, two.cells):
            assert (a.fer, a.avg_iterations) == (b.fer, b.avg_iterations), channel
        assert two.metadata["device"]["devices"] == [0, 0] and len(two.roofline) == 2
        assert all(r["achieved_gbs"] > 0 for r in two.roofline)


@pytest.mark.gpu
def test_campaign_pool_falls_back_when_flow_engine_unsupported(gpu, tmp_path):
    """Frame pool requested (device channel, ET, FP32) on a code the flow engine does not
    cover (a row of degree 16 > 12): the batched device decode runs instead, with the
    same per-frame outcomes (it used to raise QCL_EUNSUP)."""
    import paper_2004_09084_b200 as q
    from paper_2004_09084_b200.campaign import CampaignConfig, run_campaign

    rng = np.random.default_rng(4)
    shifts = np.full((3, 20), -1, dtype=np.int64)
    shifts[0, :16] = rng.integers(0, 16, 16)
    shifts[1, [0, 3, 16, 17, 18]] = rng.integers(0, 16, 5)
    shifts[2, [1, 5, 18, 19]] = rng.integers(0, 16, 4)
    path = tmp_path / "deg16.txt"
    path.write_text(q.serialize_base_matrix(q.BaseMatrix(3, 20, 16, shifts.tolist())))
    common = dict(matrix_path=str(path), snr_list=(1.0,), max_iterations=20, early_termination=True,
                  batch_size=8, min_trials=32, seed=5, channel="device")
    pooled = run_campaign(CampaignConfig(frame_pool=True, **common))
    batched = run_campaign(CampaignConfig(frame_pool=False, **common))
    assert pooled.metadata["device"]["frame_pool"] is False
    assert [(c.fer, c.avg_iterations) for c in pooled.cells] == [(c.fer, c.avg_iterations) for c in batched.cells]


@pytest.mark.gpu
def test_campaign_pool_with_two_lanes_falls_back(gpu):
    """batch_size 2 (ADVICE r1's other failing case): two lanes are below the flow
    engine's 16-byte runs, so the batched decode runs instead, same outcomes."""
    from paper_2004_09084_b200.campaign import CampaignConfig, run_campaign

    common = dict(matrix_path=str(CODES / "standin_v2_z100.txt"), snr_list=(0.2,), max_iterations=20,
                  early_termination=True, batch_size=2, min_trials=8, seed=5, channel="device")
    pooled = run_campaign(CampaignConfig(frame_pool=True, **common))
    batched = run_campaign(CampaignConfig(frame_pool=False, **common))
    assert pooled.metadata["device"]["frame_pool"] is False
    assert [(c.fer, c.avg_iterations) for c in pooled.cells] == [(c.fer, c.avg_iterations) for c in batched.cells]


def _rank(rank, world, port, out):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2004_09084_b200 as q
    from paper_2004_09084_b200.sharding import gather_outcomes, shard_range

    base, sched, index = load_code("standin_v2_z100")
    n, m = base.n_cols * base.z, base.n_rows * base.z
    a, b = shard_range(21, world, rank)
    llr = channel_llrs(n, 0.19, 11, 2, b - a, start=a)
    dec = q.LayeredDecoder(index, sched, q.DecoderConfig(max_iterations=25, early_termination=True), device=0)
    w, c, it = dec.decode_batch_arrays(llr, np.zeros((b - a, m), np.uint8))
    gw, gc, gi = gather_outcomes(w, c, it)
    if rank == 0:
        np.savez(out, w=gw, c=gc, i=gi)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_gloo_ranks_decode_on_the_gpu(gpu, tmp_path):
    """Two processes, each decoding its contiguous frame range through the CUDA path on
    cuda:0, all-gathered over gloo: equal to one process decoding all 21 frames."""
    import torch.multiprocessing as mp

    import paper_2004_09084_b200 as q

    out = tmp_path / "g.npz"
    mp.spawn(_rank, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    g = np.load(out)
    base, sched, index = load_code("standin_v2_z100")
    n, m = base.n_cols * base.z, base.n_rows * base.z
    llr = channel_llrs(n, 0.19, 11, 2, 21)
    dec = q.LayeredDecoder(index, sched, q.DecoderConfig(max_iterations=25, early_termination=True))
    w, c, it = dec.decode_batch_arrays(llr, np.zeros((21, m), np.uint8))
    assert np.array_equal(g["w"], w) and np.array_equal(g["c"], c) and np.array_equal(g["i"], it)


@pytest.mark.gpu
def test_bench_two_ranks_plumbing(gpu):
    """`bench.py --gpus 2` on a one-GPU box: relaunched under torchrun, two ranks (gloo for
    the timing all-reduce since they share the GPU), one JSON line for the whole job."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--batch", "16"], capture_output=True, text=True, timeout=900, env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = lines[0]
    assert line["n_gpus"] == 2 and line["config"]["global_batch"] == 32 and line["config"]["batch_per_gpu"] == 16
    assert "ranks_share_gpus" in line and line["value"] > 0 and line["e2e"]["value"] > 0


def _nccl_rank(rank, port, out):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    from paper_2004_09084_b200.sharding import gather_outcomes

    rng = np.random.default_rng(3)
    w = (rng.random((5, 1003)) < 0.5).astype(np.uint8)
    c = rng.random(5) < 0.5
    it = rng.integers(1, 50, 5)
    gw, gc, gi = gather_outcomes(w, c, it)
    np.savez(out, ok=np.array(np.array_equal(gw, w) and np.array_equal(gc, c) and np.array_equal(gi, it)))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_gather_outcomes_over_nccl(gpu, tmp_path):
    """The result gather on an NCCL group exchanges device tensors (one rank here: the
    packing, the device round trip and the unpacking are what is checked)."""
    import torch.multiprocessing as mp

    out = tmp_path / "n.npz"
    mp.spawn(_nccl_rank, args=(_free_port(), str(out)), nprocs=1, join=True)
    assert bool(np.load(out)["ok"])
