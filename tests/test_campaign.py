"""Device campaigns (paper_2004_09084_b200.campaign) against the reference's own
campaign reports (tests/golden/campaign_*.json, made by make_campaign_golden.py from
the unmodified reference ``qcldpc.bench.run_campaign``).

* host channel (bit-identical PCG64 frames), FP64 parity path: FER and average
  iterations EXACTLY equal to the reference's;
* host channel, FP32 path, and device (Philox) channel: FER inside the reference's
  confidence interval, the acceptance-test form 1.96 * sqrt(p1 q1 / N + p2 q2 / N)
  (tests/test_acceptance.py:194,236), with one frame of slack for p = 0 or 1.
CPU-only tests cover validation and the CSV/JSON report schema.
"""

import csv
import json
import math

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, load_code

CASES = ["campaign_demo4x8z32_et50", "campaign_demo4x8z100_noet10", "campaign_demo4x8z32_encode"]


def golden(name):
    return json.loads((GOLDEN / f"{name}.json").read_text())


def config_of(g, **over):
    from paper_2004_09084_b200.campaign import CampaignConfig

    c = g["metadata"]["campaign"]
    kw = dict(
        matrix_path=str(ROOT / "codes" / g["metadata"]["matrix"]["path"]),
        snr_list=[x["snr"] for x in g["cells"]],
        max_iterations=g["metadata"]["decoder"]["max_iterations"],
        early_termination=g["metadata"]["decoder"]["early_termination"],
        batch_size=c["batch_size"],
        min_trials=c["min_trials"],
        seed=c["seed"],
        encode_mode=c["encode_mode"],
    )
    kw.update(over)
    return CampaignConfig(**kw)


def within_ci(p1, p2, n):
    band = 1.96 * math.sqrt(p1 * (1 - p1) / n + p2 * (1 - p2) / n) + 1.0 / n
    return abs(p1 - p2) <= band


# ------------------------------------------------------------------------ CPU tests


def test_config_validation_messages():
    from paper_2004_09084_b200.campaign import CampaignConfig

    path = str(ROOT / "codes" / "demo_4x8_z32.txt")
    for kw, msg in [
        (dict(snr_list=()), "snr_list must not be empty"),
        (dict(snr_list=(1.0, -1.0)), "every snr must be positive"),
        (dict(snr_list=(1.0,), batch_size=0), "batch_size must be at least 1"),
        (dict(snr_list=(1.0,), batch_size=64, min_trials=8), "min_trials must be at least batch_size"),
        (dict(snr_list=(1.0,), max_iterations=0), "max_iterations must be at least 1"),
        (dict(snr_list=(1.0,), workers=0), "workers must be at least 1"),
        (dict(snr_list=(1.0,), lane_budget=0), "lane_budget must be positive"),
        (dict(snr_list=(1.0,), precision="fp16"), "precision must be one of"),
        (dict(snr_list=(1.0,), channel="wire"), "channel must be one of"),
    ]:
        with pytest.raises(ValueError, match=msg):
            CampaignConfig(matrix_path=path, **kw)
    cfg = CampaignConfig(matrix_path=path, snr_list=[1, 2], batch_size=48, min_trials=100)
    assert cfg.snr_list == (1.0, 2.0) and cfg.frames_per_point == 144


def test_report_schema_csv_and_json(tmp_path):
    from paper_2004_09084_b200.campaign import (
        CSV_COLUMNS,
        SCHEMA_VERSION,
        CampaignCell,
        CampaignReport,
        ScheduleComparison,
        emit_report,
        report_to_dict,
    )

    cell = CampaignCell(1.0, 0.5, 7.5, 1e-3, 12.0, 0.9, 96, 0.01)
    rep = CampaignReport(cells=(cell,), metadata={"schema_version": SCHEMA_VERSION})
    d = report_to_dict(rep)
    assert d["schema_version"] == 1 and d["cells"][0]["fer"] == 0.5
    assert tuple(d["cells"][0]) == CSV_COLUMNS
    p = emit_report(rep, "csv", tmp_path / "r.csv")
    rows = list(csv.reader(p.open()))
    assert tuple(rows[0]) == CSV_COLUMNS and float(rows[1][1]) == 0.5
    cmp = ScheduleComparison(single=rep, merged=rep, single_layer_count=4, merged_layer_count=2)
    p = emit_report(cmp, "csv", tmp_path / "c.csv")
    rows = list(csv.reader(p.open()))
    assert rows[0][0] == "schedule" and [r[0] for r in rows[1:]] == ["single", "merged"]
    p = emit_report(cmp, "json", tmp_path / "c.json")
    assert json.loads(p.read_text())["merged_layer_count"] == 2
    with pytest.raises(ValueError, match="unknown report format"):
        emit_report(rep, "xml", tmp_path / "r.xml")


def test_golden_reports_have_reference_schema():
    from paper_2004_09084_b200.campaign import CSV_COLUMNS, METRIC_DEFINITIONS

    for name in CASES:
        g = golden(name)
        assert g["schema_version"] == 1
        assert g["metadata"]["definitions"] == METRIC_DEFINITIONS
        for cell in g["cells"]:
            assert tuple(cell) == CSV_COLUMNS


# ------------------------------------------------------------------------ GPU tests


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_host_channel_fp64_matches_reference_exactly(gpu, name):
    from paper_2004_09084_b200.campaign import run_campaign

    g = golden(name)
    rep = run_campaign(config_of(g, precision="fp64"))
    for got, want in zip(rep.cells, g["cells"]):
        assert got.fer == want["fer"] and got.avg_iterations == want["avg_iterations"], (got, want)
        assert got.beta == pytest.approx(want["beta"]) and got.total_expanded_edges == want["total_expanded_edges"]
        assert got.utilization == pytest.approx(want["utilization"])
        assert got.throughput_mbits_per_s > 0 and got.latency_per_iteration_s > 0
    for key in ("matrix", "schedule", "decoder", "campaign", "definitions"):
        want = dict(g["metadata"][key])
        have = dict(rep.metadata[key])
        if key == "matrix":
            want.pop("path"), have.pop("path")
        assert have == want, key


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("channel", ["host", "device"])
def test_fp32_and_device_channel_within_reference_ci(gpu, name, channel):
    from paper_2004_09084_b200.campaign import run_campaign

    g = golden(name)
    cfg = config_of(g, precision="fp32", channel=channel)
    rep = run_campaign(cfg)
    n = cfg.frames_per_point
    for got, want in zip(rep.cells, g["cells"]):
        assert within_ci(got.fer, want["fer"], n), (channel, got.snr, got.fer, want["fer"])


@pytest.mark.gpu
def test_device_channel_is_deterministic_and_shard_invariant(gpu):
    """Same seed -> same FER/iterations, whatever the batch size (frames keyed by index)."""
    from paper_2004_09084_b200.campaign import run_campaign

    g = golden("campaign_demo4x8z32_et50")
    a = run_campaign(config_of(g, channel="device", batch_size=64, min_trials=512))
    b = run_campaign(config_of(g, channel="device", batch_size=128, min_trials=512))
    for x, y in zip(a.cells, b.cells):
        assert x.fer == y.fer and x.avg_iterations == y.avg_iterations


@pytest.mark.gpu
def test_compare_schedules_on_device(gpu, tmp_path):
    from paper_2004_09084_b200.campaign import CampaignConfig, compare_schedules, emit_report

    cfg = CampaignConfig(matrix_path=str(ROOT / "codes" / "demo_6x12_z16.txt"), snr_list=(2.0,),
                         max_iterations=20, early_termination=True, batch_size=64, min_trials=128,
                         channel="device")
    cmp = compare_schedules(cfg)
    assert cmp.single_layer_count == 6 and cmp.merged_layer_count < 6
    assert emit_report(cmp, "csv", tmp_path / "cmp.csv").exists()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["campaign_demo4x8z32_et50", "standin_z100_et", "standin_z100_et_128"])
def test_frame_pool_matches_batched_decode_per_frame(gpu, name):
    """The frame pool changes only the timing: FER and average iterations identical to the
    batched device-channel decode (frames are independent; each runs its own sweeps)."""
    from paper_2004_09084_b200.campaign import CampaignConfig, run_campaign

    if name.startswith("standin_z100_et"):
        lanes = 128 if name.endswith("_128") else 16  # 128 lanes: two group blocks per sweep
        kw = dict(matrix_path=str(ROOT / "codes" / "standin_v2_z100.txt"), snr_list=(0.17, 0.2), max_iterations=40,
                  early_termination=True, batch_size=lanes, min_trials=6 * lanes, seed=5, channel="device")
        cfg = CampaignConfig(**kw)
    else:
        cfg = config_of(golden(name), channel="device", batch_size=32, min_trials=256)
    a = run_campaign(cfg.__class__(**{**cfg.__dict__, "frame_pool": False}))
    b = run_campaign(cfg.__class__(**{**cfg.__dict__, "frame_pool": "always"}))
    c = run_campaign(cfg)  # adaptive: pool or batched per SNR point after a first-batch probe
    assert b.metadata["device"]["frame_pool"] and not a.metadata["device"]["frame_pool"]
    assert all(r["path"] == "pool" for r in b.roofline) and all(r["path"] == "batched" for r in a.roofline)
    for x, y, w in zip(a.cells, b.cells, c.cells):
        assert x.fer == y.fer == w.fer and x.avg_iterations == y.avg_iterations == w.avg_iterations, (x, y, w)


@pytest.mark.gpu
def test_frame_pool_per_frame_outcomes_against_states(gpu):
    """qcl_state_decode_pool per frame vs one batched decode per frame range."""
    import paper_2004_09084_b200 as q
    from paper_2004_09084_b200 import _native

    base, sched, index = load_code("standin_v2_z100")
    plan = _native.Plan(index, sched, 0)
    qcfg = _native.make_config(q.DecoderConfig(max_iterations=30, early_termination=True), "fp32")
    pool = _native.State(plan, 8, "fp32")
    conv, iters, err, _ = pool.decode_pool(qcfg, 11, 2, 100, 40, 0.19)
    ref = _native.State(plan, 40, "fp32")
    ref.set_llr_synthetic(seed=11, snr_idx=2, first_frame=100, snr=0.19)
    ref.decode(qcfg)
    _, rconv, riters = ref.results(words=False)
    rerr = ref.frame_errors()
    assert np.array_equal(conv, rconv) and np.array_equal(iters, riters)
    assert np.array_equal(err, ~rconv | rerr)


@pytest.mark.gpu
def test_campaign_command_line(gpu, tmp_path):
    """`python -m paper_2004_09084_b200.campaign` (the reference's `decode-bench run`,
    cli.py:94-139): a JSON report with the reference schema plus the device block."""
    from paper_2004_09084_b200.campaign import main

    out = tmp_path / "r.json"
    rc = main(["--matrix", str(ROOT / "codes" / "demo_4x8_z100.txt"), "--snr", "1.5", "2.5", "--iterations", "10",
               "--early-termination", "--batch-size", "16", "--min-trials", "32", "--channel", "device",
               "--out", str(out)])
    assert rc == 0
    rep = json.loads(out.read_text())
    assert rep["schema_version"] == 1 and len(rep["cells"]) == 2 and len(rep["roofline"]) == 2
    assert rep["metadata"]["device"]["channel"] == "device"
    assert rep["cells"][1]["fer"] <= rep["cells"][0]["fer"]
