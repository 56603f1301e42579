"""FER over a seeded SNR sweep on the MET stand-in falls inside the reference's confidence
interval (north_star; BASELINE configs[4]; SURVEY.md section 8(c) protocol (5)).

``standin_v2_z100`` (the z = 100 twin of the n = 10^6 stand-in: same base matrix and
schedule), SNR {0.14, 0.16, 0.18, 0.20} (the waterfall of the rate-0.1 code), 512
frames per point, early termination, 50-iteration cap.  The C oracle (the reference
decoder restated in FP64) decodes the reference's own PCG64 frames
(``frame_rng(seed, snr_idx, frame)``); the device FP32 campaign runs once on those same
frames (host channel) and once on device-drawn Philox frames (device channel, the frame
pool).  Every device FER must lie within the reference acceptance test's interval
``1.96 * sqrt(p1 (1 - p1) / N + p2 (1 - p2) / N)``
(``/root/reference/pkg/tests/test_acceptance.py:190-196,236``); frame errors are
counted as in ``/root/reference/pkg/src/qcldpc/bench.py:236-238``.
"""

import json
import math

import numpy as np
import pytest

from conftest import CODES, channel_llrs, load_code

pytestmark = pytest.mark.gpu

SNRS = (0.14, 0.16, 0.18, 0.20)
FRAMES = 512
SEED = 20241017
CAP = 50


def ci(p1, p2, n):
    return 1.96 * math.sqrt(p1 * (1 - p1) / n + p2 * (1 - p2) / n)


@pytest.fixture(scope="module")
def table():
    from oracle import oracle
    from paper_2004_09084_b200.campaign import CampaignConfig, run_campaign

    base, sched, index = load_code("standin_v2_z100")
    n = base.n_cols * base.z
    code = oracle.OracleCode(index, sched)
    rows = []
    common = dict(matrix_path=str(CODES / "standin_v2_z100.txt"), snr_list=SNRS, max_iterations=CAP,
                  early_termination=True, batch_size=64, min_trials=FRAMES, seed=SEED, precision="fp32")
    host = run_campaign(CampaignConfig(channel="host", **common))
    dev = run_campaign(CampaignConfig(channel="device", **common))
    for i, snr in enumerate(SNRS):
        llr = channel_llrs(n, snr, SEED, i, FRAMES)
        w, c, it = oracle.decode(code, llr, None, CAP, True)
        errors = int((~c).sum()) + int((c & w.any(axis=1)).sum())
        rows.append({
            "snr": snr, "frames": FRAMES,
            "oracle_fer": errors / FRAMES, "oracle_avg_iterations": float(it.mean()),
            "host_channel_fer": host.cells[i].fer, "host_channel_avg_iterations": host.cells[i].avg_iterations,
            "device_channel_fer": dev.cells[i].fer, "device_channel_avg_iterations": dev.cells[i].avg_iterations,
            "device_channel_mbit_s": dev.cells[i].throughput_mbits_per_s,
        })
    print(json.dumps(rows, indent=1))
    return rows


def test_host_channel_fer_inside_reference_ci(gpu, table):
    for r in table:
        p1, p2 = r["oracle_fer"], r["host_channel_fer"]
        assert abs(p1 - p2) <= ci(p1, p2, FRAMES), r


def test_device_channel_fer_inside_reference_ci(gpu, table):
    for r in table:
        p1, p2 = r["oracle_fer"], r["device_channel_fer"]
        assert abs(p1 - p2) <= ci(p1, p2, FRAMES), r


def test_sweep_is_the_waterfall(gpu, table):
    """The grid spans the code's waterfall: FER falls with SNR (both channels)."""
    fer = [r["oracle_fer"] for r in table]
    assert fer[0] > 0.9 and fer[-1] < 0.5
    assert all(a >= b for a, b in zip(fer, fer[1:]))
