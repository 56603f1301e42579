"""BASELINE configs[4]: SNR sweep 0.14-0.20 with seeded noise, FER / throughput vs the
iteration cap (1-100), early termination on, on the rate-0.1 n=1e6 stand-in.

    python tools/campaign_sweep.py [--trials 1024] [--batch 64] [--no-pool] [--out profiles/r02_campaign_sweep.json]

Device channel (Philox frames drawn on the GPU), FP32 flow engine, one campaign per
iteration cap; prints one line per (cap, snr) and writes all reports as one JSON.
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2004_09084_b200.campaign import CampaignConfig, report_to_dict, run_campaign  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--trials", type=int, default=1024)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--caps", type=int, nargs="+", default=[1, 2, 5, 10, 20, 50, 100])
ap.add_argument("--snr", type=float, nargs="+", default=[0.14, 0.15, 0.16, 0.161, 0.17, 0.18, 0.19, 0.20])
ap.add_argument("--out", default=str(ROOT / "profiles" / "r02_campaign_sweep.json"))
ap.add_argument("--no-pool", action="store_true", help="batched decodes (fused ET) instead of the frame pool")
a = ap.parse_args()
out = {"config": vars(a), "reports": {}}
for cap in a.caps:
    cfg = CampaignConfig(matrix_path=str(ROOT / "codes" / "standin_v2_z2500.txt"), snr_list=a.snr,
                         max_iterations=cap, early_termination=True, batch_size=a.batch, min_trials=a.trials,
                         seed=0, channel="device", precision="fp32", frame_pool=not a.no_pool)
    t0 = time.time()
    rep = run_campaign(cfg)
    out["reports"][str(cap)] = report_to_dict(rep)
    for c in rep.cells:
        print(f"cap {cap:3d} snr {c.snr:.3f}: FER {c.fer:.4f} avg it {c.avg_iterations:6.2f} "
              f"{c.throughput_mbits_per_s:8.1f} Mbit/s", flush=True)
    print(f"  ({time.time() - t0:.1f} s)", flush=True)
Path(a.out).write_text(json.dumps(out, indent=1) + "\n")
