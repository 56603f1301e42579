"""Golden campaign reports FROM THE REFERENCE ITSELF (its ``qcldpc.bench.run_campaign``).

    python tests/golden/make_campaign_golden.py        # needs /root/reference/pkg/src

Writes tests/golden/campaign_*.json: the reference's report dict (schema v1) for small
campaigns on the reference's demo codes.  tests/test_campaign.py runs the same
campaigns through ``paper_2004_09084_b200.campaign`` on the GPU: on the host channel
(bit-identical PCG64 frames) FER and average iterations must match exactly on the FP64
parity path, and within the reference's confidence interval on the FP32 path and on
the device (Philox) channel.  Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_SRC = Path("/root/reference/pkg/src")
REF_CODES = Path("/root/reference/pkg/codes")
sys.path.insert(0, str(REF_SRC))

from qcldpc.bench import CampaignConfig, report_to_dict, run_campaign  # noqa: E402  (the reference)

CASES = {
    # acceptance-style waterfall (tests/test_acceptance.py:190-196 uses demo_4x8_z32, ET, 50 it)
    "campaign_demo4x8z32_et50": dict(matrix="demo_4x8_z32.txt", snr_list=(1.0, 1.4, 2.0), max_iterations=50,
                                     early_termination=True, batch_size=64, min_trials=512, seed=20240901),
    # config 1 (demo_4x8_z100, 10 it, no ET) at two SNRs
    "campaign_demo4x8z100_noet10": dict(matrix="demo_4x8_z100.txt", snr_list=(1.0, 2.5), max_iterations=10,
                                        early_termination=False, batch_size=64, min_trials=256, seed=7),
    # encode mode: random words toward their own syndromes (odd-parity sign path)
    "campaign_demo4x8z32_encode": dict(matrix="demo_4x8_z32.txt", snr_list=(1.4, 2.0), max_iterations=30,
                                       early_termination=True, batch_size=32, min_trials=256, seed=3,
                                       encode_mode=True),
}


def main():
    for name, c in CASES.items():
        c = dict(c)
        matrix = c.pop("matrix")
        cfg = CampaignConfig(matrix_path=str(REF_CODES / matrix), **c)
        rep = report_to_dict(run_campaign(cfg))
        for cell in rep["cells"]:  # timing columns are not reproducible; keep the schema
            cell["latency_per_iteration_s"] = None
            cell["throughput_mbits_per_s"] = None
        rep["metadata"]["matrix"]["path"] = matrix
        (HERE / f"{name}.json").write_text(json.dumps(rep, indent=1) + "\n")
        print(name, [(x["snr"], x["fer"], x["avg_iterations"]) for x in rep["cells"]])


if __name__ == "__main__":
    main()
