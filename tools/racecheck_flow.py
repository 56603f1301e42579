"""Small flow-engine decodes (FP32, FP16 messages, fused ET) for compute-sanitizer racecheck.

    compute-sanitizer --tool racecheck python tools/racecheck_flow.py
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import paper_2004_09084_b200 as q  # noqa: E402

base = q.load_base_matrix(ROOT / "codes" / "standin_v2_z100.txt")
sched = q.greedy_schedule(base)
index = q.build_compact_index(base, sched)
n, m = base.n_cols * base.z, base.n_rows * base.z
rng = np.random.default_rng(0)
llr = rng.normal(0.5, 2.0, size=(16, n))
syn = (rng.random((16, m)) < 0.3).astype(np.uint8)
for precision in ("fp32", "fp32-msg16"):
    dec = q.LayeredDecoder(index, sched, q.DecoderConfig(max_iterations=2, early_termination=False),
                           precision=precision)
    w, c, it = dec.decode_batch_arrays(llr, syn)
    print(precision, "decoded", int(c.sum()), flush=True)
# fused early termination (round 2): snapshots, check items, decisions
dec = q.LayeredDecoder(index, sched, q.DecoderConfig(max_iterations=3, early_termination=True))
w, c, it = dec.decode_batch_arrays(rng.normal(2.0, 2.0, size=(16, n)), np.zeros((16, m), np.uint8))
print("fused ET decoded", int(c.sum()), flush=True)
