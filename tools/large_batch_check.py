"""Large batches on the n=1e6 stand-in: flow engine (group blocks) vs the per-layer engine,
bit-identical words/convergence after a few iterations, and the flow timing.

    python tools/large_batch_check.py [batch ...]
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import paper_2004_09084_b200 as q  # noqa: E402
from paper_2004_09084_b200 import _native  # noqa: E402

base = q.load_base_matrix(ROOT / "codes" / "standin_v2_z2500.txt")
sched = q.greedy_schedule(base)
plan = _native.Plan(q.build_compact_index(base, sched), sched, 0)
n = base.n_cols * base.z
for batch in [int(x) for x in sys.argv[1:]] or [1024]:
    res = {}
    for engine in (0, 4):
        st = _native.State(plan, batch, "fp32")
        st.set_engine(engine)
        st.set_llr_synthetic(seed=1, snr_idx=0, first_frame=0, snr=0.2)
        st.set_syndrome(None)
        cfg = _native.make_config(q.DecoderConfig(max_iterations=4, early_termination=False), "fp32")
        ms = st.decode(cfg)
        res[engine] = (st.results(), ms)
        del st
    same = all(np.array_equal(a, b) for a, b in zip(res[0][0], res[4][0]))
    print(f"B={batch}: engines identical={same}; 4 iterations: engine 0 {res[0][1]:.1f} ms, flow {res[4][1]:.1f} ms "
          f"({batch * n / (res[4][1] / 1e3) / 1e6 * 4 / 50:.0f} Mbit/s at 50-iteration cost)", flush=True)
