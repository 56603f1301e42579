"""Race stress for the flow engine: repeated decodes compared bit-for-bit with the
per-layer engine (0).  Prints the number of mismatching trials per case.

    python tools/flow_stress.py [trials]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import paper_2004_09084_b200 as q  # noqa: E402
from paper_2004_09084_b200 import _native  # noqa: E402

trials = int(sys.argv[1]) if len(sys.argv) > 1 else 10
bad_total = 0
for name, batch, iters in (("standin_v2_z100", 64, 20), ("standin_v2_z2500", 64, 6), ("standin_v2_z100", 8, 30),
                           ("standin_v2_z100", 128, 10), ("standin_v2_z100", 32, 20)):
    base = q.load_base_matrix(ROOT / "codes" / f"{name}.txt")
    sched = q.greedy_schedule(base)
    index = q.build_compact_index(base, sched)
    plan = _native.Plan(index, sched, 0)
    cfg = _native.make_config(q.DecoderConfig(max_iterations=iters, early_termination=False), "fp32")
    res = {}
    for engine in (0, 4):
        st = _native.State(plan, batch, "fp32")
        st.set_engine(engine)
        st.set_llr_synthetic(seed=3, snr_idx=0, first_frame=0, snr=0.161)
        st.set_syndrome(None)
        outs = []
        for _ in range(1 if engine == 0 else trials):
            st.decode(cfg)
            outs.append(st.download()[0])
        res[engine] = outs
    ref = res[0][0]
    bad = sum(not np.array_equal(o, ref) for o in res[4])
    bad_total += bad
    print(f"{name} B={batch} it={iters}: {bad}/{trials} trials differ from engine 0", flush=True)
print("STRESS OK" if bad_total == 0 else f"STRESS FAIL ({bad_total})", flush=True)
