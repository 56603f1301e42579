"""Short decode for ncu: 64 codewords of the rate-0.1 n=1e6 stand-in, device LLRs,
`--iters` layered iterations (default 2), FP32 (or --precision fp64).  Used by the
launch-list and full-capture commands recorded in profiles/README.md."""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2004_09084_b200 as q  # noqa: E402
from paper_2004_09084_b200 import _native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--precision", default="fp32")
ap.add_argument("--code", default="standin_v2_z2500")
ap.add_argument("--engine", type=int, default=0)
a = ap.parse_args()
base = q.load_base_matrix(ROOT / "codes" / f"{a.code}.txt")
sched = q.greedy_schedule(base)
index = q.build_compact_index(base, sched)
plan = _native.Plan(index, sched, 0)
st = _native.State(plan, a.batch, a.precision)
st.set_engine(a.engine)
st.set_llr_synthetic(seed=0, snr_idx=0, first_frame=0, snr=0.161)
st.set_syndrome(None)
cfg = _native.make_config(q.DecoderConfig(max_iterations=a.iters, early_termination=False), a.precision)
ms = st.decode(cfg)
print(f"decode {a.batch} x {a.iters} it: {ms:.3f} ms")
