"""ET decode for a launch list: 64 codewords of the n=1e6 stand-in, device LLRs at SNR
0.14 (no frame converges), `--iters` cap, early termination on (one flow launch per
sweep plus the per-sweep hard-decision/syndrome/bookkeeping kernels)."""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2004_09084_b200 as q  # noqa: E402
from paper_2004_09084_b200 import _native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--snr", type=float, default=0.14)
ap.add_argument("--sync", type=int, default=1)
a = ap.parse_args()
base = q.load_base_matrix(ROOT / "codes" / "standin_v2_z2500.txt")
sched = q.greedy_schedule(base)
index = q.build_compact_index(base, sched)
plan = _native.Plan(index, sched, 0)
st = _native.State(plan, 64, "fp32")
st.set_llr_synthetic(seed=0, snr_idx=0, first_frame=0, snr=a.snr)
cfg = _native.make_config(q.DecoderConfig(max_iterations=a.iters, early_termination=True), "fp32")
for rep in range(3):
    if a.sync:
        ms = st.decode(cfg)
    else:
        st.decode_async(cfg)
        ms = st.wait()
    print(f"ET decode {a.iters} it (sync={a.sync}): {ms:.3f} ms", flush=True)
