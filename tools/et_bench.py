"""Early-termination throughput (configs[4] flavour): 64 codewords of the rate-0.1 n=1e6
stand-in, device LLRs, 50 max iterations with ET, at several SNRs."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import paper_2004_09084_b200 as q  # noqa: E402
from paper_2004_09084_b200 import _native  # noqa: E402

base = q.load_base_matrix(ROOT / "codes" / "standin_v2_z2500.txt")
sched = q.greedy_schedule(base)
index = q.build_compact_index(base, sched)
plan = _native.Plan(index, sched, 0)
n = base.n_cols * base.z
B = 64
st = _native.State(plan, B, "fp32")
for snr_idx, snr in enumerate([0.161, 0.171, 0.181, 0.2]):
    st.set_llr_synthetic(seed=0, snr_idx=snr_idx, first_frame=0, snr=snr)
    st.set_syndrome(None)
    for et in (True, False):
        cfg = _native.make_config(q.DecoderConfig(max_iterations=50, early_termination=et), "fp32")
        st.decode(cfg)
        ms = min(st.decode(cfg) for _ in range(2))
        w, c, it = st.results()
        fer = float((~c | w.any(axis=1)).mean())
        print(f"snr {snr}: ET={et} {ms:.1f} ms, {B * n / ms / 1e3:.0f} Mbit/s, FER {fer:.3f}, "
              f"mean it {it.mean():.1f}", flush=True)
