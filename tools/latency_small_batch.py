"""Latency of one 50-iteration decode for 1-64 codewords (BASELINE configs[1]), flow
engine against the per-layer TMA engine.

    python tools/latency_small_batch.py
    QCL_MIN_LANES=4 python tools/latency_small_batch.py   # B < 4 padded to 4 lanes
"""
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2004_09084_b200 as q  # noqa: E402
from paper_2004_09084_b200 import _native  # noqa: E402

base = q.load_base_matrix(ROOT / "codes" / "standin_v2_z2500.txt")
sched = q.greedy_schedule(base)
plan = _native.Plan(q.build_compact_index(base, sched), sched, 0)
cfg = _native.make_config(q.DecoderConfig(max_iterations=50, early_termination=False), "fp32")
for B in (1, 2, 4, 8, 16, 32, 64):
    for engine, name in ((6, "flow"), (2, "per-layer")):
        st = _native.State(plan, B, "fp32")
        st.set_engine(engine)
        st.set_llr_synthetic(seed=0, snr_idx=0, first_frame=0, snr=0.161)
        st.set_syndrome(None)
        ms = [st.decode(cfg) for _ in range(8)][3:]
        lanes, flow = st.info()
        print(f"B={B} {name}: lanes={lanes} flow={flow} launches={st.kernel_stats()[0]}: median "
              f"{statistics.median(ms):.2f} ms (min {min(ms):.2f}) -> "
              f"{B * base.n_cols * base.z / statistics.median(ms) / 1e3:.0f} Mbit/s", flush=True)
        del st
