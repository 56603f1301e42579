"""ET decode (no frame converges: SNR 0.14, cap 20, 64 codewords): total device time vs the
flow launches' own time (engine 6 records CUDA events around every sweep's launch)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2004_09084_b200 as q  # noqa: E402
from paper_2004_09084_b200 import _native  # noqa: E402

base = q.load_base_matrix(ROOT / "codes" / "standin_v2_z2500.txt")
sched = q.greedy_schedule(base)
plan = _native.Plan(q.build_compact_index(base, sched), sched, 0)
for engine in (4, 6):
    st = _native.State(plan, 64, "fp32")
    st.set_engine(engine)
    st.set_llr_synthetic(seed=0, snr_idx=0, first_frame=0, snr=0.14)
    st.set_syndrome(None)
    cfg = _native.make_config(q.DecoderConfig(max_iterations=20, early_termination=True), "fp32")
    st.decode(cfg)
    ms = st.decode(cfg)
    stats = st.kernel_stats() if hasattr(st, "kernel_stats") else None
    print(f"engine {engine}: decode {ms:.2f} ms = {ms / 20:.3f} ms/sweep; stats {stats}", flush=True)
