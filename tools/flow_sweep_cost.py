"""Per-sweep cost of a 64-codeword decode at SNR 0.14 (no frame converges) with a cap of
20: ET on (fused or per-sweep launches) against ET off, same device LLRs.

    [QCL_LIB_VARIANT=...] [QCL_FLOW_ET_FUSED=0] python tools/flow_sweep_cost.py [snr [cap]]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2004_09084_b200 as q  # noqa: E402
from paper_2004_09084_b200 import _native  # noqa: E402

base = q.load_base_matrix(ROOT / "codes" / "standin_v2_z2500.txt")
sched = q.greedy_schedule(base)
plan = _native.Plan(q.build_compact_index(base, sched), sched, 0)
st = _native.State(plan, 64, "fp32")
snr = float(sys.argv[1]) if len(sys.argv) > 1 else 0.14
cap = int(sys.argv[2]) if len(sys.argv) > 2 else 20
st.set_llr_synthetic(seed=0, snr_idx=0, first_frame=0, snr=snr)
st.set_syndrome(None)
for et in (False, True):
    cfg = _native.make_config(q.DecoderConfig(max_iterations=cap, early_termination=et), "fp32")
    st.decode(cfg)
    ms = min(st.decode(cfg) for _ in range(3))
    w, c, it = st.results()
    print(f"snr {snr} cap {cap} ET={et}: {ms:.2f} ms = {ms / cap:.3f} ms/sweep "
          f"(mean iterations {it.mean():.1f}, converged {int(c.sum())})", flush=True)
