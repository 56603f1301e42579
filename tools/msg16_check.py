"""FP16 edge messages (precision "fp32-msg16") against FP32: converged counts, bit errors
and iterations on a few codes, then the 64-codeword n=1e6 decode time of both (bursts).

    python tools/msg16_check.py
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import paper_2004_09084_b200 as q  # noqa: E402
from paper_2004_09084_b200 import _native  # noqa: E402

def code(name):
    base = q.load_base_matrix(ROOT / "codes" / f"{name}.txt")
    sched = q.greedy_schedule(base)
    return base, sched, q.build_compact_index(base, sched)

for name, B, it, snr, et in [("standin_v2_z100", 64, 50, 0.2, True), ("standin_v2_z100", 64, 50, 0.161, False),
                              ("demo_4x8_z100", 33, 10, 1.0, True), ("standin_v2_z2500", 16, 50, 0.2, True)]:
    base, sched, index = code(name)
    n, m = base.n_cols * base.z, base.n_rows * base.z
    chan = q.ChannelConfig(snr=snr, seed=0)
    llr = np.stack([q.init_llr(q.transmit(np.zeros(n, np.uint8), chan, q.frame_rng(0, 0, i)), chan) for i in range(B)])
    cfg = q.DecoderConfig(max_iterations=it, early_termination=et)
    res = {}
    for prec in ("fp32", "fp32-msg16"):
        dec = q.LayeredDecoder(index, sched, cfg, precision=prec)
        res[prec] = dec.decode_batch_arrays(llr, np.zeros((B, m), np.uint8))
    a, b = res["fp32"], res["fp32-msg16"]
    print(f"{name} B={B} it={it} snr={snr} et={et}: conv fp32 {a[1].sum()} msg16 {b[1].sum()}; "
          f"bit errors fp32 {int(a[0].sum())} msg16 {int(b[0].sum())}; mean iters {a[2].mean():.2f} / {b[2].mean():.2f}", flush=True)

base, sched, index = code("standin_v2_z2500")
plan = _native.Plan(index, sched, 0)
n = base.n_cols * base.z
for prec in ("fp32", "fp32-msg16", "fp32", "fp32-msg16"):
    st = _native.State(plan, 64, prec)
    st.set_llr_synthetic(seed=0, snr_idx=0, first_frame=0, snr=0.161)
    st.set_syndrome(None)
    cfg = _native.make_config(q.DecoderConfig(max_iterations=50, early_termination=False), prec)
    st.decode(cfg)
    ms = [st.decode(cfg) for _ in range(5)]
    w, c, itr = st.results()
    print(f"timing {prec}: {min(ms):.2f} ms -> {64 * n / (min(ms) / 1e3) / 1e6:.0f} Mbit/s (bit errors {int(w.sum())})", flush=True)
